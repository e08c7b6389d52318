// K3 — sufficient-factor pack (step (1) "Decouple grad W_p into two vectors
// u_p and v_p"; Eq. 5) and the bias update of the SFB path
// (reading Z9: b += alpha * sum over all workers' error messages).
//
// The factors already exist after the layer's backward (grad_out G [K x M] and
// the layer input X [K x N], row-major).  K3 writes them TRANSPOSED into this
// rank's slot of the gather buffers — [M x ldk] and [N x ldk], K contiguous,
// ldk = roundup(K,4) — because the tensor cores consume TF32 operands K-major
// (reading D1 in DESIGN.md), optionally rounding to TF32 (round-to-nearest,
// cvt.rna; the tensor core would otherwise truncate, reading Z12).  For U it
// also emits the per-worker column sums sum_k G[k][m] (of the unrounded
// values) that the bias update needs, so the bias costs M floats on the wire
// instead of a second pass over the gathered U.
//
// Transpose through a 32x33 shared tile: the global reads are coalesced along
// M (N), the writes along K.  A block owns a 32-column strip and walks all K
// rows, so the column sums are formed in a fixed order (bit-identical on
// every rank).
#include <algorithm>

#include "internal.h"

namespace poseidon {

namespace {

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// block (32, 8): x = column within the strip (load) / k within the tile (store)
template <bool kRound, bool kColsum>
__global__ void __launch_bounds__(256) pack_t_kernel(const float* __restrict__ src, int64_t ld_src,
                                                     float* __restrict__ dst, int64_t ldk, int64_t K, int64_t cols,
                                                     float* __restrict__ colsum) {
  __shared__ float tile[32][33];
  __shared__ float part[8][32];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int64_t c = c0 + tx;
  float acc = 0.f;
  // without column sums the K range is split over gridDim.y (more blocks in flight)
  const int64_t kspan = kColsum ? K : ((K + 31) / 32 + gridDim.y - 1) / gridDim.y * 32;
  const int64_t kbeg = kColsum ? 0 : (int64_t)blockIdx.y * kspan;
  const int64_t kend = kColsum ? K : (kbeg + kspan < K ? kbeg + kspan : K);
  for (int64_t k0 = kbeg; k0 < kend; k0 += 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = k0 + ty + 8 * i;
      float v = 0.f;
      if (k < kend && c < cols) v = src[k * ld_src + c];
      if (kColsum) acc += v;
      tile[ty + 8 * i][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t cc = c0 + ty + 8 * i;
      const int64_t k = k0 + tx;
      if (cc < cols && k < kend) {
        float v = tile[tx][ty + 8 * i];
        if (kRound) v = tf32_rn(v);
        dst[cc * ldk + k] = v;
      }
    }
    __syncthreads();
  }
  if (kColsum) {
    part[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && c < cols) {
      float s = part[0][tx];
#pragma unroll
      for (int r = 1; r < 8; ++r) s += part[r][tx];
      colsum[c] = s;
    }
  }
}

__global__ void __launch_bounds__(256) bias_update_kernel(const float* __restrict__ bs, int64_t ld, int P,
                                                          float* __restrict__ bias, int64_t M, float alpha) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float s = 0.f;
  for (int p = 0; p < P; ++p) s += bs[(int64_t)p * ld + m];
  bias[m] = fmaf(alpha, s, bias[m]);
}

__global__ void __launch_bounds__(256) bias_momentum_kernel(const float* __restrict__ bs, int64_t ld, int P,
                                                            float* __restrict__ bias, float* __restrict__ vb,
                                                            int64_t M, float lr, float mu, float wd) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float s = 0.f;
  for (int p = 0; p < P; ++p) s += bs[(int64_t)p * ld + m];
  const float b = bias[m];
  const float v = fmaf(mu, vb[m], lr * fmaf(wd, b, s * (1.0f / (float)P)));
  vb[m] = v;
  bias[m] = b - v;
}

}  // namespace

cudaError_t launch_bias_momentum(const float* bs, int64_t ld, int32_t P, float* bias, float* vb, int64_t M,
                                 float lr, float mu, float wd, cudaStream_t s) {
  if (M <= 0 || bias == nullptr) return cudaSuccess;
  bias_momentum_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(bs, ld, P, bias, vb, M, lr, mu, wd);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_pack_t(const float* src, int64_t ld_src, float* dst, int64_t ldk, int64_t K, int64_t cols,
                          bool round_tf32, float* colsum, cudaStream_t s) {
  if (K <= 0 || cols <= 0) return cudaSuccess;
  const int64_t cblocks = (cols + 31) / 32;
  int64_t ksplit = 1;
  if (!colsum) {  // aim for >= 4 blocks per SM
    const int64_t want = (148 * 4 + cblocks - 1) / cblocks;
    ksplit = std::max<int64_t>(1, std::min<int64_t>(want, (K + 31) / 32));
  }
  const dim3 grid((unsigned)cblocks, (unsigned)ksplit), block(32, 8);
  if (round_tf32) {
    if (colsum) pack_t_kernel<true, true><<<grid, block, 0, s>>>(src, ld_src, dst, ldk, K, cols, colsum);
    else pack_t_kernel<true, false><<<grid, block, 0, s>>>(src, ld_src, dst, ldk, K, cols, nullptr);
  } else {
    if (colsum) pack_t_kernel<false, true><<<grid, block, 0, s>>>(src, ld_src, dst, ldk, K, cols, colsum);
    else pack_t_kernel<false, false><<<grid, block, 0, s>>>(src, ld_src, dst, ldk, K, cols, nullptr);
  }
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_bias_update(const float* bs, int64_t ld, int32_t P, float* bias, int64_t M, float alpha,
                               cudaStream_t s) {
  if (M <= 0 || bias == nullptr) return cudaSuccess;
  bias_update_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(bs, ld, P, bias, M, alpha);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace poseidon
