// K3 — sufficient-factor pack (step (1) "Decouple grad W_p into two vectors
// u_p and v_p"; Eq. 5) and the bias update of the SFB path
// (reading Z9: b += alpha * sum over all workers' error messages).
//
// The factors already exist after the layer's backward ("the vectors already
// exist"); K3 copies them into this rank's slot of the gather
// buffers (row stride padded to a multiple of 4 floats so TMA can describe
// them), optionally rounds them to TF32 (round-to-nearest, cvt.rna — the
// tensor core would otherwise truncate, reading Z12), and for U also emits the
// per-worker column sums that the bias update needs, so the bias costs M extra
// floats on the wire instead of a second pass over the gathered U.
#include "internal.h"

namespace poseidon {

namespace {

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 256 threads = 32 column lanes x 8 row groups; a block covers 128 columns.
template <bool kVec, bool kRound>
__global__ void __launch_bounds__(256) pack_colsum_kernel(const float* __restrict__ src, int64_t ld_src,
                                                          float* __restrict__ dst, int64_t ld_dst, int64_t K,
                                                          int64_t cols, float* __restrict__ colsum) {
  __shared__ float4 part[8][32];
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * 32 + lane) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c0 < cols) {
    for (int64_t k = rg; k < K; k += 8) {
      const float* s = src + k * ld_src + c0;
      float* d = dst + k * ld_dst + c0;
      float4 v;
      if (kVec) {
        v = *reinterpret_cast<const float4*>(s);
      } else {
        v.x = s[0];
        v.y = c0 + 1 < cols ? s[1] : 0.f;
        v.z = c0 + 2 < cols ? s[2] : 0.f;
        v.w = c0 + 3 < cols ? s[3] : 0.f;
      }
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      if (kRound) { v.x = tf32_rn(v.x); v.y = tf32_rn(v.y); v.z = tf32_rn(v.z); v.w = tf32_rn(v.w); }
      if (kVec) {
        *reinterpret_cast<float4*>(d) = v;
      } else {
        d[0] = v.x;
        if (c0 + 1 < cols) d[1] = v.y;
        if (c0 + 2 < cols) d[2] = v.z;
        if (c0 + 3 < cols) d[3] = v.w;
      }
    }
  }
  if (colsum == nullptr) return;
  part[rg][lane] = acc;
  __syncthreads();
  if (rg == 0 && c0 < cols) {
    float4 s = part[0][lane];
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const float4 t = part[r][lane];
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    colsum[c0] = s.x;
    if (c0 + 1 < cols) colsum[c0 + 1] = s.y;
    if (c0 + 2 < cols) colsum[c0 + 2] = s.z;
    if (c0 + 3 < cols) colsum[c0 + 3] = s.w;
  }
}

// Plain 2-D copy (+ optional rounding), float4 grid-stride over rows x cols/4.
template <bool kRound>
__global__ void __launch_bounds__(256) pack_copy_vec(const float* __restrict__ src, int64_t ld_src,
                                                     float* __restrict__ dst, int64_t ld_dst, int64_t K,
                                                     int64_t cols4) {
  const int64_t total = K * cols4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / cols4, c = (i - k * cols4) * 4;
    float4 v = *reinterpret_cast<const float4*>(src + k * ld_src + c);
    if (kRound) { v.x = tf32_rn(v.x); v.y = tf32_rn(v.y); v.z = tf32_rn(v.z); v.w = tf32_rn(v.w); }
    *reinterpret_cast<float4*>(dst + k * ld_dst + c) = v;
  }
}

template <bool kRound>
__global__ void __launch_bounds__(256) pack_copy_scalar(const float* __restrict__ src, int64_t ld_src,
                                                        float* __restrict__ dst, int64_t ld_dst, int64_t K,
                                                        int64_t cols) {
  const int64_t total = K * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / cols, c = i - k * cols;
    float v = src[k * ld_src + c];
    if (kRound) v = tf32_rn(v);
    dst[k * ld_dst + c] = v;
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

int copy_grid(int64_t items) {
  int64_t b = (items + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_pack(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int64_t K,
                        int64_t cols, bool round_tf32, float* colsum, cudaStream_t s) {
  if (K <= 0 || cols <= 0) return cudaSuccess;
  const bool vec = (ld_src % 4 == 0) && (ld_dst % 4 == 0) && (cols % 4 == 0) && aligned16(src) && aligned16(dst);
  if (colsum) {
    const dim3 grid((unsigned)((cols + 127) / 128));
    if (vec) {
      if (round_tf32) pack_colsum_kernel<true, true><<<grid, 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols, colsum);
      else pack_colsum_kernel<true, false><<<grid, 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols, colsum);
    } else {
      if (round_tf32) pack_colsum_kernel<false, true><<<grid, 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols, colsum);
      else pack_colsum_kernel<false, false><<<grid, 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols, colsum);
    }
  } else if (vec) {
    const int64_t cols4 = cols / 4;
    if (round_tf32) pack_copy_vec<true><<<copy_grid(K * cols4), 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols4);
    else pack_copy_vec<false><<<copy_grid(K * cols4), 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols4);
  } else {
    if (round_tf32) pack_copy_scalar<true><<<copy_grid(K * cols), 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols);
    else pack_copy_scalar<false><<<copy_grid(K * cols), 256, 0, s>>>(src, ld_src, dst, ld_dst, K, cols);
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
