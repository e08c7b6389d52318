// K3 — sufficient-factor pack (step (1) "Decouple grad W_p into two vectors
// u_p and v_p"; Eq. 5) and the bias update of the SFB path
// (reading Z9: b += alpha * sum over all workers' error messages).
//
// The factors already exist after the layer's backward (grad_out G [K x M] and
// the layer input X [K x N], row-major).  K3 writes them TRANSPOSED into this
// rank's slot of the gather buffers — [M x ldk] and [N x ldk], K contiguous,
// ldk = roundup(K,4) — the K-major operands K1 reads fastest (reading D1 in
// DESIGN.md; round 2: K1 also reads MN-major factors in place, so at P = 1 the
// bench runs no K3 at all), optionally rounding to TF32 (round-to-nearest,
// cvt.rna; the tensor core would otherwise truncate, reading Z12).  For U it
// also emits the per-worker column sums sum_k G[k][m] (of the unrounded
// values) that the bias update needs, so the bias costs M floats on the wire
// instead of a second pass over the gathered U.
//
// Layout of the work (round 2; the round-1 kernel walked all K rows of a 32-column strip with 4 loads in
// flight per thread and launched U and V separately, 0.19 of HBM): a CTA transposes a 32-column x 256-k
// strip through a 256 x 33 shared tile with all 32 loads per thread in flight at once (global reads
// coalesced along the columns, writes along k), so C3's layers need one wave; U (with column sums) and V
// are packed by ONE launch (the first column blocks are U's, the rest V's).  K > 256 is split over a
// thread-block CLUSTER of up to 8 CTAs along k whose column sums are reduced through distributed shared
// memory in a fixed order (CTA rank 0..cs-1): deterministic, no atomics.
#include <algorithm>
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace poseidon {

namespace {

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

constexpr int kTileK = 256;  // k rows per tile: a CTA holds a whole 32-column x 256-k strip in flight
constexpr int kLoads = kTileK / 8;
constexpr int kMaxCluster = 8;

struct PackSeg {
  const float* src;  // K x cols, row stride ld
  int64_t ld;
  float* dst;        // cols x ldk
  int64_t cols;
  float* colsum;     // cols or NULL
  int64_t cblocks;   // ceil(cols / 32)
};

// grid (cblocks(U) + cblocks(V), cs), cluster (1, cs, 1), block (32, 8).  Each tile: 32 loads in flight per
// thread (the whole 32 x 256 strip, 32 KB per CTA), transposed through a 256 x 33 shared tile, 32 stores.
template <bool kRound>
__global__ void __launch_bounds__(256) pack_uv_kernel(PackSeg a, PackSeg b, int64_t K, int64_t ldk,
                                                      int tiles_per_cta) {
  __shared__ float tile[kTileK][33];
  __shared__ float part8[8][32];
  __shared__ float part[32];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const bool in_a = (int64_t)blockIdx.x < a.cblocks;
  const PackSeg& sg = in_a ? a : b;
  const int64_t c0 = ((int64_t)blockIdx.x - (in_a ? 0 : a.cblocks)) * 32;
  const int64_t c = c0 + tx;
  const bool want_sum = sg.colsum != nullptr;
  float acc = 0.f;
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_cta;
  for (int t = 0; t < tiles_per_cta; ++t) {
    const int64_t k0 = (t0 + t) * kTileK;
    if (k0 >= K) break;
    float v[kLoads];
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      const int64_t k = k0 + ty + 8 * i;
      v[i] = (k < K && c < sg.cols) ? __ldcs(sg.src + k * sg.ld + c) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      acc += v[i];
      tile[ty + 8 * i][tx] = v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t cc = c0 + ty + 8 * i;
      if (cc < sg.cols) {
        float* drow = sg.dst + cc * ldk;
#pragma unroll
        for (int h = 0; h < kTileK / 32; ++h) {
          const int64_t k = k0 + tx + 32 * h;
          if (k < K) {
            float x = tile[tx + 32 * h][ty + 8 * i];
            if (kRound) x = tf32_rn(x);
            drow[k] = x;   // plain store: K1 / the all-gather read the slot next (L2)
          }
        }
      }
    }
    __syncthreads();
  }
  if (!want_sum) return;   // uniform over the cluster (one segment per column block)
  // column sums of the unrounded values: rows of this CTA in a fixed order, then (K > 256) the cluster's
  // CTAs in rank order through distributed shared memory
  part8[ty][tx] = acc;
  __syncthreads();
  if (ty == 0) {
    float s = part8[0][tx];
#pragma unroll
    for (int r = 1; r < 8; ++r) s += part8[r][tx];
    part[tx] = s;
  }
  cg::cluster_group cluster = cg::this_cluster();
  if (cluster.num_blocks() == 1) {
    if (ty == 0 && c < sg.cols) sg.colsum[c] = part[tx];
    return;
  }
  cluster.sync();
  if (cluster.block_rank() == 0 && ty == 0 && c < sg.cols) {
    float s = 0.f;
    for (unsigned r = 0; r < cluster.num_blocks(); ++r) s += cluster.map_shared_rank(part, r)[tx];
    sg.colsum[c] = s;
  }
  cluster.sync();   // keep every CTA's shared memory alive until rank 0 has read it
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

static cudaError_t launch_pack(const PackSeg& a, const PackSeg& b, int64_t K, int64_t ldk, bool round_tf32,
                               cudaStream_t s) {
  const int64_t tiles_k = (K + kTileK - 1) / kTileK;
  const int cs = (int)std::min<int64_t>(kMaxCluster, tiles_k);
  const int tpc = (int)((tiles_k + cs - 1) / cs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.cblocks + b.cblocks), (unsigned)cs, 1);
  cfg.blockDim = dim3(32, 8, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)cs;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributePriority;   // kept by a captured graph node (internal.h launch_prio)
  attr[1].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = round_tf32 ? cudaLaunchKernelEx(&cfg, pack_uv_kernel<true>, a, b, K, ldk, tpc)
                             : cudaLaunchKernelEx(&cfg, pack_uv_kernel<false>, a, b, K, ldk, tpc);
  g_launches.fetch_add(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

static PackSeg seg(const float* src, int64_t ld, float* dst, int64_t cols, float* colsum) {
  return PackSeg{src, ld, dst, cols, colsum, cols > 0 ? (cols + 31) / 32 : 0};
}

cudaError_t launch_pack_t(const float* src, int64_t ld_src, float* dst, int64_t ldk, int64_t K, int64_t cols,
                          bool round_tf32, float* colsum, cudaStream_t s) {
  if (K <= 0 || cols <= 0) return cudaSuccess;
  return launch_pack(seg(src, ld_src, dst, cols, colsum), seg(nullptr, 0, nullptr, 0, nullptr), K, ldk, round_tf32, s);
}

cudaError_t launch_pack_uv(const float* U, int64_t ldU, float* u_dst, int64_t M, float* colsum, const float* V,
                           int64_t ldV, float* v_dst, int64_t N, int64_t ldk, int64_t K, bool round_tf32,
                           cudaStream_t s) {
  if (K <= 0 || (M <= 0 && N <= 0)) return cudaSuccess;
  return launch_pack(seg(U, ldU, u_dst, M, colsum), seg(V, ldV, v_dst, V ? N : 0, nullptr), K, ldk, round_tf32, s);
}

cudaError_t launch_bias_update(const float* bs, int64_t ld, int32_t P, float* bias, int64_t M, float alpha,
                               cudaStream_t s) {
  if (M <= 0 || bias == nullptr) return cudaSuccess;
  bias_update_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(bs, ld, P, bias, M, alpha);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace poseidon
