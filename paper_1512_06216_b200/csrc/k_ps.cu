// K2 — parameter-server shard update (Alg. 1 master "Updates the part of model
// parameters for which a corresponding gradient is received"; Eq. 4
// P:L146 with alpha = -lr/P, readings Z1-Z4).
//
// HBM-bound elementwise kernel: 12 bytes per element (read g, read W, write W).
// 128-bit (float4) loads/stores, grid-stride, grid sized as a multiple of the
// SM count; the optional statistics (sum of squared updates, non-finite count)
// are reduced with warp shuffles, then once per block into two global floats.
#include "internal.h"

namespace poseidon {

namespace {

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void warp_stats_flush(float sq, float bad, float* stats) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ float s_sq[32], s_bad[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s_sq[warp] = sq; s_bad[warp] = bad; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    sq = lane < nw ? s_sq[lane] : 0.f;
    bad = lane < nw ? s_bad[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
      bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
      atomicAdd(stats, sq);
      atomicAdd(stats + 1, bad);
    }
  }
}

template <bool kStats>
__global__ void __launch_bounds__(256) ps_shard_sgd_kernel(const float* __restrict__ g, float* __restrict__ W,
                                                            int64_t count, float alpha, float* stats) {
  float sq = 0.f, bad = 0.f;
  const int64_t n4 = count >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* W4 = reinterpret_cast<float4*>(W);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // two independent float4 updates in flight per thread per iteration
  for (; i + stride < n4; i += 2 * stride) {
    float4 a0 = ld_stream(g4 + i), a1 = ld_stream(g4 + i + stride);
    float4 w0 = W4[i], w1 = W4[i + stride];
    w0.x = fmaf(alpha, a0.x, w0.x); w0.y = fmaf(alpha, a0.y, w0.y);
    w0.z = fmaf(alpha, a0.z, w0.z); w0.w = fmaf(alpha, a0.w, w0.w);
    w1.x = fmaf(alpha, a1.x, w1.x); w1.y = fmaf(alpha, a1.y, w1.y);
    w1.z = fmaf(alpha, a1.z, w1.z); w1.w = fmaf(alpha, a1.w, w1.w);
    W4[i] = w0; W4[i + stride] = w1;
    if (kStats) {
      const float u[8] = {alpha * a0.x, alpha * a0.y, alpha * a0.z, alpha * a0.w,
                          alpha * a1.x, alpha * a1.y, alpha * a1.z, alpha * a1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) { sq = fmaf(u[j], u[j], sq); bad += isfinite(u[j]) ? 0.f : 1.f; }
    }
  }
  for (; i < n4; i += stride) {
    float4 a0 = ld_stream(g4 + i);
    float4 w0 = W4[i];
    w0.x = fmaf(alpha, a0.x, w0.x); w0.y = fmaf(alpha, a0.y, w0.y);
    w0.z = fmaf(alpha, a0.z, w0.z); w0.w = fmaf(alpha, a0.w, w0.w);
    W4[i] = w0;
    if (kStats) {
      const float u[4] = {alpha * a0.x, alpha * a0.y, alpha * a0.z, alpha * a0.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) { sq = fmaf(u[j], u[j], sq); bad += isfinite(u[j]) ? 0.f : 1.f; }
    }
  }
  // scalar tail (count % 4)
  const int64_t t = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) {
    const float u = alpha * g[t];
    W[t] = fmaf(alpha, g[t], W[t]);
    if (kStats) { sq = fmaf(u, u, sq); bad += isfinite(u) ? 0.f : 1.f; }
  }
  if (kStats) warp_stats_flush(sq, bad, stats);
}

// Unaligned fallback (scalar, still coalesced).
__global__ void __launch_bounds__(256) ps_shard_sgd_scalar(const float* __restrict__ g, float* __restrict__ W,
                                                           int64_t count, float alpha) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    W[i] = fmaf(alpha, g[i], W[i]);
}

__global__ void __launch_bounds__(256) ps_sim_kernel(const float* __restrict__ g, int64_t ld, int P,
                                                     float* __restrict__ W, int64_t count, float alpha) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < P; ++p) s += g[(int64_t)p * ld + i];
    W[i] = fmaf(alpha, s, W[i]);
  }
}

int grid_for(int64_t work_items, int threads) {
  const int64_t blocks = (work_items + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;  // 8 x 256 threads resident per SM
  return (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

}  // namespace

cudaError_t launch_ps_shard_update(const float* g, float* W, int64_t count, float alpha, float* stats,
                                   cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int threads = 256;
  if (!aligned16(g) || !aligned16(W)) {
    ps_shard_sgd_scalar<<<grid_for(count, threads), threads, 0, s>>>(g, W, count, alpha);
  } else {
    const int64_t n4 = count >> 2;
    const int grid = grid_for(n4 > 0 ? (n4 + 1) / 2 : 1, threads);
    if (stats)
      ps_shard_sgd_kernel<true><<<grid, threads, 0, s>>>(g, W, count, alpha, stats);
    else
      ps_shard_sgd_kernel<false><<<grid, threads, 0, s>>>(g, W, count, alpha, nullptr);
  }
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_ps_sim_update(const float* g, int64_t ld, int32_t P, float* W, int64_t count,
                                 float alpha, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  ps_sim_kernel<<<grid_for(count, 256), 256, 0, s>>>(g, ld, P, W, count, alpha);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace poseidon
