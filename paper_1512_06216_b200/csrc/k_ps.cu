// K2 — parameter-server shard update (Alg. 1 master "Updates the part of model
// parameters for which a corresponding gradient is received"; Eq. 4
// P:L146 with alpha = -lr/P, readings Z1-Z4).
//
// HBM-bound elementwise kernel: 12 bytes per element (read g, read W, write W).
// 128-bit (float4) loads/stores, one pass with 4 float4 per thread (all loads
// in flight before use; 5.9 TB/s = 91% of measured HBM on 37.7M elements,
// profiles/microbench_r1.txt); the optional statistics (sum of squared updates, non-finite count)
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

// Coherent streaming load for the kZero variant, whose gradient buffer is cleared by the same kernel:
// no .nc (the read-only path may not alias a buffer the kernel writes) and a memory clobber, so the
// compiler keeps every clear store after the loads.
__device__ __forceinline__ float4 ld_stream_rw(const float4* p) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p)
               : "memory");
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

// One pass, no grid-stride loop: each thread owns 4 float4 (16 elements) spaced a block apart, all
// loads issued before any use (8 x 16 B in flight per thread), grid = ceil(n / 4096).
// kZero (PS_ZERO_GRAD): the kernel also clears the layer's whole padded gradient buffer zbase[0, zpad)
// for the next iteration's accumulation — each thread zeroes the shard elements it has read (through
// the same pointer, after its coherent loads), and the grid-strided rest covers [0, zb) and [ze, zpad)
// — which saves the separate memset launch.  g aliases zbase + zb there, so g is neither __restrict__
// nor read through the non-coherent path.
template <bool kStats, bool kZero>
__global__ void __launch_bounds__(256) ps_shard_sgd_kernel(float* g, float* __restrict__ W, int64_t count,
                                                            float alpha, float* stats, float* zbase, int64_t zb,
                                                            int64_t ze, int64_t zpad) {
  constexpr int U = 4;
  const int64_t n4 = count >> 2;
  float4* g4 = reinterpret_cast<float4*>(g);
  float4* W4 = reinterpret_cast<float4*>(W);
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  float4 a[U], w[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < n4) {
      a[j] = kZero ? ld_stream_rw(g4 + i) : ld_stream(g4 + i);
      w[j] = W4[i];
    }
  }
  if (kZero) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = base + (int64_t)j * blockDim.x;
      if (i < n4) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  float sq = 0.f, bad = 0.f;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < n4) {
      float4 v = w[j];
      v.x = fmaf(alpha, a[j].x, v.x); v.y = fmaf(alpha, a[j].y, v.y);
      v.z = fmaf(alpha, a[j].z, v.z); v.w = fmaf(alpha, a[j].w, v.w);
      W4[i] = v;
      if (kStats) {
        const float u[4] = {alpha * a[j].x, alpha * a[j].y, alpha * a[j].z, alpha * a[j].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) { sq = fmaf(u[k], u[k], sq); bad += isfinite(u[k]) ? 0.f : 1.f; }
      }
    }
  }
  // scalar tail (count % 4), block 0
  if (blockIdx.x == 0 && threadIdx.x < (count & 3)) {
    const int64_t t = (n4 << 2) + threadIdx.x;
    const float gt = kZero ? *static_cast<volatile float*>(g + t) : g[t];
    const float u = alpha * gt;
    W[t] = fmaf(alpha, gt, W[t]);
    if (kZero) g[t] = 0.f;
    if (kStats) { sq = fmaf(u, u, sq); bad += isfinite(u) ? 0.f : 1.f; }
  }
  if (kZero) {
    // the rest of the padded buffer: [0, zb) (zb is a multiple of 32) and [ze, zpad) (zpad = P*S,
    // a multiple of 32; ze arbitrary -> scalar up to the next multiple of 4)
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    float4* z4 = reinterpret_cast<float4*>(zbase);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = tid; i < (zb >> 2); i += nth) z4[i] = z;
    const int64_t ze4 = (ze + 3) & ~int64_t(3);
    if (tid < ze4 - ze && ze + tid < zpad) zbase[ze + tid] = 0.f;
    for (int64_t i = (ze4 >> 2) + tid; i < (zpad >> 2); i += nth) z4[i] = z;
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

// f4: v = mu v + lr (g * inv_p + wd w); w -= v   (float4 where aligned, fp32 FMA chain of O4m)
__global__ void __launch_bounds__(256) ps_momentum_kernel(const float* __restrict__ g, float* __restrict__ W,
                                                          float* __restrict__ V, int64_t count, float inv_p,
                                                          float lr, float mu, float wd) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[i];
    const float v = fmaf(mu, V[i], lr * fmaf(wd, w, g[i] * inv_p));
    V[i] = v;
    W[i] = w - v;
  }
}

__global__ void __launch_bounds__(256) momentum_apply_kernel(float* __restrict__ W, float* __restrict__ V,
                                                             int64_t count, float lr_wd) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[i];
    const float v = fmaf(lr_wd, w, V[i]);
    V[i] = v;
    W[i] = w - v;
  }
}

int grid_for(int64_t work_items, int threads) {
  const int64_t blocks = (work_items + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;  // 8 x 256 threads resident per SM
  return (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

// Ordering fuzz (POSEIDON_FUZZ_US, test aid): one thread spins for `ns` nanoseconds.
__global__ void fuzz_sleep_kernel(uint32_t ns) {
  uint32_t left = ns;
  while (left > 0) {
    const uint32_t step = left > 1000u ? 1000u : left;
    __nanosleep(step);
    left -= step;
  }
}

}  // namespace

cudaError_t launch_fuzz_sleep(uint32_t ns, cudaStream_t s) {
  fuzz_sleep_kernel<<<1, 1, 0, s>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_ps_shard_update(const float* g, float* W, int64_t count, float alpha, float* stats,
                                   cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int threads = 256;
  if (!aligned16(g) || !aligned16(W)) {
    ps_shard_sgd_scalar<<<grid_for(count, threads), threads, 0, s>>>(g, W, count, alpha);
  } else {
    const int64_t n4 = count >> 2;
    const int64_t per_block = (int64_t)threads * 4;
    const int64_t blocks = n4 > 0 ? (n4 + per_block - 1) / per_block : 1;
    const dim3 grid((unsigned)blocks);
    cudaError_t e = stats ? launch_prio(ps_shard_sgd_kernel<true, false>, grid, dim3(threads), 0, s,
                                        const_cast<float*>(g), W, count, alpha, stats, (float*)nullptr, (int64_t)0,
                                        (int64_t)0, (int64_t)0)
                          : launch_prio(ps_shard_sgd_kernel<false, false>, grid, dim3(threads), 0, s,
                                        const_cast<float*>(g), W, count, alpha, (float*)nullptr, (float*)nullptr,
                                        (int64_t)0, (int64_t)0, (int64_t)0);
    if (e != cudaSuccess) return e;
  }
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

bool ps_shard_update_zero_supported(const float* gbase, const float* Wbase, int64_t b) {
  return aligned16(gbase) && aligned16(Wbase) && (b & 3) == 0;
}

cudaError_t launch_ps_shard_update_zero(float* gbase, float* Wbase, int64_t b, int64_t e, int64_t padded,
                                        float alpha, cudaStream_t s) {
  const int threads = 256;
  const int64_t count = e > b ? e - b : 0;
  const int64_t n4 = count >> 2;
  const int64_t per_block = (int64_t)threads * 4;
  int64_t blocks = (n4 + per_block - 1) / per_block;
  const int64_t zero_blocks = ((padded - count) / 4 + per_block * 4 - 1) / (per_block * 4);  // ~16 float4 / thread
  if (blocks < zero_blocks) blocks = zero_blocks;
  if (blocks < 1) blocks = 1;
  cudaError_t err = launch_prio(ps_shard_sgd_kernel<false, true>, dim3((unsigned)blocks), dim3(threads), 0, s,
                                gbase + b, Wbase + b, count, alpha, (float*)nullptr, gbase, b, b + count, padded);
  g_launches.fetch_add(1);
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_ps_momentum(const float* gsum, float* W, float* V, int64_t count, float inv_p, float lr,
                               float mu, float wd, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  ps_momentum_kernel<<<grid_for(count, 256), 256, 0, s>>>(gsum, W, V, count, inv_p, lr, mu, wd);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_momentum_apply(float* W, float* V, int64_t count, float lr_wd, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  momentum_apply_kernel<<<grid_for(count, 256), 256, 0, s>>>(W, V, count, lr_wd);
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
