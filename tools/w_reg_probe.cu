// Register-path W streaming probe (round 2, K1's HBM regime): can 8 epilogue warps of a one-CTA-per-SM
// persistent kernel stream W = W + x (read + write) at the plain-copy rate if they keep several 32-column
// chunks of W loads in flight in registers, with K1's TMEM fragment layout (tcgen05.ld 16x256b: thread t
// holds rows t/4 and t/4+8 of a 16-row half, columns 8j + 2(t%4) + {0,1}, so every LDG.64 / STG.64 warp
// instruction covers 8 rows x one full 32-B sector)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/w_reg_probe tools/w_reg_probe.cu
// V3      plain coalesced LDG.128/STG.128, full occupancy (the copy ceiling for this size)
// R<D>    K1 fragment, 8 working warps (+4 idle warps like K1's producers), D chunks of loads in flight per warp
// Q8<D>   32x32b ownership with 256-bit LDG/STG (ld.global.v8.f32): 32 rows x one full sector per instr
// Q<D>    same with 32x32b ownership (thread = row, 32 consecutive columns, LDG.128): 32 rows x 16 B per instr
#include <cstdint>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int M = 4096, N = 9216, TM = 128, TN = 256, CW = 32;   // CTA tile 128 x 256, chunk 32 columns
constexpr int TILES = (M / TM) * (N / TN), CHUNKS = TN / CW;

__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float2 ldg64_ef(const float* p) {
  float2 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ void stg64_na(float* p, float2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float4 ldg128_ef(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
struct f8 { float4 a, b; };
__device__ __forceinline__ f8 ldg256_ef(const float* p) {
  f8 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y), "=f"(v.b.z), "=f"(v.b.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ void stg256_na(float* p, f8 v) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v.a.x), "f"(v.a.y),
               "f"(v.a.z), "f"(v.a.w), "f"(v.b.x), "f"(v.b.y), "f"(v.b.z), "f"(v.b.w)
               : "memory");
}
__device__ __forceinline__ void stg128_na(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// chunk sequence of one warp: tiles blockIdx.x, +gridDim.x, ...; chunks c = e, e+2, e+4, e+6 of each tile
struct Seq {
  int tile, c;
  __device__ bool valid() const { return tile < TILES; }
};
__device__ __forceinline__ Seq seq_at(int i, int e) {
  const int per = CHUNKS / 2;
  return Seq{(int)blockIdx.x + (i / per) * (int)gridDim.x, e + 2 * (i % per)};
}

// R: K1's 16x256b fragment; buf = 16 float2 per chunk
template <int D>
__global__ void __launch_bounds__(384, 1) probe_r(float* W) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) return;                      // K1's producer / MMA / relay warps
  const int e = (warp - 4) >> 2, q = (warp - 4) & 3, t0 = lane & 3, tr = lane >> 2;
  float2 buf[D][16];
  auto addr = [&](const Seq& s, int h, int k, int j) -> float* {
    const int mt = s.tile / (N / TN), nt = s.tile % (N / TN);
    const int row = mt * TM + q * 32 + h * 16 + tr + 8 * k;
    return W + (size_t)row * N + nt * TN + s.c * CW + 8 * j + 2 * t0;
  };
  auto load = [&](int i, float2 (&b)[16]) {
    const Seq s = seq_at(i, e);
    if (!s.valid()) return;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) b[h * 8 + k * 4 + j] = ldg64_ef(addr(s, h, k, j));
  };
  auto store = [&](int i, float2 (&b)[16]) {
    const Seq s = seq_at(i, e);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 v = b[h * 8 + k * 4 + j];
          v.x += 1e-3f;
          v.y += 1e-3f;
          stg64_na(addr(s, h, k, j), v);
        }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, buf[d]);
  for (int i = 0;; i += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (!seq_at(i + d, e).valid()) return;
      store(i + d, buf[d]);
      load(i + d + D, buf[d]);
    }
  }
}

// Q: thread = row (32x32b ownership), 32 consecutive columns = 8 float4 per chunk
template <int D>
__global__ void __launch_bounds__(384, 1) probe_q(float* W) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) return;
  const int e = (warp - 4) >> 2, q = (warp - 4) & 3;
  float4 buf[D][8];
  auto addr = [&](const Seq& s, int j) -> float* {
    const int mt = s.tile / (N / TN), nt = s.tile % (N / TN);
    return W + (size_t)(mt * TM + q * 32 + lane) * N + nt * TN + s.c * CW + 4 * j;
  };
  auto load = [&](int i, float4 (&b)[8]) {
    const Seq s = seq_at(i, e);
    if (!s.valid()) return;
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = ldg128_ef(addr(s, j));
  };
  auto store = [&](int i, float4 (&b)[8]) {
    const Seq s = seq_at(i, e);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v = b[j];
      v.x += 1e-3f; v.y += 1e-3f; v.z += 1e-3f; v.w += 1e-3f;
      stg128_na(addr(s, j), v);
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, buf[d]);
  for (int i = 0;; i += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (!seq_at(i + d, e).valid()) return;
      store(i + d, buf[d]);
      load(i + d + D, buf[d]);
    }
  }
}

// Q8: thread = row, 256-bit loads / stores (32 rows x one full sector per warp instruction)
template <int D>
__global__ void __launch_bounds__(384, 1) probe_q8(float* W) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) return;
  const int e = (warp - 4) >> 2, q = (warp - 4) & 3;
  f8 buf[D][4];
  auto addr = [&](const Seq& s, int j) -> float* {
    const int mt = s.tile / (N / TN), nt = s.tile % (N / TN);
    return W + (size_t)(mt * TM + q * 32 + lane) * N + nt * TN + s.c * CW + 8 * j;
  };
  auto load = [&](int i, f8 (&b)[4]) {
    const Seq s = seq_at(i, e);
    if (!s.valid()) return;
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = ldg256_ef(addr(s, j));
  };
  auto store = [&](int i, f8 (&b)[4]) {
    const Seq s = seq_at(i, e);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      f8 v = b[j];
      v.a.x += 1e-3f; v.a.y += 1e-3f; v.a.z += 1e-3f; v.a.w += 1e-3f;
      v.b.x += 1e-3f; v.b.y += 1e-3f; v.b.z += 1e-3f; v.b.w += 1e-3f;
      stg256_na(addr(s, j), v);
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, buf[d]);
  for (int i = 0;; i += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (!seq_at(i + d, e).valid()) return;
      store(i + d, buf[d]);
      load(i + d + D, buf[d]);
    }
  }
}

__global__ void v3(float4* W, size_t n4) {
  size_t base = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x;
  float4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) if (base + j * blockDim.x < n4) v[j] = W[base + j * blockDim.x];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (base + j * blockDim.x < n4) {
      v[j].x += 1e-3f; v[j].y += 1e-3f; v[j].z += 1e-3f; v[j].w += 1e-3f;
      W[base + j * blockDim.x] = v[j];
    }
}

template <class F>
void timeit(const char* name, F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 8; ++it) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  printf("%-8s %6.1f us  %5.0f GB/s  (%s)\n", name, best * 1e3, 8.0 * M * N / best / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* W;
  cudaMalloc(&W, (size_t)M * N * 4);
  cudaMemset(W, 0, (size_t)M * N * 4);
  const int grid = getenv("GRID") ? atoi(getenv("GRID")) : 148;
  // one CTA per SM, as K1 (215 KB of shared memory per CTA)
  const int smem = 200 * 1024;
#define SET(k) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
  SET(probe_r<1>); SET(probe_r<2>); SET(probe_r<3>); SET(probe_r<4>);
  SET(probe_q<1>); SET(probe_q<2>); SET(probe_q<3>);
  SET(probe_q8<1>); SET(probe_q8<2>); SET(probe_q8<3>); SET(probe_q8<4>);
  timeit("V3", [&] { v3<<<(M * N / 4 + 1023) / 1024, 256>>>((float4*)W, (size_t)M * N / 4); });
  timeit("R1", [&] { probe_r<1><<<grid, 384, smem>>>(W); });
  timeit("R2", [&] { probe_r<2><<<grid, 384, smem>>>(W); });
  timeit("R3", [&] { probe_r<3><<<grid, 384, smem>>>(W); });
  timeit("R4", [&] { probe_r<4><<<grid, 384, smem>>>(W); });
  timeit("Q1", [&] { probe_q<1><<<grid, 384, smem>>>(W); });
  timeit("Q2", [&] { probe_q<2><<<grid, 384, smem>>>(W); });
  timeit("Q3", [&] { probe_q<3><<<grid, 384, smem>>>(W); });
  timeit("Q8_1", [&] { probe_q8<1><<<grid, 384, smem>>>(W); });
  timeit("Q8_2", [&] { probe_q8<2><<<grid, 384, smem>>>(W); });
  timeit("Q8_3", [&] { probe_q8<3><<<grid, 384, smem>>>(W); });
  timeit("Q8_4", [&] { probe_q8<4><<<grid, 384, smem>>>(W); });
  return 0;
}
