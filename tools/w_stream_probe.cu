// W read-modify-write streaming probe (debug tool): how fast can a persistent kernel stream a
// 4096 x 9216 fp32 matrix through shared memory with TMA, depending on the box shape?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/w_stream_probe tools/w_stream_probe.cu -lcuda
// V1: 128B-swizzled boxes {32 cols, 128 rows} (K1's current epilogue pattern), coalesced STG write-back
// V2: unswizzled boxes {256 cols, 16 rows} (1 KB contiguous row segments), coalesced STG write-back
// V3: plain coalesced LDG/STG (no TMA, no smem)
// V4: V1's boxes, result written back into the smem slot and stored with a TMA bulk tensor store
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@P bra.uni D1;\nbra.uni W1;\nD1:\n}" ::"r"(
                   su32(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap* m, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma2d_store(const CUtensorMap* m, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m), "r"(su32(src)),
               "r"(x), "r"(y)
               : "memory");
}

constexpr int M = 4096, N = 9216, TM = 128, TN = 256;
#ifndef SLOTS_
#define SLOTS_ 8
#endif
constexpr int SLOTS = SLOTS_, CH = 16384;

__device__ int g_raster = 0;   // 0: tile t -> (t / NT, t % NT) (K1's N walk); 1: M walk; 2: contiguous tiles per CTA
__device__ __forceinline__ void tile_of(int i, int& mt, int& nt) {
  constexpr int NT = N / TN, MT = M / TM;
  if (g_raster == 1) {
    const int t = blockIdx.x + i * gridDim.x;
    mt = t % MT; nt = t / MT;
  } else if (g_raster == 2) {
    const int per = (MT * NT + gridDim.x - 1) / gridDim.x;
    const int t = blockIdx.x * per + i;
    mt = t / NT; nt = t % NT;
  } else {
    const int t = blockIdx.x + i * gridDim.x;
    mt = t / NT; nt = t % NT;
  }
}
__device__ __forceinline__ int tiles_of_cta() {
  constexpr int T = (M / TM) * (N / TN);
  if (g_raster == 2) {
    const int per = (T + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per;
    return lo >= T ? 0 : (T - lo < per ? T - lo : per);
  }
  return (T - (int)blockIdx.x + gridDim.x - 1) / gridDim.x;
}

template <int V>
__global__ void __launch_bounds__(160, 1) probe(const __grid_constant__ CUtensorMap map, float* W) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(s + SLOTS * CH);
  uint64_t* empty = full + SLOTS;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SLOTS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int my_tiles = tiles_of_cta();
  if (warp == 4) {  // loader
    if (lane == 0) {
      uint32_t g = 0;
      for (int i = 0; i < my_tiles; ++i) {
        int mt, nt;
        tile_of(i, mt, nt);
        for (int c = 0; c < 8; ++c, ++g) {
          const uint32_t slot = g % SLOTS, ph = (g / SLOTS) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_expect(&full[slot], CH);
          if (V == 1 || V == 4) tma2d(&map, &full[slot], s + slot * CH, nt * TN + c * 32, mt * TM);
          else tma2d(&map, &full[slot], s + slot * CH, nt * TN, mt * TM + c * 16);
        }
      }
    }
    return;
  }
  const int t = threadIdx.x;  // 0..127
  uint32_t g = 0;
  for (int i = 0; i < my_tiles; ++i) {
    int mt, nt;
    tile_of(i, mt, nt);
    for (int c = 0; c < 8; ++c, ++g) {
      const uint32_t slot = g % SLOTS, ph = (g / SLOTS) & 1;
      mbar_wait(&full[slot], ph);
      const uint8_t* base = s + slot * CH;
      if (V == 4) {
        const int jj = t & 7;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 16 + (t >> 3);
          float4* pv = (float4*)(base + rr * 128 + ((jj ^ (rr & 7)) << 4));
          float4 v = *pv;
          v.x += 1e-3f; v.y += 1e-3f; v.z += 1e-3f; v.w += 1e-3f;
          *pv = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t == 0) {
          tma2d_store(&map, base, nt * TN + c * 32, mt * TM);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          // allow 2 stores in flight: the store of chunk g-2 has finished reading its slot
          asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
          if (g >= 2) mbar_arrive(&empty[(g - 2) % SLOTS]);
        }
        continue;
      } else if (V == 1) {
        const int jj = t & 7;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 16 + (t >> 3);
          float4 v = *(const float4*)(base + rr * 128 + ((jj ^ (rr & 7)) << 4));
          v.x += 1e-3f; v.y += 1e-3f; v.z += 1e-3f; v.w += 1e-3f;
          *(float4*)(W + (size_t)(mt * TM + rr) * N + nt * TN + c * 32 + jj * 4) = v;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int idx = i * 128 + t;          // float4 index within 16 rows x 64 float4
          const int rr = idx >> 6, cc = idx & 63;
          float4 v = *(const float4*)(base + idx * 16);
          v.x += 1e-3f; v.y += 1e-3f; v.z += 1e-3f; v.w += 1e-3f;
          *(float4*)(W + (size_t)(mt * TM + c * 16 + rr) * N + nt * TN + cc * 4) = v;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t == 0) mbar_arrive(&empty[slot]);
    }
  }
  if (V == 4 && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

int main() {
  float* W;
  cudaMalloc(&W, (size_t)M * N * 4);
  cudaMemset(W, 0, (size_t)M * N * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m1, m2;
  cuuint64_t dims[2] = {N, M}, str[1] = {(cuuint64_t)N * 4};
  cuuint32_t b1[2] = {32, 128}, b2[2] = {256, 16}, es[2] = {1, 1};
  enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, str, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, str, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = SLOTS * CH + 2048;
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 8.0 * M * N;
  const int grid = getenv("GRID") ? atoi(getenv("GRID")) : 148;
  const int raster = getenv("RASTER") ? atoi(getenv("RASTER")) : 0;
  cudaMemcpyToSymbol(g_raster, &raster, sizeof(int));
  printf("RASTER=%d GRID=%d SLOTS=%d\n", raster, grid, SLOTS);
  for (int v = 1; v <= 4; ++v) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaEventRecord(a);
      if (v == 1) probe<1><<<grid, 160, smem>>>(m1, W);
      else if (v == 2) probe<2><<<grid, 160, smem>>>(m2, W);
      else if (v == 4) probe<4><<<grid, 160, smem>>>(m1, W);
      else v3<<<(M * N / 4 + 1023) / 1024, 256>>>((float4*)W, (size_t)M * N / 4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("V%d: %.1f us  %.0f GB/s  (%s)\n", v, best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
