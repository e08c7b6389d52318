// Standalone probe of the tcgen05 building blocks used by K1 (debug tool, not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe tools/tc_probe.cu
// Test 1: TMEM st/ld round trip.  Test 2: one tcgen05.mma kind::tf32 M=128 N=256 K=8 with A/B in
// SWIZZLE_128B smem, for (a) MN-major operands and (b) K-major operands.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tmem_roundtrip(float* out) {
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_s;
  const int row = warp * 32 + lane;
  uint32_t v[4];
  for (int j = 0; j < 4; ++j) v[j] = __float_as_uint((float)(row * 1000 + 7 + j));
  uint32_t taddr = base + ((uint32_t)(warp * 32) << 16) + 7;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 4; ++j) out[row * 4 + j] = __uint_as_float(r[j]);
  out[512 + row] = (float)base;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// mode 0: MN-major A and B; mode 1: K-major A and B
__global__ void mma_probe(const float* A /*128x8 (m,k)*/, const float* B /*256x8 (n,k)*/, float* D, int mode,
                          uint32_t idesc_override, uint32_t mn_lbo, uint32_t mn_sbo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sbase = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sbase;               // 16 KB
  uint8_t* sb = sbase + 16384;       // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // zero then fill
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) ((float*)sbase)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    uint32_t off;
    if (mode & 1) {  // MN-major: chunk j=m/32 at j*4096; row k (128B); 16B chunk c=(m%32)/4 swizzled
      int j = m / 32, mm = m % 32, c = mm / 4;
      off = j * 4096 + k * 128 + ((c ^ (k & 7)) * 16) + (mm % 4) * 4;
    } else {          // K-major: row m (128B of k), 8-row atoms of 1 KB
      int c = k / 4;
      off = (m / 8) * 1024 + (m % 8) * 128 + ((c ^ (m % 8)) * 16) + (k % 4) * 4;
    }
    *(float*)(sa + off) = A[i];
  }
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    int n = i / 8, k = i % 8;
    uint32_t off;
    if (mode & 2) {
      int j = n / 32, nn = n % 32, c = nn / 4;
      off = j * 4096 + k * 128 + ((c ^ (k & 7)) * 16) + (nn % 4) * 4;
    } else {
      int c = k / 4;
      off = (n / 8) * 1024 + (n % 8) * 128 + ((c ^ (n % 8)) * 16) + (k % 4) * 4;
    }
    *(float*)(sb + off) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_s;
  if (warp == 0 && lane == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t ad, bd;
    if (mode & 1) { idesc |= (1u << 15); ad = desc_sw128(smem_u32(sa), mn_lbo, mn_sbo); }
    else ad = desc_sw128(smem_u32(sa), 16, 1024);
    if (mode & 2) { idesc |= (1u << 16); bd = desc_sw128(smem_u32(sb), mn_lbo, mn_sbo); }
    else bd = desc_sw128(smem_u32(sb), 16, 1024);
    if (idesc_override) idesc = idesc_override;
    uint32_t acc = 0;
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(base),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // everyone waits for the MMA
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra.uni D;\nbra.uni W;\nD:\n}\n" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 256; c += 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(base + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 4; ++j) D[row * 256 + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  float* out;
  cudaMallocManaged(&out, 1024 * 4);
  tmem_roundtrip<<<1, 128>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int j = 0; j < 4; ++j)
      if (out[r * 4 + j] != (float)(r * 1000 + 7 + j)) ++bad;
  printf("tmem roundtrip: err=%s bad=%d base=%g\n", cudaGetErrorString(e), bad, out[512]);

  std::vector<float> hA(128 * 8), hB(256 * 8);
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 5 - 2);
  for (int i = 0; i < 256 * 8; ++i) hB[i] = (float)((i * 3) % 4);
  float *A, *B, *D;
  cudaMallocManaged(&A, hA.size() * 4);
  cudaMallocManaged(&B, hB.size() * 4);
  cudaMallocManaged(&D, 128 * 256 * 4);
  for (size_t i = 0; i < hA.size(); ++i) A[i] = hA[i];
  for (size_t i = 0; i < hB.size(); ++i) B[i] = hB[i];
  cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  const uint32_t cfg[][3] = {{0, 0, 0}, {1, 4096, 1024}, {2, 4096, 1024}, {3, 4096, 1024}, {1, 1024, 4096},
                             {2, 1024, 4096}, {3, 1024, 4096}};
  for (auto& cf : cfg) {
    int mode = (int)cf[0];
    for (int i = 0; i < 128 * 256; ++i) D[i] = -99.f;
    mma_probe<<<1, 128, 50 * 1024>>>(A, B, D, mode, 0, cf[1], cf[2]);
    e = cudaDeviceSynchronize();
    double maxerr = 0, maxref = 0;
    int nz = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double ref = 0;
        for (int k = 0; k < 8; ++k) ref += (double)hA[m * 8 + k] * hB[n * 8 + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n]));
        maxref = fmax(maxref, fabs(ref));
        nz += D[m * 256 + n] != 0.f;
      }
    printf("mma A%s B%s lbo=%u sbo=%u: err=%s maxerr=%g maxref=%g nonzero=%d D[0..3]=%g %g %g %g\n",
           (mode & 1) ? "MN" : "K", (mode & 2) ? "MN" : "K", cf[1], cf[2], cudaGetErrorString(e), maxerr, maxref, nz,
           D[0], D[1], D[2], D[3]);
  }
  return 0;
}
