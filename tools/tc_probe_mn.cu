// Probe (round 2): tcgen05.mma.kind::tf32 with MN-major operands (retry the MN-major TF32
// descriptors).  One M=128 N=256 K=8 MMA, A and/or B MN-major, for the canonical CUTLASS layouts
// (cute/atom/mma_traits_sm100.hpp make_umma_desc<Major::MN>, in 16-byte units):
//   SWIZZLE_128B : Sw<3,4,3> o ((8,n),(8,k)) : ((1,LBO),(8,SBO))   (128-B MN rows, 8 K rows per atom)
//   INTERLEAVE   : ((1,n),(8,k)) : ((X,SBO),(1,LBO))                 (8 K rows x 16 B core matrices)
// with LBO / SBO candidates, descriptor version 1, lbo_mode 0/1.  Prints max error vs the fp64 product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe_mn tools/tc_probe_mn.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Cfg {
  int a_mn, b_mn;     // operand MN-major?
  int layout;         // 2 = SWIZZLE_128B, 0 = INTERLEAVE (for the MN-major operands)
  uint32_t lbo, sbo;  // bytes
  int lbo_mode;
};

// byte offset of element (mn, k) of an MN-major operand with MN extent `mn_ext` (K = 8)
__device__ uint32_t mn_off(int mn, int k, int layout, uint32_t lbo, uint32_t sbo) {
  if (layout == 1) {                  // SWIZZLE_128B_BASE32B (CUTLASS Layout_MN_SW128_32B_Atom: the only MN-major
                                      // tf32 layout): 128-B rows (one per k), 32-B chunks XOR (k mod 4); MN
                                      // chunks of 32 at LBO, groups of 4 k rows at SBO
    int j = mn / 32, s = (mn % 32) / 8, t = mn % 8;
    return j * lbo + (k / 4) * sbo + (k % 4) * 128 + ((s ^ (k % 4)) << 5) + t * 4;
  }
  if (layout == 2) {                  // 32 tf32 per 128-B row; chunk j = mn / 32 at j * LBO; row k at 128 k
    int j = mn / 32, s = (mn % 32) / 4, t = mn % 4;
    return j * lbo + k * 128 + ((s ^ (k & 7)) << 4) + t * 4;
  }
  // INTERLEAVE: core matrix = 8 K rows x 16 B (4 MN elements); MN groups of 4 at SBO, K groups of 8 at LBO
  int g = mn / 4, t = mn % 4;
  return g * sbo + k * 16 + t * 4;
}
__device__ uint32_t k_off(int mn, int k) {   // K-major SW128 (the production layout)
  int c = k / 4;
  return (mn / 8) * 1024 + (mn % 8) * 128 + ((c ^ (mn % 8)) * 16) + (k % 4) * 4;
}
__device__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout, int lbo_mode) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)lbo_mode << 52) |
         ((uint64_t)layout << 61);
}

__global__ void probe(const float* A, const float* B, float* D, Cfg cf) {
  extern __shared__ uint8_t sm[];
  uint8_t* base8 = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = base8;            // 64 KB region
  uint8_t* sb = base8 + 65536;    // 128 KB region
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) ((float*)base8)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    *(float*)(sa + (cf.a_mn ? mn_off(m, k, cf.layout, cf.lbo, cf.sbo) : k_off(m, k))) = A[i];
  }
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    int n = i / 8, k = i % 8;
    *(float*)(sb + (cf.b_mn ? mn_off(n, k, cf.layout, cf.lbo, cf.sbo) : k_off(n, k))) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tb;
  if (warp == 0 && lane == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    if (cf.a_mn) idesc |= 1u << 15;
    if (cf.b_mn) idesc |= 1u << 16;
    uint64_t ad = cf.a_mn ? desc(smem_u32(sa), cf.lbo, cf.sbo, cf.layout, cf.lbo_mode) : desc(smem_u32(sa), 16, 1024, 2, 0);
    uint64_t bd = cf.b_mn ? desc(smem_u32(sb), cf.lbo, cf.sbo, cf.layout, cf.lbo_mode) : desc(smem_u32(sb), 16, 1024, 2, 0);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(ad), "l"(bd),
                 "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra.uni D;\n"
               "bra.uni W;\nD:\n}\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 256; c += 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 4; ++j) D[row * 256 + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  std::vector<float> hA(128 * 8), hB(256 * 8);
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 5 - 2);
  for (int i = 0; i < 256 * 8; ++i) hB[i] = (float)((i * 3) % 4 + 1);
  float *A, *B, *D;
  cudaMallocManaged(&A, hA.size() * 4);
  cudaMallocManaged(&B, hB.size() * 4);
  cudaMallocManaged(&D, 128 * 256 * 4);
  for (size_t i = 0; i < hA.size(); ++i) A[i] = hA[i];
  for (size_t i = 0; i < hB.size(); ++i) B[i] = hB[i];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  std::vector<Cfg> cfgs = {{0, 0, 2, 16, 1024, 0}};
  const uint32_t sw_lbo[] = {128, 1024, 2048, 4096, 8192};
  const uint32_t sw_sbo[] = {128, 1024, 4096};
  for (int ab = 1; ab <= 3; ++ab)
    for (uint32_t l : sw_lbo)
      for (uint32_t s : sw_sbo)
        for (int lm = 0; lm < 2; ++lm) cfgs.push_back({ab & 1, (ab >> 1) & 1, 2, l, s, lm});
  // SWIZZLE_128B_BASE32B (layout type 1): packed LBO = 8 k rows x 128 B = 1024, SBO = 4 rows = 512
  const uint32_t b32_pairs[][2] = {{1024, 512}, {512, 1024}, {4096, 512}, {1024, 128}, {128, 512}, {2048, 512}};
  for (int ab = 1; ab <= 3; ++ab)
    for (auto& pr : b32_pairs)
      for (int lm = 0; lm < 2; ++lm) cfgs.push_back({ab & 1, (ab >> 1) & 1, 1, pr[0], pr[1], lm});
  // INTERLEAVE: core matrices 128 B; MN groups at SBO (= 128 when packed), K groups at LBO (one group here)
  for (int ab = 1; ab <= 3; ++ab)
    for (int lm = 0; lm < 2; ++lm) {
      cfgs.push_back({ab & 1, (ab >> 1) & 1, 0, 4096, 128, lm});
      cfgs.push_back({ab & 1, (ab >> 1) & 1, 0, 128, 4096, lm});
    }
  for (const Cfg& cf : cfgs) {
    for (int i = 0; i < 128 * 256; ++i) D[i] = -99.f;
    probe<<<1, 128, 200 * 1024>>>(A, B, D, cf);
    cudaError_t e = cudaDeviceSynchronize();
    double maxerr = 0;
    int nz = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double ref = 0;
        for (int k = 0; k < 8; ++k) ref += (double)hA[m * 8 + k] * hB[n * 8 + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n]));
        nz += D[m * 256 + n] != 0.f;
      }
    printf("A %s B %s layout %s lbo %5u sbo %5u lbo_mode %d: %s maxerr %g nonzero %d%s\n", cf.a_mn ? "MN" : "K ",
           cf.b_mn ? "MN" : "K ", cf.layout == 2 ? "SW128" : cf.layout == 1 ? "SW128_32B" : "INTLV", cf.lbo, cf.sbo, cf.lbo_mode, cudaGetErrorString(e),
           maxerr, nz, maxerr == 0 ? "   <== EXACT" : "");
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
