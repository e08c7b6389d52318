// K1r — reconstruction + SGD on CUDA cores in fp32 (step (3) of SFB, P:L331:
// "Reconstruct {grad W_i} using {u_i, v_i} as in Eq. (5), and apply the
// updates locally"; Alg. 3 line 8).
//
//   W[M x N] += alpha * sum_p sum_k Ug[p][m][k] * Vg[p][n][k]
//   Ug: P blocks of ldm x ldk (rows [0, M) of each used: a row block of the gather buffer
//   when ldm > M, SF-PS), Vg: P blocks of N x ldk (the gather layout)
//
// The 1e-5 path (fp32 FMA, no TF32 rounding).  64 x 64 output tile per
// 256-thread block, 4 x 4 outputs per thread, 16-k slabs of Ug/Vg staged in
// shared memory (loads coalesced along k), fused epilogue W = fmaf(alpha, acc, beta * W)
// (beta = 1 for SGD; the momentum coefficient when the target is a velocity buffer).
#include "internal.h"

namespace poseidon {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) recon_simt_kernel(const float* __restrict__ Ug, const float* __restrict__ Vg,
                                                         int P, int64_t K, int64_t ldk, int64_t M, int64_t ldm,
                                                         int64_t N, float* __restrict__ W, float alpha, float beta) {
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  float acc[4][4] = {};
  for (int p = 0; p < P; ++p) {
    const float* Up = Ug + (int64_t)p * ldm * ldk;
    const float* Vp = Vg + (int64_t)p * N * ldk;
    for (int64_t k0 = 0; k0 < K; k0 += TK) {
      // 64 rows x 16 k per operand = 1024 floats, 4 per thread, coalesced along k
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = threadIdx.x + j * 256;
        const int r = idx >> 4, kk = idx & 15;
        const int64_t k = k0 + kk;
        As[kk][r] = (k < K && m0 + r < M) ? Up[(m0 + r) * ldk + k] : 0.f;
        Bs[kk][r] = (k < K && n0 + r < N) ? Vp[(n0 + r) * ldk + k] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n < N) W[m * N + n] = fmaf(alpha, acc[i][j], beta * W[m * N + n]);
    }
  }
}

}  // namespace

cudaError_t launch_recon_simt(const float* Ug, const float* Vg, int32_t P, int64_t K, int64_t ldk, int64_t M,
                              int64_t N, float* W, float alpha, float beta, cudaStream_t s, int64_t ldm) {
  if (M <= 0 || N <= 0 || K <= 0 || P <= 0) return cudaSuccess;
  if (ldm <= 0) ldm = M;
  const dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM));
  recon_simt_kernel<<<grid, 256, 0, s>>>(Ug, Vg, P, K, ldk, M, ldm, N, W, alpha, beta);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace poseidon
