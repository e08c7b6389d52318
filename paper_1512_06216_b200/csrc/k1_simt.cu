// K1r — reconstruction + SGD on CUDA cores in fp32 (step (3) of SFB, P:L331:
// "Reconstruct {grad W_i} using {u_i, v_i} as in Eq. (5), and apply the
// updates locally"; Alg. 3 line 8).
//
//   W[M x N] += alpha * Ug^T Vg,   Ug: rows x M (ld ldu), Vg: rows x N (ld ldv)
//
// The 1e-5 path (fp32 FMA, no TF32 rounding).  64 x 64 output tile per
// 256-thread block, 4 x 4 outputs per thread, 16-row slabs of Ug/Vg staged in
// shared memory (both operands are M/N-contiguous, so the staging loads are
// coalesced along the row), fused epilogue W = fmaf(alpha, acc, W).
#include "internal.h"

namespace poseidon {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) recon_simt_kernel(const float* __restrict__ Ug, int64_t ldu,
                                                         const float* __restrict__ Vg, int64_t ldv, int64_t rows,
                                                         int64_t M, int64_t N, float* __restrict__ W, int64_t ldw,
                                                         float alpha) {
  __shared__ float As[TK][TM];
  __shared__ float Bs[TK][TN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < rows; k0 += TK) {
    // 16 x 64 = 1024 floats per operand, 4 per thread
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = threadIdx.x + j * 256;
      const int kk = idx >> 6, c = idx & 63;
      const int64_t r = k0 + kk;
      As[kk][c] = (r < rows && m0 + c < M) ? Ug[r * ldu + m0 + c] : 0.f;
      Bs[kk][c] = (r < rows && n0 + c < N) ? Vg[r * ldv + n0 + c] : 0.f;
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
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n < N) W[m * ldw + n] = fmaf(alpha, acc[i][j], W[m * ldw + n]);
    }
  }
}

}  // namespace

cudaError_t launch_recon_simt(const float* Ug, int64_t ldu, const float* Vg, int64_t ldv, int64_t rows,
                              int64_t M, int64_t N, float* W, int64_t ldw, float alpha, cudaStream_t s) {
  if (M <= 0 || N <= 0 || rows <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM));
  recon_simt_kernel<<<grid, 256, 0, s>>>(Ug, ldu, Vg, ldv, rows, M, N, W, ldw, alpha);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace poseidon
