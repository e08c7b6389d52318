// Internal declarations shared by the libposeidon translation units.
#pragma once

#include <cuda_runtime.h>

#include <utility>
#include <stdint.h>

#include <atomic>
#include <string>

#include "poseidon.h"

namespace poseidon {

// ---- error plumbing (thread-local message, status codes) ----
void set_error(const std::string& msg);
poseidon_status_t fail(poseidon_status_t code, const std::string& msg);
poseidon_status_t cuda_fail(cudaError_t e, const char* what);

extern std::atomic<uint64_t> g_launches;

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- kernels (each returns the launch error) ----

// K2: W[i] = fmaf(alpha, g[i], W[i]), i in [0, count). stats: optional 2 floats.
// K2 with the PS_ZERO_GRAD clear fused in: update W[b, e) from g[b, e), then zero g[0, padded).
bool ps_shard_update_zero_supported(const float* gbase, const float* Wbase, int64_t b);
cudaError_t launch_ps_shard_update_zero(float* gbase, float* Wbase, int64_t b, int64_t e, int64_t padded,
                                        float alpha, cudaStream_t s);
cudaError_t launch_ps_shard_update(const float* g, float* W, int64_t count, float alpha, float* stats,
                                   cudaStream_t s);
// PS with P simulated workers: W[i] = fmaf(alpha, sum_p g[p*ld + i], W[i]), i in [0,count).
cudaError_t launch_ps_sim_update(const float* g, int64_t ld, int32_t P, float* W, int64_t count,
                                 float alpha, cudaStream_t s);

// K3: transpose-pack K rows x `cols` columns of src (row stride ld_src) into dst[cols x ldk]
// (dst[c*ldk + k] = src[k*ld_src + c]); optional TF32 round-to-nearest; if colsum != NULL
// also writes colsum[c] = sum_k src[k][c] (fp32, fixed order, UNROUNDED values).
cudaError_t launch_pack_t(const float* src, int64_t ld_src, float* dst, int64_t ldk, int64_t K, int64_t cols,
                          bool round_tf32, float* colsum, cudaStream_t s);
// K3 for one SFB sync in ONE launch: U (K x M, + column sums) into u_dst [M x ldk] and V (K x N) into
// v_dst [N x ldk] (V == NULL: U only, the early-V path).
cudaError_t launch_pack_uv(const float* U, int64_t ldU, float* u_dst, int64_t M, float* colsum, const float* V,
                           int64_t ldV, float* v_dst, int64_t N, int64_t ldk, int64_t K, bool round_tf32,
                           cudaStream_t s);
// Momentum / weight decay (f4, oracle O4m):  v = mu v + lr (g + wd w);  w -= v.
// PS shard: g = gsum * inv_p.   SFB: K1 already left v_partial = mu v + lr/P * acc in V, so
// momentum_apply does v += lr*wd*w; w -= v.   Bias: g = inv_p * sum_p bs[p][m].
cudaError_t launch_ps_momentum(const float* gsum, float* W, float* V, int64_t count, float inv_p, float lr,
                               float mu, float wd, cudaStream_t s);
cudaError_t launch_momentum_apply(float* W, float* V, int64_t count, float lr_wd, cudaStream_t s);
cudaError_t launch_bias_momentum(const float* bs, int64_t ld, int32_t P, float* bias, float* vb, int64_t M,
                                 float lr, float mu, float wd, cudaStream_t s);
// bias[m] = fmaf(alpha, sum_p bs[p*ld + m], bias[m]) for m in [0, M), p in worker order.
cudaError_t launch_bias_update(const float* bs, int64_t ld, int32_t P, float* bias, int64_t M, float alpha,
                               cudaStream_t s);

// Ordering fuzz (test aid, POSEIDON_FUZZ_US): a single-thread kernel that sleeps `ns` on stream s.
cudaError_t launch_fuzz_sleep(uint32_t ns, cudaStream_t s);

// K1r: W[M x N] += alpha * sum_p sum_k Ug[p][m][k] Vg[p][n][k] on CUDA cores (fp32 FMA).
// ldm (0 = M): rows per worker block of Ug, so Ug may point at row m0 of a larger gather buffer and
// M be the number of rows of the block (SF-PS reconstructs only its master's rows).
cudaError_t launch_recon_simt(const float* Ug, const float* Vg, int32_t P, int64_t K, int64_t ldk, int64_t M,
                              int64_t N, float* W, float alpha, float beta, cudaStream_t s, int64_t ldm = 0);

// K1: the same on tcgen05 (TF32 operands, fp32 TMEM accumulators).  Returns cudaErrorNotSupported
// when TMA cannot describe the buffers.  Tensor maps are encoded per call (host only, ~us).
// Both compute W' = fmaf(alpha, acc, beta * W) (beta = 1: SGD; beta = mu: velocity update, f4).
// f4 momentum fused into K1's epilogue (2-SM kernel): v' = mu v + (lr/P) acc + lr wd w; w' = w - v'
// (pass alpha = lr/P, beta unused); vel has W's layout; vel_b (M or NULL) takes the bias the same way.
struct K1Momentum {
  float* vel;
  float* vel_b;
  float mu, lr, wd;
};
cudaError_t launch_recon_tcgen05(const float* Ug, const float* Vg, int32_t P, int64_t K, int64_t ldk, int64_t M,
                                 int64_t N, float* W, float alpha, float beta, cudaStream_t s, float* dbg = nullptr,
                                 int64_t ldm = 0, const float* bs = nullptr, float* bias = nullptr,
                                 bool* bias_done = nullptr, const K1Momentum* mom = nullptr);
// K1 on MN-major factors (round 2): U block p at U + p*ublk, k-th row at + k*ldu (M contiguous), V alike; the
// factors as the layer produced them (grad_out [K x M], input [K x N]), no transposing pack
bool recon_tcgen05_mn_supported(const float* U, int64_t ldu, int64_t ublk, const float* V, int64_t ldv, int64_t vblk,
                                int32_t P, int64_t K, int64_t M, int64_t N, const float* W);
cudaError_t launch_recon_tcgen05_mn(const float* U, int64_t ldu, int64_t ublk, const float* V, int64_t ldv,
                                    int64_t vblk, int32_t P, int64_t K, int64_t M, int64_t N, float* W, float alpha,
                                    float beta, cudaStream_t s, const float* bs = nullptr, float* bias = nullptr,
                                    bool* bias_done = nullptr, const K1Momentum* mom = nullptr,
                                    bool bias_from_u = false);
// (bs, bias, bias_done): optional plain-SGD bias update fused into K1 (bias[m] = fmaf(alpha, sum_p bs[p*M+m],
// bias[m]), bs [P][M] with M the block's row count); *bias_done tells whether the kernel took it.
bool recon_tcgen05_supported(const float* Ug, const float* Vg, int64_t ldk, int64_t M, int64_t N, const float* W);

// Launch with the stream's priority as a launch attribute: a kernel node captured into a CUDA graph keeps it
// (stream priorities are not part of a captured graph), so the sync kernels still take SMs ahead of the
// backward's kernels when a whole step is replayed (bench.py --graph).
template <typename... KArgs, typename... Args>
cudaError_t launch_prio(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributePriority;
  la[0].val.priority = prio;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace poseidon
