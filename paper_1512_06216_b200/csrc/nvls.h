// NVLink-SHARP fused PS path (k_ps_nvls.cu): NCCL device-API state and launcher.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace poseidon {

struct NvlsState;
NvlsState* nvls_create(ncclComm_t comm, int barriers, std::string* err);
void nvls_destroy(ncclComm_t comm, NvlsState* st);
cudaError_t launch_ps_nvls(const NvlsState* st, ncclWindow_t wg, ncclWindow_t ww, size_t off_g, size_t off_w,
                           int64_t b, int64_t e, int64_t padded, float alpha, bool zero_grad, int max_blocks,
                           int64_t shard, float* vel, float inv_p, float lr, float mu, float wd, cudaStream_t s);

// One-shot PS sync of a small layer (K2o): peer stores of the local gradient into slot [P][roundup(n,4)] of
// every rank (byte offset off_s in the scratch window ws), one LSA barrier, rank-ordered sum, replicated update
// of W[0,n) and clear of g[0,n) (both local arena pointers).
cudaError_t launch_ps_oneshot(const NvlsState* st, ncclWindow_t ws, size_t off_s, float* g, float* W, int64_t n,
                              float alpha, cudaStream_t s);

// NVLS factor broadcast (SFB step 2 done by the switch): barrier; multimem.st of this rank's three
// slots (byte offsets within the layer's window, float counts); barrier.
cudaError_t launch_sfb_bcast_nvls(const NvlsState* st, ncclWindow_t win, size_t off_u, int64_t n_u, size_t off_v,
                                  int64_t n_v, size_t off_b, int64_t n_b, int max_blocks, cudaStream_t s);

}  // namespace poseidon
