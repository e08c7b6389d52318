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

}  // namespace poseidon
