// K2n — fused one-kernel parameter-server sync over NVLink SHARP.
//
// Alg. 1's master ("Collect gradients ... Updates the part of model
// parameters ... Push updated model parameters") and Alg. 3 lines 1-3 in ONE
// kernel per layer, with the NVSwitch acting as the paper's "master node":
//   1. LSA barrier: every rank's local gradient (accumulated by autograd into
//      its symmetric-window copy) is complete and visible;
//   2. for this rank's shard [b, e): g = multimem.ld_reduce.add(G_mc + i) —
//      the switch reads and sums all P ranks' copies (the reduce-scatter);
//      W' = fmaf(alpha, g, W_local) (K2's update); multimem.st(W_mc + i, W')
//      — the switch writes the updated shard into every rank's W (the
//      all-gather);
//   3. LSA barrier: all ranks' stores landed and all reads of the local
//      gradient are done; the local gradient buffer is then zeroed for the
//      next iteration's accumulation.
// LSA barrier j only pairs block j of every rank, so block j may clear only the
// gradient elements that block j of every rank has reduced: for each owner q the
// shard-relative float4 indices i with (i mod stride) / 256 == j, at q*S + 4i
// (the owner's scalar tail is reduced by the block that owns its float4 index).
// Clearing any other element could run before the owning block of another rank
// has reduced it (the round-1 race; tests/mp_sync_check.py check 10 exposes it
// with the in-kernel fuzz below).
// Buffers live in NCCL symmetric windows (ncclMemAlloc +
// ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)); pointers come from the NCCL
// device API (ncclGetLsaMultimemPointer / ncclGetLocalPointer).
#include <nccl.h>
#include <nccl_device.h>

#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "nvls.h"

namespace poseidon {

namespace {

__device__ __forceinline__ float4 mm_ld_reduce_v4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st_v4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

struct NvlsMomentum {
  float* v;     // velocity of this rank's shard (index k - b), NULL -> plain SGD
  float inv_p, lr, mu, wd;
};

__device__ __forceinline__ float nvls_update(float w, float g, float alpha, const NvlsMomentum& m, int64_t j) {
  if (m.v == nullptr) return fmaf(alpha, g, w);
  const float v = fmaf(m.mu, m.v[j], m.lr * fmaf(m.wd, w, g * m.inv_p));
  m.v[j] = v;
  return w - v;
}

// Ordering fuzz inside the kernel (test aid, POSEIDON_FUZZ_US): after the entry barrier each CTA sleeps a
// pseudo-random time below fuzz_ns, so CTAs of different ranks (and of one rank) reach their reads in
// arbitrary order, as they do when DWBP schedules them around the backward's kernels.
__device__ __forceinline__ void cta_fuzz(uint32_t fuzz_ns, uint32_t seed, int rank) {
  if (fuzz_ns == 0) return;
  if (threadIdx.x == 0) {
    uint32_t h = seed * 0x9E3779B1u ^ (blockIdx.x * 0x85EBCA77u) ^ ((uint32_t)rank * 0xC2B2AE3Du);
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
    uint32_t left = h % fuzz_ns;
    while (left > 0) {
      const uint32_t step = left > 1000u ? 1000u : left;
      __nanosleep(step);
      left -= step;
    }
  }
  __syncthreads();
}

template <int U>
__global__ void __launch_bounds__(256) ps_nvls_kernel(const __grid_constant__ ncclDevComm comm, ncclWindow_t wg,
                                                      ncclWindow_t ww, size_t off_g, size_t off_w, int64_t b,
                                                      int64_t e, int64_t shard, int nranks, float alpha,
                                                      int zero_grad, NvlsMomentum mom, uint32_t fuzz_ns,
                                                      uint32_t fuzz_seed) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  cta_fuzz(fuzz_ns, fuzz_seed, ncclTeamLsa(comm).rank);

  const float* gmc = static_cast<const float*>(ncclGetLsaMultimemPointer(wg, off_g, comm));
  float* wmc = static_cast<float*>(ncclGetLsaMultimemPointer(ww, off_w, comm));
  const float* wloc = static_cast<const float*>(ncclGetLocalPointer(ww, off_w));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = (e - b) >> 2;  // b is 32-element aligned (shard map), so b + 4i is 16-B aligned
  // U independent switch reductions in flight per thread (each is a round trip through the NVSwitch)
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float4 g[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n4) {
        g[u] = mm_ld_reduce_v4(gmc + b + 4 * i);
        w[u] = *reinterpret_cast<const float4*>(wloc + b + 4 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n4) {
        const int64_t j = 4 * i;
        float4 v = w[u];
        v.x = nvls_update(v.x, g[u].x, alpha, mom, j + 0);
        v.y = nvls_update(v.y, g[u].y, alpha, mom, j + 1);
        v.z = nvls_update(v.z, g[u].z, alpha, mom, j + 2);
        v.w = nvls_update(v.w, g[u].w, alpha, mom, j + 3);
        mm_st_v4(wmc + b + j, v);
      }
    }
  }
  // scalar tail (e - b) % 4: reduced by the block that owns float4 index n4 (the block that clears it)
  if (blockIdx.x == (unsigned)((n4 % stride) / blockDim.x) && threadIdx.x < ((e - b) & 3)) {
    const int64_t k = b + 4 * n4 + threadIdx.x;
    mm_st(wmc + k, nvls_update(wloc[k], mm_ld_reduce(gmc + k), alpha, mom, k - b));
  }

  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  if (zero_grad) {
    // exactly the float4 indices block j of every rank reduced, in every owner's shard
    float4* gl = static_cast<float4*>(ncclGetLocalPointer(wg, off_g));
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t s4 = shard >> 2;   // S is a multiple of 32
    for (int q = 0; q < nranks; ++q)
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s4; i += stride) gl[q * s4 + i] = z;
  }
}

// K2o — one-shot PS sync of a small layer (round 2): ONE LSA barrier instead of K2n's two, for layers whose
// sync is latency-bound (a few microseconds of barrier round trips dominate; C2, C4's small convolutions).
// Every rank owns a slot [P][np] (np = roundup(n, 4)) in a symmetric scratch window, reused every iteration:
//   1. block j stores its float4 range of this rank's whole gradient into slot[rank] of every rank (peer
//      stores over NVLink, itself included);
//   2. LSA barrier j (acq_rel): block j of every rank has stored the same range;
//   3. block j sums slot[0..P-1] of its range in rank order -- the same arithmetic on every rank, so every
//      replica gets the same W -- applies W = fmaf(alpha, sum, W) to the whole layer (the update is
//      replicated, no all-gather) and clears its range of the local gradient, which only step 1 read.
// The slot of iteration t+1 is written only after the writing rank has passed another barrier kernel that
// every rank reaches only after finishing iteration t's reads (the host enables K2o only when at least two
// barrier-synced layers exist, and every rank issues the syncs in the same order).
template <int U>
__global__ void __launch_bounds__(256) ps_oneshot_kernel(const __grid_constant__ ncclDevComm comm, ncclWindow_t ws,
                                                         size_t off_s, float* __restrict__ g, float* __restrict__ W,
                                                         int64_t n, int64_t np, float alpha, uint32_t fuzz_ns,
                                                         uint32_t fuzz_seed) {
  const ncclTeam lsa = ncclTeamLsa(comm);
  const int64_t n4 = n >> 2;
  const int64_t per = (int64_t)blockDim.x * U;             // float4 per block
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < n4 ? lo + per : n4;
  const bool tail_block = blockIdx.x == gridDim.x - 1;     // also owns the scalar tail n % 4
  // 1. this rank's gradient range -> slot[rank] of every rank
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = lo + u * blockDim.x + threadIdx.x;
    if (i < hi) v[u] = reinterpret_cast<const float4*>(g)[i];
  }
  for (int d = 0; d < lsa.nRanks; ++d) {
    const int q = (lsa.rank + d) % lsa.nRanks;
    float* dst = static_cast<float*>(ncclGetLsaPointer(ws, off_s + (size_t)lsa.rank * np * 4, q));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = lo + u * blockDim.x + threadIdx.x;
      if (i < hi) reinterpret_cast<float4*>(dst)[i] = v[u];
    }
    if (tail_block && threadIdx.x < (n & 3)) dst[4 * n4 + threadIdx.x] = g[4 * n4 + threadIdx.x];
  }
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  cta_fuzz(fuzz_ns, fuzz_seed, lsa.rank);
  // 3. sum in rank order, update, clear
  const float* slot = static_cast<const float*>(ncclGetLocalPointer(ws, off_s));
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = lo + u * blockDim.x + threadIdx.x;
    if (i < hi) {
      float4 sum = reinterpret_cast<const float4*>(slot)[i];
      for (int p = 1; p < lsa.nRanks; ++p) {
        const float4 x = reinterpret_cast<const float4*>(slot + (size_t)p * np)[i];
        sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
      }
      float4 w = reinterpret_cast<float4*>(W)[i];
      w.x = fmaf(alpha, sum.x, w.x); w.y = fmaf(alpha, sum.y, w.y);
      w.z = fmaf(alpha, sum.z, w.z); w.w = fmaf(alpha, sum.w, w.w);
      reinterpret_cast<float4*>(W)[i] = w;
      reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (tail_block && threadIdx.x < (n & 3)) {
    const int64_t k = 4 * n4 + threadIdx.x;
    float sum = slot[k];
    for (int p = 1; p < lsa.nRanks; ++p) sum += slot[(size_t)p * np + k];
    W[k] = fmaf(alpha, sum, W[k]);
    g[k] = 0.f;
  }
}

struct BcastSeg {
  size_t off;   // byte offset of this rank's slot within the layer's window
  int64_t n;    // floats
};

// SFB step 2 ("Broadcast ... to all other workers") done by the NVSwitch: each rank stores its
// own factor slots once into the multicast address and the switch writes them into every rank's
// gather buffers.  Barrier first (every rank has packed its slots and finished reading the previous
// iteration's gather buffers), barrier last (every rank's stores have landed before K1 reads them).
// P2P = false: one multimem.st per 16 B (the switch replicates it to every rank);
// P2P = true: plain st.global of the same 16 B into each peer's window copy over NVLink (P-1 stores)
template <int U, bool P2P>
__global__ void __launch_bounds__(256) sfb_bcast_kernel(const __grid_constant__ ncclDevComm comm, ncclWindow_t win,
                                                        BcastSeg s0, BcastSeg s1, BcastSeg s2, uint32_t fuzz_ns,
                                                        uint32_t fuzz_seed) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  cta_fuzz(fuzz_ns, fuzz_seed, ncclTeamLsa(comm).rank);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const BcastSeg segs[3] = {s0, s1, s2};
#pragma unroll 1
  for (int sgi = 0; sgi < 3; ++sgi) {
    const BcastSeg sg = segs[sgi];
    // slots of odd length (the bias sums, M floats) start off 16-B alignment on ranks > 0: scalar head
    const int64_t head = sg.n < ((4 - ((int64_t)(sg.off >> 2) & 3)) & 3) ? sg.n : ((4 - ((int64_t)(sg.off >> 2) & 3)) & 3);
    const float* src0 = static_cast<const float*>(ncclGetLocalPointer(win, sg.off));
    const int64_t nb = sg.n - head;
    const int64_t n4 = nb >> 2;
    const float* src = src0 + head;
    if (!P2P) {
      float* dst0 = static_cast<float*>(ncclGetLsaMultimemPointer(win, sg.off, comm));
      if (blockIdx.x == 0 && threadIdx.x < head) mm_st(dst0 + threadIdx.x, src0[threadIdx.x]);
      float* dst = dst0 + head;
      for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = i0 + u * stride;
          if (i < n4) v[u] = *reinterpret_cast<const float4*>(src + 4 * i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = i0 + u * stride;
          if (i < n4) mm_st_v4(dst + 4 * i, v[u]);
        }
      }
      if (blockIdx.x == 0 && threadIdx.x < (nb & 3)) mm_st(dst + 4 * n4 + threadIdx.x, src[4 * n4 + threadIdx.x]);
    } else {
      const ncclTeam lsa = ncclTeamLsa(comm);
      for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = i0 + u * stride;
          if (i < n4) v[u] = *reinterpret_cast<const float4*>(src + 4 * i);
        }
        for (int d = 1; d < lsa.nRanks; ++d) {
          const int q = (lsa.rank + d) % lsa.nRanks;   // each rank starts with a different peer
          float* dst = static_cast<float*>(ncclGetLsaPointer(win, sg.off, q)) + head;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n4) *reinterpret_cast<float4*>(dst + 4 * i) = v[u];
          }
        }
      }
      if (blockIdx.x == 0 && (threadIdx.x < head || threadIdx.x < (nb & 3))) {
        for (int d = 1; d < lsa.nRanks; ++d) {
          const int q = (lsa.rank + d) % lsa.nRanks;
          float* dst0 = static_cast<float*>(ncclGetLsaPointer(win, sg.off, q));
          if (threadIdx.x < head) dst0[threadIdx.x] = src0[threadIdx.x];
          if (threadIdx.x < (nb & 3)) dst0[head + 4 * n4 + threadIdx.x] = src[4 * n4 + threadIdx.x];
        }
      }
    }
  }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

struct NvlsState {
  ncclDevComm dev{};
  bool dev_ok = false;
};

// POSEIDON_FUZZ_US (test aid): in-kernel CTA fuzz bound in ns, and a per-launch seed
static uint32_t fuzz_bound_ns() {
  static const uint32_t ns = [] {
    const char* v = getenv("POSEIDON_FUZZ_US");
    return v ? (uint32_t)(atof(v) * 1000.0) : 0u;
  }();
  return ns;
}
static uint32_t next_fuzz_seed() {
  static uint32_t seed = 0;
  return ++seed;
}

cudaError_t launch_ps_nvls(const NvlsState* st, ncclWindow_t wg, ncclWindow_t ww, size_t off_g, size_t off_w,
                           int64_t b, int64_t e, int64_t padded, float alpha, bool zero_grad, int max_blocks,
                           int64_t shard, float* vel, float inv_p, float lr, float mu, float wd, cudaStream_t s) {
  // The grid must be identical on every rank (block j of every rank meets at LSA barrier j), so it
  // is sized from the shard size S, not from this rank's (possibly shorter or empty) range.
  const int nranks = ncclTeamLsa(st->dev).nRanks;
  if (padded != shard * nranks || (shard & 31) != 0) return cudaErrorInvalidValue;
  const int64_t n4 = (shard + 3) / 4;
  static const int env_grid = [] {
    const char* v = getenv("POSEIDON_NVLS_GRID");
    return v ? atoi(v) : 0;
  }();
  static const int env_u = [] {
    const char* v = getenv("POSEIDON_NVLS_U");
    return v ? atoi(v) : 4;
  }();
  if (env_grid > 0 && env_grid < max_blocks) max_blocks = env_grid;
  // one pass of U float4 per thread: small layers get few CTAs (a CTA waiting at the entry barrier for
  // a slower rank occupies an SM slot the backward could use)
  const int64_t per_block = 256 * (int64_t)(env_u == 8 ? 8 : env_u == 2 ? 2 : 4);
  int blocks = (int)((n4 + per_block - 1) / per_block);
  if (blocks < 1) blocks = 1;
  if (blocks > max_blocks) blocks = max_blocks;
  NvlsMomentum mom{vel, inv_p, lr, mu, wd};
  const uint32_t fz = fuzz_bound_ns(), seed = fz ? next_fuzz_seed() : 0u;
  const int zg = zero_grad ? 1 : 0;
  auto kern = env_u == 8 ? ps_nvls_kernel<8> : env_u == 2 ? ps_nvls_kernel<2> : ps_nvls_kernel<4>;
  cudaError_t err = launch_prio(kern, dim3(blocks), dim3(256), 0, s, st->dev, wg, ww, off_g, off_w, b, e, shard, nranks,
                                alpha, zg, mom, fz, seed);
  g_launches.fetch_add(1);
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_ps_oneshot(const NvlsState* st, ncclWindow_t ws, size_t off_s, float* g, float* W, int64_t n,
                              float alpha, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  constexpr int U = 4;
  const int64_t n4 = n >> 2;
  int blocks = (int)((n4 + 256 * U - 1) / (256 * U));
  if (blocks < 1) blocks = 1;   // identical on every rank (n is)
  if (blocks > 128) return cudaErrorInvalidValue;   // one LSA barrier per block
  const uint32_t fz = fuzz_bound_ns(), seed = fz ? next_fuzz_seed() : 0u;
  cudaError_t err = launch_prio(ps_oneshot_kernel<U>, dim3(blocks), dim3(256), 0, s, st->dev, ws, off_s, g, W, n,
                                (n + 3) / 4 * 4, alpha, fz, seed);
  g_launches.fetch_add(1);
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_sfb_bcast_nvls(const NvlsState* st, ncclWindow_t win, size_t off_u, int64_t n_u, size_t off_v,
                                  int64_t n_v, size_t off_b, int64_t n_b, int max_blocks, cudaStream_t s) {
  // default: per-peer NVLink stores (measured faster than one multicast store for 8-25 MB slots,
  // profiles/collectives_r1.md); POSEIDON_SFB_BCAST=mc selects the multicast variant
  static const bool p2p = [] {
    const char* v = getenv("POSEIDON_SFB_BCAST");
    return !(v != nullptr && v[0] == 'm');
  }();
  // identical grid on every rank (the slot sizes are the same everywhere)
  const int64_t n4 = (n_u + n_v + n_b) / 4;
  int blocks = (int)((n4 + 1023) / 1024);
  if (blocks < 1) blocks = 1;
  static const int env_grid = [] {   // experiment knob: cap the broadcast's CTAs (SM share vs bandwidth)
    const char* v = getenv("POSEIDON_SFB_BCAST_GRID");
    return v ? atoi(v) : 0;
  }();
  // Default cap (tools/collective_bench.py + bench.py sweeps, profiles/collectives_r1.md): 32 CTAs move the
  // slots as fast as 128 at P = 2 and 4 and leave the SMs to the backward that DWBP overlaps them with (128
  // CTAs cost ~1% images/s in the step); with more peers to feed, 64 (P > 4; not measured: 4-GPU pool).
  const int nranks = ncclTeamLsa(st->dev).nRanks;
  int cap = env_grid > 0 ? env_grid : (p2p ? (nranks > 4 ? 64 : 32) : max_blocks);
  if (cap < max_blocks) max_blocks = cap;
  if (blocks > max_blocks) blocks = max_blocks;
  const uint32_t fz = fuzz_bound_ns(), seed = fz ? next_fuzz_seed() : 0u;
  cudaError_t err = launch_prio(p2p ? sfb_bcast_kernel<4, true> : sfb_bcast_kernel<4, false>, dim3(blocks), dim3(256),
                                0, s, st->dev, win, BcastSeg{off_u, n_u}, BcastSeg{off_v, n_v}, BcastSeg{off_b, n_b},
                                fz, seed);
  g_launches.fetch_add(1);
  return err != cudaSuccess ? err : cudaGetLastError();
}

NvlsState* nvls_create(ncclComm_t comm, int barriers, std::string* err) {
  auto* st = new NvlsState();
  ncclDevCommRequirements reqs;
  memset(&reqs, 0, sizeof(reqs));
  reqs.lsaMultimem = true;
  reqs.lsaBarrierCount = barriers;
  ncclResult_t r = ncclDevCommCreate(comm, &reqs, &st->dev);
  if (r != ncclSuccess) {
    *err = std::string("ncclDevCommCreate(lsaMultimem): ") + ncclGetErrorString(r);
    delete st;
    return nullptr;
  }
  st->dev_ok = true;
  return st;
}

void nvls_destroy(ncclComm_t comm, NvlsState* st) {
  if (!st) return;
  if (st->dev_ok) ncclDevCommDestroy(comm, &st->dev);
  delete st;
}

}  // namespace poseidon
