// libposeidon C ABI: context, per-layer plans, NCCL communicator, DWBP
// scheduling (Alg. 2) and the two sync schemes of SACP (Alg. 3).
//
// Streams of a context:
//   producer (caller's)  K3 pack of SFB factors; ready_i recorded here
//   comm_stream          all collectives in call order (identical on every
//                        rank), plus the PS shard update K2 between the
//                        reduce-scatter and the all-gather
//   recon_stream         K1 / K1r + bias update of SFB layers, so the next
//                        layer's collective does not queue behind a GEMM
// Both library streams run at the highest priority: the tail of DWBP is the
// bottom layers' sync, which is on the critical path of the next forward.
#include <nccl.h>

#include <cstdio>
#include <deque>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"
#include "nvls.h"

namespace poseidon {

std::atomic<uint64_t> g_launches{0};

thread_local std::string t_err;

void set_error(const std::string& msg) { t_err = msg; }
poseidon_status_t fail(poseidon_status_t code, const std::string& msg) {
  set_error(msg);
  return code;
}
poseidon_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(POSEIDON_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// POSEIDON_DEBUG_SYNC=1: synchronise the library stream after every kernel launch and report the
// kernel that faulted (debugging aid for asynchronous launch failures; off in production).
// K2o (one-shot small-layer PS sync): largest layer it takes (floats); POSEIDON_ONESHOT=1 enables it
constexpr int64_t kOneShotMax = 65536;
bool knobs_oneshot() {
  static const bool on = [] {
    const char* v = getenv("POSEIDON_ONESHOT");
    return v && v[0] == '1';
  }();
  return on;
}

// experiment knob: POSEIDON_ASYNC_PACK=0 keeps K3 on the producer stream with POSEIDON_FLAG_INPLACE_FACTORS
bool knobs_async_pack() {
  static const bool on = [] {
    const char* v = getenv("POSEIDON_ASYNC_PACK");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool debug_sync_enabled() {
  static const bool on = [] {
    const char* v = getenv("POSEIDON_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  return on;
}
cudaError_t debug_sync(cudaStream_t s, const char* what) {
  if (!debug_sync_enabled()) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) fprintf(stderr, "[poseidon] %s faulted: %s\n", what, cudaGetErrorString(e));
  return e;
}

}  // namespace poseidon

using namespace poseidon;

namespace {

constexpr int RING = 8;           // iterations of events kept for statistics
constexpr int kNvlsBlocks = 128;  // max grid of the fused NVLS PS kernel = LSA barriers requested
constexpr int MAX_LAYERS = 4096;

#define CU_TRY(expr)                                      \
  do {                                                    \
    cudaError_t e_ = (expr);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);   \
  } while (0)
#define NC_TRY(expr)                                                                          \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return fail(POSEIDON_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));     \
  } while (0)

struct EvSet {
  cudaEvent_t ready = nullptr, start = nullptr, gathered = nullptr, kstart = nullptr, kend = nullptr,
              done = nullptr;
  // early input broadcast (FLAG_EARLY_V): V packed (producer stream), V broadcast done (comm stream)
  cudaEvent_t vready = nullptr, vgath = nullptr;
  // K3 pack of a factor layer: pstart recorded on the producer stream before the pack (ready after it)
  cudaEvent_t pstart = nullptr;
  bool packed = false;
  // FLAG_INPLACE_FACTORS with the pack kept: K3 runs on the sync's own stream; pend = after it (pack_ms)
  cudaEvent_t pend = nullptr;
  bool pack_async = false;
  // The events the statistics read for "collective done", "kernel start" and "kernel end".  An event
  // record costs ~1 us of stream time, so a sync records only the events whose time differs from
  // one already recorded (e.g. the fused NVLS kernel: ready, start, done) and aliases the rest.
  cudaEvent_t g_eff = nullptr, ks_eff = nullptr, ke_eff = nullptr;
};

struct Layer {
  bool registered = false;
  int kind = 0, scheme = 0, recon = POSEIDON_RECON_TF32;
  int64_t M = 0, N = 0, K = 0;
  bool has_bias = false;
  // SFB: library-owned gather buffers (rank-major, K-major blocks): Ug [P][M][ldk],
  // Vg [P][N][ldk], Bs [P][M] (per-worker column sums of U); optional staging [K][M], [K][N]
  int64_t ldk = 0;
  float *Ug = nullptr, *Vg = nullptr, *Bs = nullptr;
  // POSEIDON_FLAG_SSP1: a second gather set (sync t packs/gathers into set t % 2 while the deferred
  // update of sync t-1 still reads set (t-1) % 2)
  // sets 1..s (staleness s): xU[i], xV[i], xB[i] is gather set i + 1
  std::vector<float*> xU, xV, xB;
  // POSEIDON_FLAG_SYMM_SFB: Ug|Vg|Bs are one ncclMemAlloc buffer registered as a symmetric window
  void* symm = nullptr;
  ncclWindow_t win = nullptr;
  ncclComm_t win_comm = nullptr;
  bool bcast = false;   // POSEIDON_FLAG_NVLS_SFB: factors broadcast by the multicast kernel
  // POSEIDON_FLAG_INPLACE_MN at world > 1 (round 2): MN-major gather layout Ug [P][K][M], Vg [P][K][N] -- the
  // factors exactly as the layer wrote them; this rank's slot is filled by a copy-engine memcpy (no K3), K1
  // reads MN-major and forms the bias sums from Ug (no Bs travels)
  bool mn = false;
  // SF-PS (scheme 2, reading Z20): output rows [rb, re) this rank is the master of (O2 on the rows)
  int64_t rb = 0, re = 0;
  // FLAG_EARLY_V: this sync's V was packed and broadcast by poseidon_sfb_post_input (events in ev[v_iter])
  bool v_posted = false;
  int64_t v_iter = -1;
  float *stU = nullptr, *stV = nullptr;
  float *W = nullptr, *bias = nullptr;  // bound SFB params
  // PS: caller-owned padded flat buffers
  float *grad = nullptr, *Wps = nullptr;
  int64_t n = 0, S = 0, padded = 0, begin = 0, end = 0;
  uint32_t ps_flags = 0;
  bool in_arena = false;     // PS buffers live in the library's (symmetric) arena
  // f4 momentum / weight decay (oracle O4m): velocity of W (SFB: M x N, replicated; PS: this
  // rank's shard only) and of the bias (SFB)
  float mu = 0.f, wd = 0.f;
  float *vel = nullptr, *vel_b = nullptr;
  size_t arena_off = 0;      // byte offset of this layer in both arenas
  std::vector<float*> gsets;   // arena gradient buffers (SSP: s + 1, used round robin per sync)
  int64_t os_off = -1;         // K2o one-shot sync: byte offset of this layer's [P][np] slot in the scratch window
  // PS bucketing (poseidon_set_ps_buckets): a member layer points at its bucket; a bucket is a hidden
  // pseudo-layer over the members' contiguous arena span, synced once all members are ready
  int32_t bucket = -1;
  std::vector<int32_t> members;
  size_t members_ready = 0;
  int64_t nsync = 0;         // syncs issued so far (SSP set parity)
  // SSP (staleness s): the syncs whose updates are deferred, oldest first; the one of iteration t - s is applied
  // at this layer's hook of iteration t (or by poseidon_flush)
  struct Pend {
    int64_t iter;
    int set;
    float lr;
    float *W, *bias, *grad;
  };
  std::deque<Pend> pend;
  EvSet ev[RING];
  bool events_created = false;
  int64_t last_iter = -1;  // iteration of the latest sync
  // deferred (DWBP off) work
  bool pending = false;
  float pending_lr = 0.f;
  float* pending_W = nullptr;
  float* pending_bias = nullptr;
  float* pending_grad = nullptr;
};

struct IterRecord {
  int64_t iter = -1;
  std::vector<int32_t> layers;
  uint64_t sent = 0, recv = 0;
  cudaEvent_t bwd_end = nullptr;
  bool closed = false;
};

}  // namespace

struct poseidon_ctx {
  int rank = 0, world = 1, device = 0;
  uint32_t flags = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr, recon_stream = nullptr;
  float lr = 0.f;
  std::vector<Layer> layers;
  int64_t iter = 0;  // current (open) iteration
  IterRecord rec[RING];
  std::vector<int32_t> pending_order;  // DWBP off: hook order of deferred syncs
  // PS arena (poseidon_ps_arena): one gradient and one parameter buffer for all PS layers; NCCL
  // symmetric windows + device communicator when the fused NVLS path is enabled and available
  bool want_nvls = false;      // FLAG_NVLS_PS
  bool want_nvls_sfb = false;  // FLAG_NVLS_SFB
  bool ps_nvls = false;        // PS arena is symmetric and the device communicator exists
  std::string devcomm_error;
  float *arena_g = nullptr, *arena_w = nullptr;
  size_t arena_bytes = 0;
  bool arena_nccl_mem = false;
  ncclWindow_t win_g = nullptr, win_w = nullptr;
  std::vector<float*> arena_gx;          // SSP: gradient sets 1..s of the arena
  void* os_buf = nullptr;                // K2o one-shot scratch (symmetric window win_s)
  ncclWindow_t win_s = nullptr;
  std::vector<ncclWindow_t> win_gx;
  bool ssp = false;           // FLAG_SSP1
  int stale = 0;              // SSP staleness s (1 with FLAG_SSP1; poseidon_set_staleness)
  int64_t bucket_bytes = 0;   // poseidon_set_ps_buckets
  std::vector<Layer> buckets; // pseudo-layers, addressed as MAX_LAYERS + index in records
  NvlsState* nvls = nullptr;
  std::string nvls_error;
  // CUDA-graph capture (round 2): id of the stream-capture sequence the caller is in (0 = eager), and per event
  // the internal twin the captured waits use plus the capture id of its last record (evrec / evwait)
  unsigned long long cap_id = 0;
  std::unordered_map<cudaEvent_t, std::pair<cudaEvent_t, unsigned long long>> evmeta;
  cudaEvent_t join_ev[2] = {nullptr, nullptr};   // capture: the comm / recon streams' tails, joined at iteration_end
};

namespace {

poseidon_status_t check_ctx(poseidon_ctx_t c) {
  if (!c) return fail(POSEIDON_ERR_NOT_INITIALIZED, "context is NULL");
  return POSEIDON_OK;
}

// ---- CUDA-graph capture of a training step (round 2) ----
// An event recorded on a stream that is being captured becomes a capture-internal dependency, not a timestamp.
// While the caller captures, every event the library records is recorded twice: an internal twin (the waits use
// it, so the library's streams fork from and join the capture) and the event itself as an external event-record
// node (each replay stamps it, so the statistics stay valid).  A wait on an event last recorded outside the
// current capture (an earlier iteration) is dropped: graph launches into one stream are ordered as a whole.
// SSP keeps host-side state across iterations (which gather / gradient set a sync uses, the pending update of
// the previous iteration): a captured step would replay one fixed assignment, so SSP refuses capture.
poseidon_status_t note_capture(poseidon_ctx_t c, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &id) != cudaSuccess) {
    cudaGetLastError();
    st = cudaStreamCaptureStatusNone;
  }
  c->cap_id = (st == cudaStreamCaptureStatusActive) ? id : 0;
  if (c->cap_id && c->ssp)
    return fail(POSEIDON_ERR_UNSUPPORTED, "POSEIDON_FLAG_SSP1 steps cannot be captured into a CUDA graph");
  return POSEIDON_OK;
}
cudaError_t make_twin(poseidon_ctx_t c, cudaEvent_t ev) {
  if (!ev || c->evmeta.count(ev)) return cudaSuccess;
  cudaEvent_t tw = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&tw, cudaEventDisableTiming);
  if (e == cudaSuccess) c->evmeta[ev] = {tw, 0ull};
  return e;
}
cudaError_t evrec(poseidon_ctx_t c, cudaEvent_t ev, cudaStream_t s) {
  auto it = c->evmeta.find(ev);
  if (c->cap_id == 0 || it == c->evmeta.end()) {
    if (it != c->evmeta.end()) it->second.second = 0;
    return cudaEventRecord(ev, s);
  }
  cudaError_t e = cudaEventRecord(it->second.first, s);
  if (e != cudaSuccess) return e;
  it->second.second = c->cap_id;
  return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
}
cudaError_t evwait(poseidon_ctx_t c, cudaStream_t s, cudaEvent_t ev) {
  auto it = c->evmeta.find(ev);
  if (c->cap_id == 0 || it == c->evmeta.end()) return cudaStreamWaitEvent(s, ev, 0);
  if (it->second.second != c->cap_id) return cudaSuccess;   // recorded before this capture: already ordered
  return cudaStreamWaitEvent(s, it->second.first, 0);
}

// Asynchronous NCCL failures are sticky; they surface at the next wait_layer / iteration_end /
// get_iter_stats (include/poseidon.h "Errors").  ncclCommGetAsyncError is a host-side flag read.
poseidon_status_t check_async(poseidon_ctx_t c) {
  if (!c->comm) return POSEIDON_OK;
  ncclResult_t async_err = ncclSuccess;
  if (ncclCommGetAsyncError(c->comm, &async_err) == ncclSuccess && async_err != ncclSuccess &&
      async_err != ncclInProgress)
    return fail(POSEIDON_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(async_err));
  return POSEIDON_OK;
}

// Single-node all-pairs peer access (NVLink / NVSwitch) between the devices the ranks actually use:
// every rank's PCI bus id is all-gathered through the new communicator, mapped to this process's device
// ordinals and checked with cudaDeviceCanAccessPeer.  A peer that is not visible in this process (per-rank
// CUDA_VISIBLE_DEVICES) cannot be queried here; NCCL reaches it through CUDA IPC.  Two ranks on one GPU
// are refused.
poseidon_status_t check_peers(poseidon_ctx_t c) {
  constexpr int kId = 64;
  char mine[kId] = {0};
  CU_TRY(cudaDeviceGetPCIBusId(mine, kId, c->device));
  char* dbuf = nullptr;
  CU_TRY(cudaMalloc(&dbuf, (size_t)kId * c->world));
  std::vector<char> ids((size_t)kId * c->world);
  cudaError_t ce = cudaMemcpy(dbuf + (size_t)kId * c->rank, mine, kId, cudaMemcpyHostToDevice);
  ncclResult_t nr = ncclSuccess;
  if (ce == cudaSuccess) nr = ncclAllGather(dbuf + (size_t)kId * c->rank, dbuf, kId, ncclUint8, c->comm, c->comm_stream);
  if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaStreamSynchronize(c->comm_stream);
  if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaMemcpy(ids.data(), dbuf, ids.size(), cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (nr != ncclSuccess) return fail(POSEIDON_ERR_NCCL, std::string("peer id all-gather: ") + ncclGetErrorString(nr));
  if (ce != cudaSuccess) return cuda_fail(ce, "peer id exchange");
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    const char* id = ids.data() + (size_t)kId * q;
    if (strncmp(id, mine, kId) == 0)
      return fail(POSEIDON_ERR_UNSUPPORTED, "ranks " + std::to_string(c->rank) + " and " + std::to_string(q) +
                                                " share GPU " + std::string(mine));
    int d = -1;
    if (cudaDeviceGetByPCIBusId(&d, id) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    int ok = 0;
    CU_TRY(cudaDeviceCanAccessPeer(&ok, c->device, d));
    if (!ok)
      return fail(POSEIDON_ERR_UNSUPPORTED, "GPU " + std::string(mine) + " has no peer access to rank " +
                                                std::to_string(q) + "'s GPU " + std::string(id));
  }
  return POSEIDON_OK;
}

poseidon_status_t check_layer(poseidon_ctx_t c, int32_t id, Layer** out) {
  if (!c) return fail(POSEIDON_ERR_NOT_INITIALIZED, "context is NULL");
  if (id < 0 || id >= MAX_LAYERS) return fail(POSEIDON_ERR_INVALID_ARG, "layer_id out of range [0,4096)");
  if (id >= (int32_t)c->layers.size() || !c->layers[id].registered)
    return fail(POSEIDON_ERR_STATE, "layer " + std::to_string(id) + " is not registered");
  *out = &c->layers[id];
  return POSEIDON_OK;
}

// a record entry is a layer id or MAX_LAYERS + bucket index
Layer& resolve(poseidon_ctx_t c, int32_t id) {
  return id >= MAX_LAYERS ? c->buckets[(size_t)(id - MAX_LAYERS)] : c->layers[(size_t)id];
}

poseidon_status_t ensure_events(poseidon_ctx_t c, Layer& L) {
  if (L.events_created) return POSEIDON_OK;
  for (int i = 0; i < RING; ++i) {
    EvSet& e = L.ev[i];
    cudaEvent_t* all[] = {&e.ready, &e.start, &e.gathered, &e.kstart, &e.kend, &e.done, &e.vready, &e.vgath,
                          &e.pstart, &e.pend};
    for (cudaEvent_t* p : all) {
      CU_TRY(cudaEventCreate(p));
      CU_TRY(make_twin(c, *p));   // created now: nothing is created while a caller captures
    }
  }
  L.events_created = true;
  return POSEIDON_OK;
}

IterRecord& open_record(poseidon_ctx_t c) {
  IterRecord& r = c->rec[c->iter % RING];
  if (r.iter != c->iter) {
    r.iter = c->iter;
    r.layers.clear();
    r.sent = r.recv = 0;
    r.closed = false;
  }
  return r;
}

// The NCCL device communicator (LSA multicast team + barriers) shared by the fused NVLS PS kernel and
// the NVLS factor broadcast.  ncclDevCommCreate is collective: it is reached at the same point of the
// registration sequence on every rank (first NVLS SFB layer or the PS arena, whichever comes first).
bool ensure_devcomm(poseidon_ctx_t c) {
  if (c->nvls) return true;
  if (!c->devcomm_error.empty() || !c->comm) return false;
  c->nvls = nvls_create(c->comm, kNvlsBlocks, &c->devcomm_error);
  return c->nvls != nullptr;
}

// Ordering fuzz (SURVEY §5 "ordering-fuzz mode"; test aid, off unless POSEIDON_FUZZ_US is set): after the
// dependencies of each collective leg and each update kernel are in place, a pseudo-random sleep of up to
// POSEIDON_FUZZ_US microseconds on the stream about to run it.  Results must not change
// (tests/test_gpu_dwbp.py): only timing moves.
poseidon_status_t fuzz(cudaStream_t s) {
  static const uint32_t max_ns = [] {
    const char* v = getenv("POSEIDON_FUZZ_US");
    return v ? (uint32_t)(atof(v) * 1000.0) : 0u;
  }();
  if (max_ns == 0) return POSEIDON_OK;
  static uint64_t state = 0x9E3779B97F4A7C15ull;
  state = state * 6364136223846793005ull + 1442695040888963407ull;
  CU_TRY(launch_fuzz_sleep((uint32_t)((state >> 33) % max_ns), s));
  return POSEIDON_OK;
}
#define FZ(stream)                          \
  do {                                      \
    poseidon_status_t fz_ = fuzz(stream);   \
    if (fz_) return fz_;                    \
  } while (0)

// Producer-side prologue shared by both schemes: the previous sync of this
// layer must be finished before its buffers are rewritten.
poseidon_status_t producer_guard(poseidon_ctx_t c, Layer& L, cudaStream_t producer) {
  if (L.last_iter >= 0) CU_TRY(evwait(c, producer, L.ev[L.last_iter % RING].done));
  return POSEIDON_OK;
}

struct GatherSet {
  float *U, *V, *B;
};
GatherSet gather_set(const Layer& L, int set) {
  return set ? GatherSet{L.xU[(size_t)set - 1], L.xV[(size_t)set - 1], L.xB[(size_t)set - 1]}
             : GatherSet{L.Ug, L.Vg, L.Bs};
}
// floats of one rank's U / V / bias-sum slot in the gather buffers (K-major or, L.mn, MN-major)
size_t slot_u(const Layer& L) { return L.mn ? (size_t)(L.K * L.M) : (size_t)(L.M * L.ldk); }
size_t slot_v(const Layer& L) { return L.mn ? (size_t)(L.K * L.N) : (size_t)(L.N * L.ldk); }
size_t slot_b(const Layer& L) { return L.mn ? 0 : (size_t)L.M; }

// the gather set the next sync of this layer packs into (always 0 without SSP)
int next_set(poseidon_ctx_t c, const Layer& L) { return c->ssp ? (int)(L.nsync % (c->stale + 1)) : 0; }

// SFB step 2: broadcast every worker's factors = all-gather of gather set `set`, on the
// comm stream after `wait_ev`.  Records e.start and e.gathered.
poseidon_status_t sfb_comm(poseidon_ctx_t c, Layer& L, int set, EvSet& e, cudaEvent_t wait_ev, IterRecord& r) {
  const int P = c->world;
  const GatherSet g = gather_set(L, set);
  if (P <= 1) {   // nothing to gather: the sync starts on the reconstruction stream (one stream hop less)
    CU_TRY(evwait(c, c->recon_stream, wait_ev));
    FZ(c->recon_stream);
    CU_TRY(evrec(c, e.start, c->recon_stream));
    e.g_eff = e.start;
    return POSEIDON_OK;
  }
  CU_TRY(evwait(c, c->comm_stream, wait_ev));
  FZ(c->comm_stream);
  CU_TRY(evrec(c, e.start, c->comm_stream));
  e.g_eff = e.start;
  const size_t ucount = slot_u(L), vfull = slot_v(L), bcount = slot_b(L);
  const size_t vcount = L.v_posted ? 0 : vfull;   // early V: already broadcast during the forward pass
  const uint64_t per = (uint64_t)(ucount + vcount + bcount) * 4u;
  if (L.bcast) {
    // the paper's "broadcast" done by the NVSwitch: one multicast store of this rank's slots lands in
    // every rank's gather buffers (barrier, multimem.st, barrier; k_ps_nvls.cu)
    const size_t ub = (size_t)((char*)g.U - (char*)L.symm), vb = (size_t)((char*)g.V - (char*)L.symm),
                 bb = (size_t)((char*)g.B - (char*)L.symm);
    cudaError_t err = launch_sfb_bcast_nvls(c->nvls, L.win, ub + (size_t)c->rank * ucount * 4, (int64_t)ucount,
                                            vb + (size_t)c->rank * vfull * 4, (int64_t)vcount,
                                            bb + (size_t)c->rank * bcount * 4, (int64_t)bcount, kNvlsBlocks,
                                            c->comm_stream);
    if (err != cudaSuccess) return cuda_fail(err, "NVLS factor broadcast launch");
    r.sent += per;  // one copy into the switch
  } else {
    NC_TRY(ncclGroupStart());
    NC_TRY(ncclAllGather(g.U + (size_t)c->rank * ucount, g.U, ucount, ncclFloat32, c->comm, c->comm_stream));
    if (vcount)
      NC_TRY(ncclAllGather(g.V + (size_t)c->rank * vcount, g.V, vcount, ncclFloat32, c->comm, c->comm_stream));
    if (bcount)
      NC_TRY(ncclAllGather(g.B + (size_t)c->rank * bcount, g.B, bcount, ncclFloat32, c->comm, c->comm_stream));
    NC_TRY(ncclGroupEnd());
    r.sent += per;  // handed to NCCL once; NCCL forwards it to P-1 peers
  }
  r.recv += per * (uint64_t)(P - 1);
  CU_TRY(evrec(c, e.gathered, c->comm_stream));
  e.g_eff = e.gathered;
  return POSEIDON_OK;
}

// SFB step 3: reconstruct from gather set `set` and apply the update, on the recon stream
// after `src_g` (the set's all-gather) and `extra` (SSP: this layer's current backward is done with
// W).  Records dst.kstart / kend / done.
poseidon_status_t sfb_update(poseidon_ctx_t c, Layer& L, int set, float* W, float* bias, float lr, cudaEvent_t src_g,
                             cudaEvent_t extra, EvSet& dst) {
  const int P = c->world;
  const GatherSet g = gather_set(L, set);
  CU_TRY(evwait(c, c->recon_stream, src_g));
  if (extra) CU_TRY(evwait(c, c->recon_stream, extra));
  if (L.v_posted) CU_TRY(evwait(c, c->recon_stream, L.ev[L.v_iter % RING].vgath));
  FZ(c->recon_stream);
  // an event record costs ~1 us of stream time: record only the events whose times differ (BSP at P = 1
  // the sync's start was just recorded on this stream; with nothing after K1, its end is `done`)
  if (P <= 1 && src_g == dst.start && !extra) {
    dst.ks_eff = dst.start;
  } else {
    CU_TRY(evrec(c, dst.kstart, c->recon_stream));
    dst.ks_eff = dst.kstart;
  }
  dst.ke_eff = dst.kend;
  const float alpha = -lr / (float)P;
  cudaError_t err;
  const bool mom = (L.vel != nullptr);
  bool bias_done = false;   // K1 updates the bias with otherwise idle lanes (no extra launch)
  bool fused_mom = false;
  if (L.mn) {
    // MN-major gather (round 2): K1 on the factors as the layers wrote them; bias sums from Ug on idle lanes
    const K1Momentum km{L.vel, L.vel_b, L.mu, lr, L.wd};
    err = launch_recon_tcgen05_mn(g.U, L.M, L.K * L.M, g.V, L.N, L.K * L.N, P, L.K, L.M, L.N, W,
                                  mom ? lr / (float)P : alpha, 1.0f, c->recon_stream, nullptr, bias, &bias_done,
                                  mom ? &km : nullptr, /*bias_from_u=*/true);
    if (err != cudaSuccess) return cuda_fail(err, "MN-major reconstruct+sgd launch");
    if (bias && !bias_done) return fail(POSEIDON_ERR_STATE, "MN-major sync: bias not fused");
    dst.ke_eff = dst.done;
    if ((err = debug_sync(c->recon_stream, "K1 MN")) != cudaSuccess) return cuda_fail(err, "K1 MN");
    CU_TRY(evrec(c, dst.done, c->recon_stream));
    return POSEIDON_OK;
  }
  if (mom && L.recon == POSEIDON_RECON_TF32 && recon_tcgen05_supported(g.U, g.V, L.ldk, L.M, L.N, W)) {
    // f4 fused into K1's epilogue: W and its velocity streamed once, v' = mu v + (lr/P) acc + lr wd w,
    // w' = w - v' (16 B / element); the bias likewise on idle lanes
    const K1Momentum km{L.vel, L.vel_b, L.mu, lr, L.wd};
    err = launch_recon_tcgen05(g.U, g.V, P, L.K, L.ldk, L.M, L.N, W, lr / (float)P, 1.0f, c->recon_stream, nullptr,
                               0, g.B, bias, &bias_done, &km);
    fused_mom = (err == cudaSuccess);
    if (err == cudaErrorNotSupported) err = cudaSuccess;   // fall through to the two-pass form below
  }
  // plain SGD: W = fmaf(-lr/P, acc, W).  Momentum, two-pass form (K1r / unsupported layouts): the velocity is
  // the target, v_partial = fmaf(lr/P, acc, mu * v), then momentum_apply: v += lr*wd*w, w -= v.
  float* target = mom ? L.vel : W;
  const float a1 = mom ? (lr / (float)P) : alpha, b1 = mom ? L.mu : 1.0f;
  if (fused_mom) {
  } else if (L.recon == POSEIDON_RECON_TF32 && recon_tcgen05_supported(g.U, g.V, L.ldk, L.M, L.N, target))
    err = launch_recon_tcgen05(g.U, g.V, P, L.K, L.ldk, L.M, L.N, target, a1, b1, c->recon_stream, nullptr, 0,
                               mom ? nullptr : g.B, mom ? nullptr : bias, &bias_done);
  else
    err = launch_recon_simt(g.U, g.V, P, L.K, L.ldk, L.M, L.N, target, a1, b1, c->recon_stream);
  if (err != cudaSuccess) return cuda_fail(err, "reconstruct+sgd launch");
  if (mom && !fused_mom) {
    err = launch_momentum_apply(W, L.vel, L.M * L.N, lr * L.wd, c->recon_stream);
    if (err != cudaSuccess) return cuda_fail(err, "momentum apply launch");
  }
  if ((err = debug_sync(c->recon_stream, "K1/K1r reconstruct+sgd")) != cudaSuccess) return cuda_fail(err, "K1");
  if (bias && !bias_done)
    CU_TRY(evrec(c, dst.kend, c->recon_stream));  // kernel_ms = K1/K1r alone
  else
    dst.ke_eff = dst.done;
  if (bias && !bias_done) {
    err = mom ? launch_bias_momentum(g.B, L.M, P, bias, L.vel_b, L.M, lr, L.mu, L.wd, c->recon_stream)
              : launch_bias_update(g.B, L.M, P, bias, L.M, alpha, c->recon_stream);
    if (err != cudaSuccess) return cuda_fail(err, "bias update launch");
    if ((err = debug_sync(c->recon_stream, "bias update")) != cudaSuccess) return cuda_fail(err, "bias");
  }
  CU_TRY(evrec(c, dst.done, c->recon_stream));
  return POSEIDON_OK;
}

// POSEIDON_FLAG_INPLACE_FACTORS (round 2): at world == 1 nothing travels, so the sufficient factors are consumed
// where the backward wrote them ("the vectors already exist"): K1 reads U = dl/dy [K x M] and
// V = a_i [K x N] MN-major on the reconstruction stream (no K3 pack, no gather buffer) and its idle lanes form
// the bias sums.  The caller keeps U and V until the sync is done (the glue holds them until the layer's next wait).
bool inplace_ok(poseidon_ctx_t c, const Layer& L, const float* U, const float* V, const float* W) {
  return (c->flags & POSEIDON_FLAG_INPLACE_FACTORS) && (c->flags & POSEIDON_FLAG_INPLACE_MN) && c->world == 1 &&
         !c->ssp && !(c->flags & POSEIDON_FLAG_DWBP_OFF) && L.scheme == POSEIDON_SCHEME_SFB &&
         L.recon == POSEIDON_RECON_TF32 && !L.v_posted &&
         recon_tcgen05_mn_supported(U, L.M, L.K * L.M, V, L.N, L.K * L.N, 1, L.K, L.M, L.N, W);
}

poseidon_status_t launch_factor_sync(poseidon_ctx_t c, int32_t id, Layer& L, float* W, float* bias, float lr,
                                     cudaEvent_t wait_ev);
poseidon_status_t pack_sfb(poseidon_ctx_t c, Layer& L, const float* U, int64_t ldU, const float* V, int64_t ldV,
                           cudaStream_t producer);

// FLAG_INPLACE_FACTORS where K1 keeps the K-major gather layout (world > 1, or the in-place K1 declined): the
// pack (K3) itself reads U and V in place, on the stream the sync continues on (comm at P > 1, recon at P = 1),
// so it leaves the backward's critical path; the caller keeps U and V alive as for the in-place K1.
bool async_pack_ok(poseidon_ctx_t c, const Layer& L) {
  return (c->flags & POSEIDON_FLAG_INPLACE_FACTORS) && !c->ssp && !(c->flags & POSEIDON_FLAG_DWBP_OFF) &&
         L.scheme == POSEIDON_SCHEME_SFB && knobs_async_pack();
}

poseidon_status_t sfb_async_pack(poseidon_ctx_t c, int32_t id, Layer& L, const float* U, const float* V, float* W,
                                 float* bias, float lr, cudaStream_t producer) {
  EvSet& e = L.ev[c->iter % RING];
  CU_TRY(evrec(c, e.ready, producer));   // the factors exist
  cudaStream_t ls = c->world > 1 ? c->comm_stream : c->recon_stream;
  CU_TRY(evwait(c, ls, e.ready));
  // the previous sync of this layer (its K1 on the recon stream) must be done with the gather buffers
  if (L.last_iter >= 0) CU_TRY(evwait(c, ls, L.ev[L.last_iter % RING].done));
  poseidon_status_t st = pack_sfb(c, L, U, L.M, V, L.N, ls);
  if (st) return st;
  e.pack_async = true;
  CU_TRY(evrec(c, e.pend, ls));
  L.last_iter = c->iter;
  st = launch_factor_sync(c, id, L, W, bias, lr, e.pend);
  L.v_posted = false;
  return st;
}

poseidon_status_t sfb_inplace(poseidon_ctx_t c, int32_t id, Layer& L, const float* U, const float* V, float* W,
                              float* bias, float lr, cudaStream_t producer) {
  EvSet& e = L.ev[c->iter % RING];
  e.packed = false;
  CU_TRY(evrec(c, e.ready, producer));
  L.last_iter = c->iter;
  IterRecord& r = open_record(c);
  CU_TRY(evwait(c, c->recon_stream, e.ready));
  FZ(c->recon_stream);
  CU_TRY(evrec(c, e.start, c->recon_stream));
  e.g_eff = e.start;
  e.ks_eff = e.start;
  e.ke_eff = e.done;
  const bool mom = (L.vel != nullptr);
  const K1Momentum km{L.vel, L.vel_b, L.mu, lr, L.wd};
  bool bias_done = false;
  cudaError_t err = launch_recon_tcgen05_mn(U, L.M, L.K * L.M, V, L.N, L.K * L.N, 1, L.K, L.M, L.N, W,
                                            mom ? lr : -lr, 1.0f, c->recon_stream, nullptr, bias, &bias_done,
                                            mom ? &km : nullptr, /*bias_from_u=*/true);
  if (err != cudaSuccess) return cuda_fail(err, "in-place reconstruct+sgd launch");
  if (bias && !bias_done) return fail(POSEIDON_ERR_STATE, "in-place sync: bias not fused");
  if ((err = debug_sync(c->recon_stream, "K1 in place")) != cudaSuccess) return cuda_fail(err, "K1 in place");
  CU_TRY(evrec(c, e.done, c->recon_stream));
  r.layers.push_back(id);
  return POSEIDON_OK;
}

// BSP SFB sync (steps 2 and 3 of P:L330-331) of the current iteration.
poseidon_status_t launch_sfb_comm(poseidon_ctx_t c, int32_t id, Layer& L, float* W, float* bias, float lr,
                                  cudaEvent_t wait_ev) {
  EvSet& e = L.ev[c->iter % RING];
  IterRecord& r = open_record(c);
  poseidon_status_t st = sfb_comm(c, L, 0, e, wait_ev, r);
  if (st) return st;
  st = sfb_update(c, L, 0, W, bias, lr, e.g_eff, nullptr, e);
  if (st) return st;
  r.layers.push_back(id);
  return POSEIDON_OK;
}

// SF-PS (Alg. 3 else-branch, "Send u, v to the master node; Synchronize A_i from the
// master node"; reading Z20): the master is sharded by output rows, rank q owns rows
// [qb, qe) = poseidon_shard_range(M, P, q).  Step 1 on the comm stream: every worker sends its
// error-message rows of q's block (its U slot, rows [qb, qe), contiguous in the K-major layout) to
// master q and its inputs V to everyone (all-gather, which is "send v to every master"), plus the
// per-worker bias sums.  Records e.start and e.gathered.
poseidon_status_t sfps_comm(poseidon_ctx_t c, Layer& L, EvSet& e, cudaEvent_t wait_ev, IterRecord& r) {
  const int P = c->world;
  CU_TRY(evwait(c, c->comm_stream, wait_ev));
  FZ(c->comm_stream);
  CU_TRY(evrec(c, e.start, c->comm_stream));
  e.g_eff = e.start;
  if (P <= 1) return POSEIDON_OK;
  const size_t ucount = (size_t)(L.M * L.ldk), vcount = (size_t)(L.N * L.ldk), bcount = (size_t)L.M;
  NC_TRY(ncclGroupStart());
  NC_TRY(ncclAllGather(L.Vg + (size_t)c->rank * vcount, L.Vg, vcount, ncclFloat32, c->comm, c->comm_stream));
  NC_TRY(ncclAllGather(L.Bs + (size_t)c->rank * bcount, L.Bs, bcount, ncclFloat32, c->comm, c->comm_stream));
  NC_TRY(ncclGroupEnd());
  uint64_t sent = (uint64_t)(vcount + bcount) * 4u, recv = (uint64_t)(vcount + bcount) * 4u * (uint64_t)(P - 1);
  NC_TRY(ncclGroupStart());
  const size_t own = (size_t)(L.re - L.rb) * (size_t)L.ldk;
  for (int q = 0; q < P; ++q) {
    if (q == c->rank) continue;
    int64_t qb, qe, pad;
    poseidon_shard_range(L.M, P, q, &qb, &qe, &pad);
    if (qe > qb) {
      const size_t cnt = (size_t)(qe - qb) * (size_t)L.ldk;
      NC_TRY(ncclSend(L.Ug + (size_t)c->rank * ucount + (size_t)qb * L.ldk, cnt, ncclFloat32, q, c->comm,
                      c->comm_stream));
      sent += (uint64_t)cnt * 4u;
    }
    if (own > 0) {
      NC_TRY(ncclRecv(L.Ug + (size_t)q * ucount + (size_t)L.rb * L.ldk, own, ncclFloat32, q, c->comm,
                      c->comm_stream));
      recv += (uint64_t)own * 4u;
    }
  }
  NC_TRY(ncclGroupEnd());
  r.sent += sent;
  r.recv += recv;
  CU_TRY(evrec(c, e.gathered, c->comm_stream));
  e.g_eff = e.gathered;
  return POSEIDON_OK;
}

// SF-PS step 2: master r reconstructs only its rows, W[rb:re] += alpha * sum_p U_p[rb:re]^T V_p (K1 on
// a row block of the gather buffer, recon stream), then every master broadcasts its updated rows to
// the other workers (comm stream) and the bias (M floats, from the gathered per-worker sums) is
// updated on every rank alike.  Records kstart / kend / done.
poseidon_status_t sfps_update(poseidon_ctx_t c, Layer& L, float* W, float* bias, float lr, cudaEvent_t src_g,
                              EvSet& dst, IterRecord& r) {
  const int P = c->world;
  CU_TRY(evwait(c, c->recon_stream, src_g));
  FZ(c->recon_stream);
  CU_TRY(evrec(c, dst.kstart, c->recon_stream));
  dst.ks_eff = dst.kstart;
  dst.ke_eff = dst.kend;
  const float alpha = -lr / (float)P;
  const bool mom = (L.vel != nullptr);
  const int64_t mb = L.re - L.rb;
  cudaError_t err = cudaSuccess;
  if (mb > 0) {
    float* target = (mom ? L.vel : W) + (size_t)L.rb * L.N;
    const float a1 = mom ? (lr / (float)P) : alpha, b1 = mom ? L.mu : 1.0f;
    const float* Ub = L.Ug + (size_t)L.rb * L.ldk;
    if (L.recon == POSEIDON_RECON_TF32 && recon_tcgen05_supported(Ub, L.Vg, L.ldk, mb, L.N, target))
      err = launch_recon_tcgen05(Ub, L.Vg, P, L.K, L.ldk, mb, L.N, target, a1, b1, c->recon_stream, nullptr, L.M);
    else
      err = launch_recon_simt(Ub, L.Vg, P, L.K, L.ldk, mb, L.N, target, a1, b1, c->recon_stream, L.M);
    if (err != cudaSuccess) return cuda_fail(err, "SF-PS row-block reconstruct+sgd launch");
    if (mom) {
      err = launch_momentum_apply(W + (size_t)L.rb * L.N, L.vel + (size_t)L.rb * L.N, mb * L.N, lr * L.wd,
                                  c->recon_stream);
      if (err != cudaSuccess) return cuda_fail(err, "momentum apply launch");
    }
    if ((err = debug_sync(c->recon_stream, "SF-PS K1")) != cudaSuccess) return cuda_fail(err, "SF-PS K1");
  }
  CU_TRY(evrec(c, dst.kend, c->recon_stream));
  CU_TRY(evwait(c, c->comm_stream, dst.kend));
  FZ(c->comm_stream);
  int64_t S0b, S0e, S0pad;
  poseidon_shard_range(L.M, P, 0, &S0b, &S0e, &S0pad);
  if (P > 1 && S0pad == L.M) {
    // every master owns the same number of rows and W is exactly P row blocks: the row broadcast is an
    // in-place all-gather (bandwidth-optimal, one collective)
    const size_t cnt = (size_t)(L.re - L.rb) * (size_t)L.N;
    NC_TRY(ncclAllGather(W + (size_t)L.rb * L.N, W, cnt, ncclFloat32, c->comm, c->comm_stream));
    r.sent += (uint64_t)cnt * 4u;
    r.recv += (uint64_t)cnt * 4u * (uint64_t)(P - 1);
  } else if (P > 1) {
    NC_TRY(ncclGroupStart());
    for (int q = 0; q < P; ++q) {
      int64_t qb, qe, pad;
      poseidon_shard_range(L.M, P, q, &qb, &qe, &pad);
      if (qe <= qb) continue;
      float* rows = W + (size_t)qb * L.N;
      const size_t cnt = (size_t)(qe - qb) * (size_t)L.N;
      NC_TRY(ncclBroadcast(rows, rows, cnt, ncclFloat32, q, c->comm, c->comm_stream));
      if (q == c->rank) r.sent += (uint64_t)cnt * 4u;
      else r.recv += (uint64_t)cnt * 4u;
    }
    NC_TRY(ncclGroupEnd());
  }
  if (bias) {
    err = mom ? launch_bias_momentum(L.Bs, L.M, P, bias, L.vel_b, L.M, lr, L.mu, L.wd, c->comm_stream)
              : launch_bias_update(L.Bs, L.M, P, bias, L.M, alpha, c->comm_stream);
    if (err != cudaSuccess) return cuda_fail(err, "bias update launch");
  }
  CU_TRY(evrec(c, dst.done, c->comm_stream));
  return POSEIDON_OK;
}

// BSP sync of a factor layer: SFB or SF-PS.
poseidon_status_t launch_factor_sync(poseidon_ctx_t c, int32_t id, Layer& L, float* W, float* bias, float lr,
                                     cudaEvent_t wait_ev) {
  if (L.scheme == POSEIDON_SCHEME_SFB) return launch_sfb_comm(c, id, L, W, bias, lr, wait_ev);
  EvSet& e = L.ev[c->iter % RING];
  IterRecord& r = open_record(c);
  poseidon_status_t st = sfps_comm(c, L, e, wait_ev, r);
  if (st) return st;
  st = sfps_update(c, L, W, bias, lr, e.g_eff, e, r);
  if (st) return st;
  r.layers.push_back(id);
  return POSEIDON_OK;
}

bool ps_fused(poseidon_ctx_t c, const Layer& L) { return c->world > 1 && c->ps_nvls && L.in_arena; }

// PS reduce-scatter leg (Alg. 3 line 1-2 / Alg. 1 "Collect gradients") of gradient buffer `grad` on
// the comm stream after `wait_ev`.  On the fused NVLS path the reduction happens inside the update
// kernel, so nothing is launched here.  Records e.start (and e.gathered).
poseidon_status_t ps_comm(poseidon_ctx_t c, Layer& L, float* grad, EvSet& e, cudaEvent_t wait_ev, IterRecord& r) {
  const int P = c->world;
  CU_TRY(evwait(c, c->comm_stream, wait_ev));
  FZ(c->comm_stream);
  CU_TRY(evrec(c, e.start, c->comm_stream));
  e.g_eff = e.ks_eff = e.start;
  if (ps_fused(c, L) || P <= 1) return POSEIDON_OK;
  NC_TRY(ncclReduceScatter(grad, grad + (size_t)c->rank * L.S, (size_t)L.S, ncclFloat32, ncclSum, c->comm,
                           c->comm_stream));
  r.sent += (uint64_t)L.S * 4u * (uint64_t)(P - 1);
  r.recv += (uint64_t)L.S * 4u * (uint64_t)(P - 1);
  CU_TRY(evrec(c, e.gathered, c->comm_stream));
  e.g_eff = e.ks_eff = e.gathered;
  return POSEIDON_OK;
}

// PS update + all-gather legs (K2 "Updates the part of model parameters", Alg. 1) of the
// gradient buffer `grad`, then the gradient clear (the fused NVLS kernel does all of it).
poseidon_status_t ps_update(poseidon_ctx_t c, Layer& L, float* grad, float* W, float lr, EvSet& dst, IterRecord& r) {
  const int P = c->world;
  if (ps_fused(c, L) && L.os_off >= 0 && c->win_s && !L.vel && (L.ps_flags & POSEIDON_PS_ZERO_GRAD)) {
    // K2o: one-shot sync of a small layer (peer stores, one barrier, replicated update, clear)
    dst.ke_eff = dst.done;
    cudaError_t err = launch_ps_oneshot(c->nvls, c->win_s, (size_t)L.os_off, L.grad, L.Wps, L.n, -lr / (float)P,
                                        c->comm_stream);
    if (err != cudaSuccess) return cuda_fail(err, "one-shot PS launch");
    CU_TRY(evrec(c, dst.done, c->comm_stream));
    r.sent += (uint64_t)L.n * 4u * (uint64_t)(P - 1);
    r.recv += (uint64_t)L.n * 4u * (uint64_t)(P - 1);
    return POSEIDON_OK;
  }
  if (ps_fused(c, L)) {
    // fused one-kernel PS over NVLink SHARP (reduce-scatter + K2 + all-gather + zero-grad)
    dst.ke_eff = dst.done;
    cudaError_t err = launch_ps_nvls(c->nvls, c->win_g, c->win_w, L.arena_off, L.arena_off, L.begin,
                                     L.end, L.padded, -lr / (float)P, (L.ps_flags & POSEIDON_PS_ZERO_GRAD) != 0,
                                     kNvlsBlocks, L.S, L.vel, 1.0f / (float)P, lr, L.mu, L.wd, c->comm_stream);
    if (err != cudaSuccess) return cuda_fail(err, "fused NVLS PS launch");
    CU_TRY(evrec(c, dst.done, c->comm_stream));
    // bytes through NVLink per rank: the switch reads this rank's gradient for the other P-1
    // shards and writes the other ranks' updated shards here; this rank reads its reduced shard
    // and writes its updated shard once into the switch
    r.sent += (uint64_t)L.S * 4u * (uint64_t)P;
    r.recv += (uint64_t)L.S * 4u * (uint64_t)P;
    return POSEIDON_OK;
  }
  const float alpha = -lr / (float)P;
  const bool zero = (L.ps_flags & POSEIDON_PS_ZERO_GRAD) != 0;
  // K2 with the gradient clear fused in (one launch) unless momentum or an unaligned buffer needs the
  // separate paths
  const bool fused_zero = zero && !L.vel && ps_shard_update_zero_supported(grad, W, L.begin);
  cudaError_t err;
  if (fused_zero)
    err = launch_ps_shard_update_zero(grad, W, L.begin, L.end, L.padded, alpha, c->comm_stream);
  else if (L.vel)
    err = launch_ps_momentum(grad + L.begin, W + L.begin, L.vel, L.end - L.begin, 1.0f / (float)P, lr, L.mu, L.wd,
                             c->comm_stream);
  else
    err = launch_ps_shard_update(grad + L.begin, W + L.begin, L.end - L.begin, alpha, nullptr, c->comm_stream);
  if (err != cudaSuccess) return cuda_fail(err, "ps shard update launch");
  if ((err = debug_sync(c->comm_stream, "K2 ps shard update")) != cudaSuccess) return cuda_fail(err, "K2");
  if (P > 1) {
    CU_TRY(evrec(c, dst.kend, c->comm_stream));
    dst.ke_eff = dst.kend;
    NC_TRY(ncclAllGather(W + (size_t)c->rank * L.S, W, (size_t)L.S, ncclFloat32, c->comm, c->comm_stream));
    r.sent += (uint64_t)L.S * 4u * (uint64_t)(P - 1);
    r.recv += (uint64_t)L.S * 4u * (uint64_t)(P - 1);
  } else {
    dst.ke_eff = dst.done;
  }
  if (zero && !fused_zero) {
    if (P == 1) {  // kernel_ms must not include the memset
      CU_TRY(evrec(c, dst.kend, c->comm_stream));
      dst.ke_eff = dst.kend;
    }
    CU_TRY(cudaMemsetAsync(grad, 0, (size_t)L.padded * 4u, c->comm_stream));
  }
  CU_TRY(evrec(c, dst.done, c->comm_stream));
  return POSEIDON_OK;
}

// BSP PS sync (Alg. 3 lines 1-3 / Alg. 1 master): RS -> K2 -> AG (or the fused NVLS kernel), all on
// the comm stream.
poseidon_status_t launch_ps_comm(poseidon_ctx_t c, int32_t id, Layer& L, float* grad, float* W, float lr,
                                 cudaEvent_t wait_ev) {
  EvSet& e = L.ev[c->iter % RING];
  IterRecord& r = open_record(c);
  poseidon_status_t st = ps_comm(c, L, grad, e, wait_ev, r);
  if (st) return st;
  st = ps_update(c, L, grad, W, lr, e, r);
  if (st) return st;
  r.layers.push_back(id);
  return POSEIDON_OK;
}

// SSP, PS layers: the communication of sync t is ONE all-reduce of the gradient (the reduce-scatter
// and all-gather legs of a PS sync, applied to the gradient instead of the updated shard), so the
// deferred update is local and the next forward depends on the previous iteration's collective only.
poseidon_status_t ps_comm_allreduce(poseidon_ctx_t c, Layer& L, float* grad, EvSet& e, cudaEvent_t wait_ev,
                                    IterRecord& r) {
  const int P = c->world;
  CU_TRY(evwait(c, c->comm_stream, wait_ev));
  FZ(c->comm_stream);
  CU_TRY(evrec(c, e.start, c->comm_stream));
  e.g_eff = e.start;
  if (P <= 1) return POSEIDON_OK;
  NC_TRY(ncclAllReduce(grad, grad, (size_t)L.padded, ncclFloat32, ncclSum, c->comm, c->comm_stream));
  const uint64_t wire = 2u * (uint64_t)L.S * 4u * (uint64_t)(P - 1);
  r.sent += wire;
  r.recv += wire;
  CU_TRY(evrec(c, e.gathered, c->comm_stream));
  e.g_eff = e.gathered;
  return POSEIDON_OK;
}

// SSP, PS layers: W[0, n) = fmaf(-lr/P, gsum, W) on every rank (the same fp32 operation K2 applies to
// the shard, so every rank stays bit-identical), then the gradient buffer is cleared; on the recon
// stream after the all-reduce `src_g` and `extra` (this layer's current backward is done with W).
poseidon_status_t ps_update_local(poseidon_ctx_t c, Layer& L, float* grad, float* W, float lr, cudaEvent_t src_g,
                                  cudaEvent_t extra, EvSet& dst) {
  const int P = c->world;
  CU_TRY(evwait(c, c->recon_stream, src_g));
  if (extra) CU_TRY(evwait(c, c->recon_stream, extra));
  FZ(c->recon_stream);
  CU_TRY(evrec(c, dst.kstart, c->recon_stream));
  dst.ks_eff = dst.kstart;
  dst.ke_eff = dst.done;
  const bool zero = (L.ps_flags & POSEIDON_PS_ZERO_GRAD) != 0;
  cudaError_t err;
  if (!L.vel && zero && ps_shard_update_zero_supported(grad, W, 0)) {
    err = launch_ps_shard_update_zero(grad, W, 0, L.n, L.padded, -lr / (float)P, c->recon_stream);
  } else {
    err = L.vel ? launch_ps_momentum(grad, W, L.vel, L.n, 1.0f / (float)P, lr, L.mu, L.wd, c->recon_stream)
                : launch_ps_shard_update(grad, W, L.n, -lr / (float)P, nullptr, c->recon_stream);
    if (err == cudaSuccess && zero) err = cudaMemsetAsync(grad, 0, (size_t)L.padded * 4u, c->recon_stream);
  }
  if (err != cudaSuccess) return cuda_fail(err, "SSP PS local update launch");
  if ((err = debug_sync(c->recon_stream, "SSP PS update")) != cudaSuccess) return cuda_fail(err, "SSP PS update");
  CU_TRY(evrec(c, dst.done, c->recon_stream));
  return POSEIDON_OK;
}

// SSP with staleness s (reading Z19; s = 1 by FLAG_SSP1, 2..5 by poseidon_set_staleness): this hook issues
// sync t's communication into gather / gradient set t mod (s+1) and applies the update of sync t-s —
// after this layer's backward t has finished reading W (e.ready) — so the forward of t+1 reads W with every
// update of iterations <= t-s (at the staleness bound).  The update is local (SFB: K1 on the
// gathered factors; PS: the all-reduced gradient), so a rank's next forward waits for the other ranks'
// hook t-s, not hook t: s iterations of slack.
poseidon_status_t ssp_hook(poseidon_ctx_t c, int32_t id, Layer& L, float* W, float* bias, float* grad, float lr) {
  EvSet& e = L.ev[c->iter % RING];
  IterRecord& r = open_record(c);
  const int set = next_set(c, L);
  poseidon_status_t st = (L.scheme == POSEIDON_SCHEME_SFB) ? sfb_comm(c, L, set, e, e.ready, r)
                                                           : ps_comm_allreduce(c, L, grad, e, e.ready, r);
  if (st) return st;
  L.pend.push_back(Layer::Pend{c->iter, set, lr, W, bias, grad});
  if ((int)L.pend.size() > c->stale) {
    // apply the update of iteration t - s (its collective is ordered before this one on the comm stream)
    const Layer::Pend q = L.pend.front();
    L.pend.pop_front();
    const EvSet& src = L.ev[q.iter % RING];
    st = (L.scheme == POSEIDON_SCHEME_SFB) ? sfb_update(c, L, q.set, q.W, q.bias, q.lr, src.g_eff, e.ready, e)
                                           : ps_update_local(c, L, q.grad, L.Wps, q.lr, src.g_eff, e.ready, e);
    if (st) return st;
  } else {
    // the first s syncs: nothing to apply yet; done only orders after this backward
    CU_TRY(evwait(c, c->recon_stream, e.ready));
    CU_TRY(evrec(c, e.done, c->recon_stream));
    e.ks_eff = e.ke_eff = e.done;
  }
  L.nsync += 1;
  r.layers.push_back(id);
  return POSEIDON_OK;
}

poseidon_status_t sfb_after_pack(poseidon_ctx_t c, int32_t id, Layer& L, float* W, float* bias, float lr,
                                 cudaStream_t producer) {
  EvSet& e = L.ev[c->iter % RING];
  CU_TRY(evrec(c, e.ready, producer));
  L.last_iter = c->iter;
  if (c->ssp) return ssp_hook(c, id, L, W, bias, nullptr, lr);
  if (c->flags & POSEIDON_FLAG_DWBP_OFF) {
    L.pending = true;
    L.pending_lr = lr;
    L.pending_W = W;
    L.pending_bias = bias;
    c->pending_order.push_back(id);
    open_record(c);
    return POSEIDON_OK;
  }
  poseidon_status_t st = launch_factor_sync(c, id, L, W, bias, lr, e.ready);
  L.v_posted = false;
  return st;
}

poseidon_status_t pack_sfb(poseidon_ctx_t c, Layer& L, const float* U, int64_t ldU, const float* V, int64_t ldV,
                           cudaStream_t producer) {
  const bool round = (L.recon == POSEIDON_RECON_TF32);
  const GatherSet g = gather_set(L, next_set(c, L));
  float* u_slot = g.U + (size_t)c->rank * slot_u(L);
  float* v_slot = g.V + (size_t)c->rank * slot_v(L);
  float* b_slot = g.B + (size_t)c->rank * L.M;
  // U (+ bias column sums) and, unless the early input broadcast already packed it, V: one launch
  EvSet& e = L.ev[c->iter % RING];
  CU_TRY(evrec(c, e.pstart, producer));
  e.packed = true;
  e.pack_async = false;
  if (L.mn) {   // MN-major gather: the slot is the layer's own [K x M] / [K x N] rows, copied by the copy engine
    CU_TRY(cudaMemcpy2DAsync(u_slot, (size_t)L.M * 4, U, (size_t)ldU * 4, (size_t)L.M * 4, (size_t)L.K,
                             cudaMemcpyDeviceToDevice, producer));
    if (!L.v_posted)
      CU_TRY(cudaMemcpy2DAsync(v_slot, (size_t)L.N * 4, V, (size_t)ldV * 4, (size_t)L.N * 4, (size_t)L.K,
                               cudaMemcpyDeviceToDevice, producer));
    return POSEIDON_OK;
  }
  cudaError_t err = launch_pack_uv(U, ldU, u_slot, L.M, b_slot, L.v_posted ? nullptr : V, ldV, v_slot, L.N,
                                   L.ldk, L.K, round, producer);
  if (err != cudaSuccess) return cuda_fail(err, "pack U/V launch");
  if ((err = debug_sync(producer, "K3 pack")) != cudaSuccess) return cuda_fail(err, "K3");
  return POSEIDON_OK;
}

void free_layer(poseidon_ctx_t c, Layer& L) {
  if (L.symm) {
    if (L.win) ncclCommWindowDeregister(L.win_comm, L.win);  // collective: every rank frees the layer
    ncclMemFree(L.symm);
    L.symm = nullptr;
    L.win = nullptr;
  } else {
    for (float* q : {L.Ug, L.Vg, L.Bs})
      if (q) cudaFree(q);
    for (auto* vec : {&L.xU, &L.xV, &L.xB})
      for (float* q : *vec)
        if (q) cudaFree(q);
  }
  L.xU.clear();
  L.xV.clear();
  L.xB.clear();
  if (L.stU) cudaFree(L.stU);
  if (L.stV) cudaFree(L.stV);
  if (L.vel) cudaFree(L.vel);
  if (L.vel_b) cudaFree(L.vel_b);
  L.Ug = L.Vg = L.Bs = L.stU = L.stV = L.vel = L.vel_b = nullptr;
  if (L.events_created) {
    for (int i = 0; i < RING; ++i) {
      EvSet& e = L.ev[i];
      cudaEvent_t all[] = {e.ready, e.start, e.gathered, e.kstart, e.kend, e.done, e.vready, e.vgath, e.pstart,
                           e.pend};
      for (cudaEvent_t ev : all) {
        if (!ev) continue;
        auto it = c->evmeta.find(ev);
        if (it != c->evmeta.end()) {
          cudaEventDestroy(it->second.first);
          c->evmeta.erase(it);
        }
        cudaEventDestroy(ev);
      }
      e = EvSet{};
    }
    L.events_created = false;
  }
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

}  // namespace

extern "C" {

int32_t poseidon_version(void) { return 10000; }
const char* poseidon_last_error(void) { return poseidon::t_err.c_str(); }
uint64_t poseidon_launch_count(void) { return g_launches.load(); }

poseidon_status_t poseidon_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(POSEIDON_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  NC_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
  memcpy(out, id.internal, 128);
  return POSEIDON_OK;
}

poseidon_status_t poseidon_init(int32_t world, const poseidon_topology_t* topo, poseidon_ctx_t* out) {
  if (!topo || !out) return fail(POSEIDON_ERR_INVALID_ARG, "topo/out is NULL");
  if (world < 1 || topo->world != world || topo->rank < 0 || topo->rank >= world)
    return fail(POSEIDON_ERR_INVALID_ARG, "inconsistent world/rank");
  int ndev = 0;
  CU_TRY(cudaGetDeviceCount(&ndev));
  if (topo->device < 0 || topo->device >= ndev) return fail(POSEIDON_ERR_INVALID_ARG, "device out of range");
  CU_TRY(cudaSetDevice(topo->device));
  cudaDeviceProp prop;
  CU_TRY(cudaGetDeviceProperties(&prop, topo->device));
  if (prop.major != 10)
    return fail(POSEIDON_ERR_UNSUPPORTED, "libposeidon is built for sm_100a (B200); device is sm_" +
                                              std::to_string(prop.major) + std::to_string(prop.minor));
  if ((topo->flags & POSEIDON_FLAG_SSP1) && (topo->flags & POSEIDON_FLAG_DWBP_OFF))
    return fail(POSEIDON_ERR_INVALID_ARG, "FLAG_SSP1 needs DWBP (the stale update is applied at the next hook)");
  if ((topo->flags & POSEIDON_FLAG_EARLY_V) && (topo->flags & (POSEIDON_FLAG_SSP1 | POSEIDON_FLAG_DWBP_OFF)))
    return fail(POSEIDON_ERR_INVALID_ARG, "FLAG_EARLY_V is a BSP + DWBP schedule (not with SSP1 / DWBP_OFF)");
  auto* c = new poseidon_ctx();
  c->rank = topo->rank;
  c->world = world;
  c->device = topo->device;
  c->flags = topo->flags;
  c->want_nvls = (topo->flags & POSEIDON_FLAG_NVLS_PS) != 0 && world > 1;
  c->want_nvls_sfb = (topo->flags & POSEIDON_FLAG_NVLS_SFB) != 0 && world > 1;
  c->ssp = (topo->flags & POSEIDON_FLAG_SSP1) != 0;
  c->stale = c->ssp ? 1 : 0;
  c->layers.resize(64);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  const int prio = (c->flags & POSEIDON_FLAG_NO_PRIORITY) ? lo : hi;
  cudaError_t e1 = cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio);
  cudaError_t e2 = cudaStreamCreateWithPriority(&c->recon_stream, cudaStreamNonBlocking, prio);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete c;
    return cuda_fail(e1 != cudaSuccess ? e1 : e2, "stream create");
  }
  for (auto& r : c->rec) {
    if (cudaEventCreate(&r.bwd_end) != cudaSuccess || make_twin(c, r.bwd_end) != cudaSuccess) {
      delete c;
      return fail(POSEIDON_ERR_CUDA, "event create");
    }
  }
  for (auto& j : c->join_ev) {
    if (cudaEventCreateWithFlags(&j, cudaEventDisableTiming) != cudaSuccess) {
      delete c;
      return fail(POSEIDON_ERR_CUDA, "event create");
    }
  }
  if (world > 1) {
    ncclUniqueId id;
    memcpy(id.internal, topo->nccl_id, 128);
    // POSEIDON_NCCL_CTA_POLICY (experiment knob): NCCL_CTA_POLICY_EFFICIENCY (1) / _ZERO (2; copy-engine
    // collectives on symmetric windows where NCCL supports them)
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (const char* pol = getenv("POSEIDON_NCCL_CTA_POLICY")) cfg.CTAPolicy = atoi(pol);
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, world, id, topo->rank, &cfg);
    if (r != ncclSuccess) {
      delete c;
      return fail(POSEIDON_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    poseidon_status_t pst = check_peers(c);
    if (pst != POSEIDON_OK) {
      ncclCommDestroy(c->comm);
      delete c;
      return pst;
    }
  }
  *out = c;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_finalize(poseidon_ctx_t c) {
  if (!c) return POSEIDON_OK;
  cudaSetDevice(c->device);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->recon_stream) cudaStreamSynchronize(c->recon_stream);
  for (auto& L : c->layers) free_layer(c, L);
  for (auto& B : c->buckets) {
    B.grad = B.Wps = nullptr;   // views into the arena
    free_layer(c, B);
  }
  if (c->nvls) nvls_destroy(c->comm, c->nvls);
  if (c->win_g) ncclCommWindowDeregister(c->comm, c->win_g);
  for (ncclWindow_t wg : c->win_gx)
    if (wg) ncclCommWindowDeregister(c->comm, wg);
  if (c->win_s) ncclCommWindowDeregister(c->comm, c->win_s);
  if (c->os_buf) ncclMemFree(c->os_buf);
  if (c->win_w) ncclCommWindowDeregister(c->comm, c->win_w);
  std::vector<float*> arenas = {c->arena_g, c->arena_w};
  arenas.insert(arenas.end(), c->arena_gx.begin(), c->arena_gx.end());
  for (float* q : arenas)
    if (q) {
      if (c->arena_nccl_mem) ncclMemFree(q);
      else cudaFree(q);
    }
  for (auto& r : c->rec)
    if (r.bwd_end) cudaEventDestroy(r.bwd_end);
  for (auto& kv : c->evmeta) cudaEventDestroy(kv.second.first);
  for (auto& j : c->join_ev)
    if (j) cudaEventDestroy(j);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->recon_stream) cudaStreamDestroy(c->recon_stream);
  delete c;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_register_layer(poseidon_ctx_t c, int32_t id, int32_t kind, int64_t M, int64_t N,
                                          int64_t K, int32_t has_bias, int32_t scheme_override,
                                          int32_t* chosen_scheme) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (id < 0 || id >= MAX_LAYERS) return fail(POSEIDON_ERR_INVALID_ARG, "layer_id out of range [0,4096)");
  if (kind != POSEIDON_LAYER_CONV && kind != POSEIDON_LAYER_FC) return fail(POSEIDON_ERR_INVALID_ARG, "bad kind");
  if (M <= 0 || N <= 0 || K <= 0) return fail(POSEIDON_ERR_SHAPE, "M, N, K must be positive");
  if (scheme_override < -1 || scheme_override > 2) return fail(POSEIDON_ERR_INVALID_ARG, "bad scheme_override");
  int32_t rule = poseidon_choose_scheme(kind, M, N, K, c->world, nullptr);
  if (rule < 0) return (poseidon_status_t)rule;
  int32_t scheme = scheme_override >= 0 ? scheme_override : rule;
  // FLAG_SFPS: an FC layer the rule sends to the server runs Alg. 3's else-branch literally
  if (scheme_override < 0 && scheme == POSEIDON_SCHEME_PS && kind == POSEIDON_LAYER_FC &&
      (c->flags & POSEIDON_FLAG_SFPS))
    scheme = POSEIDON_SCHEME_SFPS;
  if (scheme != POSEIDON_SCHEME_PS && kind != POSEIDON_LAYER_FC)
    return fail(POSEIDON_ERR_INVALID_ARG, "SFB / SF-PS need an FC layer (Alg. 3)");
  if (scheme == POSEIDON_SCHEME_SFPS && c->ssp)
    return fail(POSEIDON_ERR_UNSUPPORTED, "SF-PS layers are not supported with FLAG_SSP1");
  cudaSetDevice(c->device);
  if (id >= (int32_t)c->layers.size()) c->layers.resize((size_t)id + 1);
  Layer& L = c->layers[id];
  if (L.registered && L.last_iter >= 0) {
    // re-registration: wait for the layer to be idle
    cudaEventSynchronize(L.ev[L.last_iter % RING].done);
  }
  free_layer(c, L);
  L = Layer{};
  L.kind = kind;
  L.M = M;
  L.N = N;
  L.K = K;
  L.has_bias = has_bias != 0;
  L.scheme = scheme;
  if (scheme == POSEIDON_SCHEME_SFPS) {
    int64_t pad;
    poseidon_shard_range(M, c->world, c->rank, &L.rb, &L.re, &pad);
  }
  if (scheme != POSEIDON_SCHEME_PS) {
    L.ldk = round_up(K, 4);
    L.mn = scheme == POSEIDON_SCHEME_SFB && c->world > 1 && !c->ssp && !(c->flags & POSEIDON_FLAG_DWBP_OFF) &&
           (c->flags & POSEIDON_FLAG_INPLACE_FACTORS) && (c->flags & POSEIDON_FLAG_INPLACE_MN) && M % 4 == 0 &&
           N % 4 == 0 && M < (1 << 30) && N < (1 << 30);
    const size_t P = (size_t)c->world;
    const size_t ub = P * (size_t)(M * L.ldk) * 4, vb = P * (size_t)(N * L.ldk) * 4, bb = P * (size_t)M * 4;
    const int nsets = c->ssp ? c->stale + 1 : 1;
    bool placed = false;
    if (c->world > 1 && (c->flags & (POSEIDON_FLAG_SYMM_SFB | POSEIDON_FLAG_NVLS_SFB))) {
      // one symmetric window for the layer's gather buffers: NCCL then runs the factor all-gather
      // with its symmetric-memory kernels (collective call: all ranks register alike)
      const size_t ua = round_up((int64_t)ub, 4096), va = round_up((int64_t)vb, 4096);
      const size_t one = ua + va + round_up((int64_t)bb, 4096);
      const size_t total = one * (size_t)nsets;
      void* base = nullptr;
      if (ncclMemAlloc(&base, total) == ncclSuccess) {
        ncclWindow_t w = nullptr;
        if (ncclCommWindowRegister(c->comm, base, total, &w, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess) {
          L.symm = base;
          L.win = w;
          L.win_comm = c->comm;
          char* b0 = static_cast<char*>(base);
          L.Ug = reinterpret_cast<float*>(b0);
          L.Vg = reinterpret_cast<float*>(b0 + ua);
          L.Bs = reinterpret_cast<float*>(b0 + ua + va);
          for (int k = 1; k < nsets; ++k) {
            L.xU.push_back(reinterpret_cast<float*>(b0 + k * one));
            L.xV.push_back(reinterpret_cast<float*>(b0 + k * one + ua));
            L.xB.push_back(reinterpret_cast<float*>(b0 + k * one + ua + va));
          }
          placed = true;
          L.bcast = scheme == POSEIDON_SCHEME_SFB && c->want_nvls_sfb && ensure_devcomm(c);
        } else {
          ncclMemFree(base);
        }
      }
    }
    if (!placed) {
      CU_TRY(cudaMalloc(&L.Ug, ub));
      CU_TRY(cudaMalloc(&L.Vg, vb));
      CU_TRY(cudaMalloc(&L.Bs, bb));
      for (int k = 1; k < nsets; ++k) {
        float *u = nullptr, *v = nullptr, *b = nullptr;
        CU_TRY(cudaMalloc(&u, ub));
        CU_TRY(cudaMalloc(&v, vb));
        CU_TRY(cudaMalloc(&b, bb));
        L.xU.push_back(u);
        L.xV.push_back(v);
        L.xB.push_back(b);
      }
    }
    for (int k = 0; k + 1 < nsets; ++k) {
      CU_TRY(cudaMemset(L.xU[(size_t)k], 0, ub));
      CU_TRY(cudaMemset(L.xV[(size_t)k], 0, vb));
      CU_TRY(cudaMemset(L.xB[(size_t)k], 0, bb));
    }
    CU_TRY(cudaMemset(L.Ug, 0, ub));  // k columns in [K, ldk) stay zero forever
    CU_TRY(cudaMemset(L.Vg, 0, vb));
    CU_TRY(cudaMemset(L.Bs, 0, bb));
  }
  st = ensure_events(c, L);
  if (st) return st;
  L.registered = true;
  if (chosen_scheme) *chosen_scheme = scheme;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_sfb_slot(poseidon_ctx_t c, int32_t id, float** U_slot, int64_t* ld_u, float** V_slot,
                                    int64_t* ld_v) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme == POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not an SFB / SF-PS layer");
  if (!L->stU) {
    cudaSetDevice(c->device);
    CU_TRY(cudaMalloc(&L->stU, (size_t)(L->K * L->M) * 4));
    CU_TRY(cudaMalloc(&L->stV, (size_t)(L->K * L->N) * 4));
  }
  if (U_slot) *U_slot = L->stU;
  if (V_slot) *V_slot = L->stV;
  if (ld_u) *ld_u = L->M;
  if (ld_v) *ld_v = L->N;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_bind_ps_buffers(poseidon_ctx_t c, int32_t id, float* grad, float* W, int64_t n,
                                           uint32_t flags) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme != POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not a PS layer");
  if (!grad || !W) return fail(POSEIDON_ERR_INVALID_ARG, "grad/W is NULL");
  if (!aligned16(grad) || !aligned16(W)) return fail(POSEIDON_ERR_ALIGNMENT, "PS buffers must be 16-byte aligned");
  const int64_t expect = L->M * L->N + (L->has_bias ? L->M : 0);
  if (n != expect) return fail(POSEIDON_ERR_SHAPE, "n != M*N (+M if bias)");
  L->grad = grad;
  L->Wps = W;
  L->n = n;
  L->ps_flags = flags;
  int64_t b, e, padded;
  poseidon_shard_range(n, c->world, c->rank, &b, &e, &padded);
  L->S = padded / c->world;
  L->padded = padded;
  L->begin = b;
  L->end = e;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_bind_sfb_params(poseidon_ctx_t c, int32_t id, float* W, float* bias) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme == POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not an SFB / SF-PS layer");
  if (!W) return fail(POSEIDON_ERR_INVALID_ARG, "W is NULL");
  if (bias && !L->has_bias) return fail(POSEIDON_ERR_INVALID_ARG, "layer registered without bias");
  L->W = W;
  L->bias = bias;
  return POSEIDON_OK;
}

static poseidon_status_t set_momentum_one(poseidon_ctx_t c, Layer& L, float mu, float wd);

poseidon_status_t poseidon_set_ps_buckets(poseidon_ctx_t c, int64_t bucket_bytes) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (bucket_bytes < 0) return fail(POSEIDON_ERR_INVALID_ARG, "bucket_bytes must be >= 0");
  if (c->arena_g) return fail(POSEIDON_ERR_STATE, "set buckets before poseidon_ps_arena");
  if (c->ssp && bucket_bytes > 0) return fail(POSEIDON_ERR_INVALID_ARG, "PS buckets are not supported with FLAG_SSP1");
  c->bucket_bytes = bucket_bytes;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_ps_arena(poseidon_ctx_t c, int32_t* nvls_active) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (c->arena_g) return fail(POSEIDON_ERR_STATE, "PS arena already created");
  cudaSetDevice(c->device);
  size_t total = 0;
  // Buckets (poseidon_set_ps_buckets): runs of consecutive PS layers (id order) whose 128-B aligned
  // spans add up to at most bucket_bytes share one contiguous arena span and sync as one flat buffer
  // with its own shard map; a run of one stays a plain layer.
  c->buckets.clear();
  std::vector<std::vector<int32_t>> groups;
  {
    std::vector<int32_t> cur;
    size_t cur_bytes = 0;
    auto close = [&]() {
      if (!cur.empty()) groups.push_back(cur);
      cur.clear();
      cur_bytes = 0;
    };
    for (int32_t id = 0; id < (int32_t)c->layers.size(); ++id) {
      Layer& L = c->layers[(size_t)id];
      if (!L.registered || L.scheme != POSEIDON_SCHEME_PS) continue;
      const size_t seg = (size_t)round_up((L.M * L.N + (L.has_bias ? L.M : 0)) * 4, 128);
      if (c->bucket_bytes <= 0 || seg > (size_t)c->bucket_bytes) {
        close();
        groups.push_back({id});
        continue;
      }
      if (cur_bytes + seg > (size_t)c->bucket_bytes) close();
      cur.push_back(id);
      cur_bytes += seg;
    }
    close();
  }
  for (auto& g : groups) {
    if (g.size() == 1) {
      Layer& L = c->layers[(size_t)g[0]];
      const int64_t n = L.M * L.N + (L.has_bias ? L.M : 0);
      int64_t b, e, padded;
      poseidon_shard_range(n, c->world, c->rank, &b, &e, &padded);
      L.arena_off = total;
      L.bucket = -1;
      total += (size_t)round_up(padded * 4, 4096);
      continue;
    }
    c->buckets.emplace_back();
    Layer& B = c->buckets.back();
    B.registered = true;
    B.kind = POSEIDON_LAYER_CONV;
    B.scheme = POSEIDON_SCHEME_PS;
    B.members = g;
    B.arena_off = total;
    size_t off = 0;
    for (int32_t m : g) {
      Layer& L = c->layers[(size_t)m];
      L.bucket = (int32_t)c->buckets.size() - 1;
      L.arena_off = total + off;
      off += (size_t)round_up((L.M * L.N + (L.has_bias ? L.M : 0)) * 4, 128);
    }
    B.M = 1;
    B.N = (int64_t)(off / 4);  // flat length of the bucket (n of the pseudo-layer)
    int64_t b, e, padded;
    poseidon_shard_range(B.N, c->world, c->rank, &b, &e, &padded);
    total += (size_t)round_up(padded * 4, 4096);
  }
  if (total == 0) total = 4096;
  c->arena_bytes = total;
  bool symmetric = false;
  if (c->want_nvls && c->comm) {
    void *g = nullptr, *w = nullptr;
    std::vector<void*> gx((size_t)(c->ssp ? c->stale : 0), nullptr);
    ncclResult_t r = ncclMemAlloc(&g, total);
    if (r == ncclSuccess) r = ncclMemAlloc(&w, total);
    for (size_t k = 0; k < gx.size() && r == ncclSuccess; ++k) r = ncclMemAlloc(&gx[k], total);
    if (r == ncclSuccess) r = ncclCommWindowRegister(c->comm, g, total, &c->win_g, NCCL_WIN_COLL_SYMMETRIC);
    if (r == ncclSuccess) r = ncclCommWindowRegister(c->comm, w, total, &c->win_w, NCCL_WIN_COLL_SYMMETRIC);
    for (size_t k = 0; k < gx.size() && r == ncclSuccess; ++k) {
      ncclWindow_t wk = nullptr;
      r = ncclCommWindowRegister(c->comm, gx[k], total, &wk, NCCL_WIN_COLL_SYMMETRIC);
      if (r == ncclSuccess) c->win_gx.push_back(wk);
    }
    if (r == ncclSuccess) {
      c->ps_nvls = ensure_devcomm(c);
      if (!c->ps_nvls) c->nvls_error = c->devcomm_error;
      symmetric = true;
      c->arena_nccl_mem = true;
      c->arena_g = static_cast<float*>(g);
      c->arena_w = static_cast<float*>(w);
      for (void* q : gx) c->arena_gx.push_back(static_cast<float*>(q));
    } else {
      c->nvls_error = std::string("symmetric window: ") + ncclGetErrorString(r);
      if (c->win_g) { ncclCommWindowDeregister(c->comm, c->win_g); c->win_g = nullptr; }
      if (c->win_w) { ncclCommWindowDeregister(c->comm, c->win_w); c->win_w = nullptr; }
      for (ncclWindow_t wk : c->win_gx) ncclCommWindowDeregister(c->comm, wk);
      c->win_gx.clear();
      gx.push_back(g);
      gx.push_back(w);
      for (void* q : gx)
        if (q) ncclMemFree(q);
    }
  }
  if (!symmetric) {
    CU_TRY(cudaMalloc(&c->arena_g, total));
    CU_TRY(cudaMalloc(&c->arena_w, total));
    for (int k = 0; k < (c->ssp ? c->stale : 0); ++k) {
      float* q = nullptr;
      CU_TRY(cudaMalloc(&q, total));
      c->arena_gx.push_back(q);
    }
  }
  CU_TRY(cudaMemset(c->arena_g, 0, total));
  CU_TRY(cudaMemset(c->arena_w, 0, total));
  for (float* q : c->arena_gx) CU_TRY(cudaMemset(q, 0, total));
  CU_TRY(cudaDeviceSynchronize());
  auto at = [](float* base, size_t off) {
    return base ? reinterpret_cast<float*>(reinterpret_cast<char*>(base) + off) : nullptr;
  };
  for (int32_t id = 0; id < (int32_t)c->layers.size(); ++id) {
    Layer& L = c->layers[id];
    if (!L.registered || L.scheme != POSEIDON_SCHEME_PS) continue;
    const int64_t n = L.M * L.N + (L.has_bias ? L.M : 0);
    float* g = at(c->arena_g, L.arena_off);
    float* w = at(c->arena_w, L.arena_off);
    if (L.bucket >= 0) {
      // a member: its own views only (the bucket pseudo-layer holds the shard map)
      L.grad = g;
      L.Wps = w;
      L.n = n;
      L.padded = round_up(n * 4, 128) / 4;
      L.ps_flags = POSEIDON_PS_ZERO_GRAD;
    } else {
      st = poseidon_bind_ps_buffers(c, id, g, w, n, POSEIDON_PS_ZERO_GRAD);
      if (st) return st;
    }
    L.in_arena = true;
    L.gsets.assign(1, g);
    for (float* q : c->arena_gx) L.gsets.push_back(at(q, L.arena_off));
  }
  for (auto& B : c->buckets) {
    B.grad = at(c->arena_g, B.arena_off);
    B.Wps = at(c->arena_w, B.arena_off);
    B.n = B.N;
    int64_t b, e, padded;
    poseidon_shard_range(B.n, c->world, c->rank, &b, &e, &padded);
    B.begin = b;
    B.end = e;
    B.padded = padded;
    B.S = padded / c->world;
    B.ps_flags = POSEIDON_PS_ZERO_GRAD;
    B.in_arena = true;
    st = ensure_events(c, B);
    if (st) return st;
    // momentum already set on the members carries over to the bucket (all members share mu, wd)
    const Layer& M0 = c->layers[(size_t)B.members[0]];
    if (M0.vel) {
      st = set_momentum_one(c, B, M0.mu, M0.wd);
      if (st) return st;
    }
  }
  // K2o: layers whose fused sync is latency-bound (n <= kOneShotMax floats, no bucket, no SSP) get a slot in a
  // symmetric scratch window and sync with one barrier instead of two -- when at least two barrier-synced
  // layers exist (the slot reuse argument of k_ps_nvls.cu) and POSEIDON_ONESHOT is not 0
  if (c->ps_nvls && !c->ssp && knobs_oneshot()) {
    int barrier_layers = (int)c->buckets.size();
    for (const Layer& L : c->layers)
      if (L.registered && L.scheme == POSEIDON_SCHEME_PS && L.in_arena && L.bucket < 0) ++barrier_layers;
    size_t total = 0;
    if (barrier_layers >= 2)
      for (Layer& L : c->layers)
        if (L.registered && L.scheme == POSEIDON_SCHEME_PS && L.in_arena && L.bucket < 0 && L.n <= kOneShotMax) {
          L.os_off = (int64_t)total;
          total += (size_t)round_up((int64_t)c->world * round_up(L.n, 4) * 4, 4096);
        }
    if (total > 0) {
      void* buf = nullptr;
      ncclWindow_t w = nullptr;
      if (ncclMemAlloc(&buf, total) == ncclSuccess &&
          ncclCommWindowRegister(c->comm, buf, total, &w, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess) {
        c->os_buf = buf;
        c->win_s = w;
      } else {
        if (buf) ncclMemFree(buf);
        for (Layer& L : c->layers) L.os_off = -1;
      }
    }
  }
  if (nvls_active) *nvls_active = c->ps_nvls ? 1 : 0;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_ps_layer_buffers(poseidon_ctx_t c, int32_t id, float** grad, float** W, int64_t* padded) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (!L->in_arena) return fail(POSEIDON_ERR_STATE, "layer has no arena buffers (call poseidon_ps_arena)");
  // the gradient buffer the layer's NEXT sync reduces (SSP alternates two)
  if (grad) *grad = (c->ssp && L->gsets.size() > 1) ? L->gsets[(size_t)next_set(c, *L)] : L->grad;
  if (W) *W = L->Wps;
  if (padded) *padded = L->padded;
  return POSEIDON_OK;
}

int32_t poseidon_sfb_path(poseidon_ctx_t c, int32_t id) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme == POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not an SFB / SF-PS layer");
  if (L->scheme == POSEIDON_SCHEME_SFPS) return 3;
  return L->bcast ? 2 : (L->symm ? 1 : 0);
}

const char* poseidon_nvls_status(poseidon_ctx_t c) {
  if (!c) return "no context";
  if (c->ps_nvls) return "active";
  if (!c->want_nvls) return "not requested";
  return c->nvls_error.empty() ? "arena not created" : c->nvls_error.c_str();
}

static poseidon_status_t set_momentum_one(poseidon_ctx_t c, Layer& L, float mu, float wd) {
  L.mu = mu;
  L.wd = wd;
  if (mu == 0.f && wd == 0.f) {
    if (L.vel) cudaFree(L.vel);
    if (L.vel_b) cudaFree(L.vel_b);
    L.vel = L.vel_b = nullptr;
    return POSEIDON_OK;
  }
  if (L.vel) return POSEIDON_OK;  // keep the existing velocity
  cudaSetDevice(c->device);
  size_t count;
  if (L.scheme != POSEIDON_SCHEME_PS) {   // SFB: replicated; SF-PS: only the master's rows are used
    count = (size_t)(L.M * L.N);
    if (L.has_bias) {
      CU_TRY(cudaMalloc(&L.vel_b, (size_t)L.M * 4));
      CU_TRY(cudaMemset(L.vel_b, 0, (size_t)L.M * 4));
    }
  } else {
    int64_t b, e, padded;
    const int64_t n = L.M * L.N + (L.has_bias ? L.M : 0);
    poseidon_shard_range(n, c->world, c->rank, &b, &e, &padded);
    // BSP: this rank's shard only; SSP: the whole layer (every rank applies the all-reduced gradient)
    count = c->ssp ? (size_t)n : (size_t)(padded / c->world);
  }
  CU_TRY(cudaMalloc(&L.vel, count * 4));
  CU_TRY(cudaMemset(L.vel, 0, count * 4));
  return POSEIDON_OK;
}

poseidon_status_t poseidon_set_staleness(poseidon_ctx_t c, int32_t s) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (!c->ssp) return fail(POSEIDON_ERR_STATE, "staleness needs a context created with POSEIDON_FLAG_SSP1");
  if (s < 1 || s > RING - 3) return fail(POSEIDON_ERR_INVALID_ARG, "staleness must be in [1, 5]");
  for (const Layer& L : c->layers)
    if (L.registered) return fail(POSEIDON_ERR_STATE, "set the staleness before registering layers");
  if (c->arena_g) return fail(POSEIDON_ERR_STATE, "set the staleness before poseidon_ps_arena");
  c->stale = s;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_set_momentum(poseidon_ctx_t c, int32_t id, float mu, float weight_decay) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (!(mu >= 0.f && mu < 1.f) || !(weight_decay >= 0.f))
    return fail(POSEIDON_ERR_INVALID_ARG, "need 0 <= mu < 1 and weight_decay >= 0");
  if (id == -1) {
    for (auto& L : c->layers)
      if (L.registered && (st = set_momentum_one(c, L, mu, weight_decay)) != POSEIDON_OK) return st;
    for (auto& B : c->buckets)
      if ((st = set_momentum_one(c, B, mu, weight_decay)) != POSEIDON_OK) return st;
    return POSEIDON_OK;
  }
  Layer* L;
  st = check_layer(c, id, &L);
  if (st) return st;
  if (L->bucket >= 0)
    return fail(POSEIDON_ERR_STATE, "bucketed PS layers share their bucket's velocity: use layer_id -1");
  return set_momentum_one(c, *L, mu, weight_decay);
}

poseidon_status_t poseidon_set_lr(poseidon_ctx_t c, float lr) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  c->lr = lr;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_set_recon(poseidon_ctx_t c, int32_t id, int32_t recon) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (recon != POSEIDON_RECON_TF32 && recon != POSEIDON_RECON_FP32) return fail(POSEIDON_ERR_INVALID_ARG, "bad recon");
  if (id == -1) {
    for (auto& L : c->layers) {
      L.recon = recon;
      if (recon == POSEIDON_RECON_FP32) L.mn = false;
    }
    return POSEIDON_OK;
  }
  Layer* L;
  st = check_layer(c, id, &L);
  if (st) return st;
  L->recon = recon;
  if (recon == POSEIDON_RECON_FP32) L->mn = false;   // K1r reads the K-major layout (same buffer sizes)
  return POSEIDON_OK;
}

poseidon_status_t poseidon_sync_fc_sfb(poseidon_ctx_t c, int32_t id, const float* U, const float* V, float* W,
                                       float* bias, float lr, poseidon_stream_t producer) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme == POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not an SFB / SF-PS layer");
  if (!U || !V) return fail(POSEIDON_ERR_INVALID_ARG, "U/V is NULL");
  if (!W) W = L->W;
  if (!bias) bias = L->bias;
  if (!W) return fail(POSEIDON_ERR_INVALID_ARG, "no W given or bound");
  if (bias && !L->has_bias) return fail(POSEIDON_ERR_INVALID_ARG, "layer registered without bias");
  if (!aligned16(W)) return fail(POSEIDON_ERR_ALIGNMENT, "W must be 16-byte aligned");
  cudaStream_t ps = reinterpret_cast<cudaStream_t>(producer);
  if ((st = note_capture(c, ps)) != POSEIDON_OK) return st;
  st = producer_guard(c, *L, ps);
  if (st) return st;
  if (inplace_ok(c, *L, U, V, W)) return sfb_inplace(c, id, *L, U, V, W, bias, lr, ps);
  if (async_pack_ok(c, *L)) return sfb_async_pack(c, id, *L, U, V, W, bias, lr, ps);
  st = pack_sfb(c, *L, U, L->M, V, L->N, ps);
  if (st) return st;
  return sfb_after_pack(c, id, *L, W, bias, lr, ps);
}

poseidon_stream_t poseidon_stream(poseidon_ctx_t c, int32_t which) {
  if (check_ctx(c) != POSEIDON_OK) return nullptr;
  if (which == POSEIDON_STREAM_COMM) return reinterpret_cast<poseidon_stream_t>(c->comm_stream);
  if (which == POSEIDON_STREAM_RECON) return reinterpret_cast<poseidon_stream_t>(c->recon_stream);
  return nullptr;
}

poseidon_status_t poseidon_sfb_post_input(poseidon_ctx_t c, int32_t id, const float* V, int64_t ldV,
                                          poseidon_stream_t stream) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (!(c->flags & POSEIDON_FLAG_EARLY_V)) return fail(POSEIDON_ERR_STATE, "context created without FLAG_EARLY_V");
  if (L->scheme != POSEIDON_SCHEME_SFB) return fail(POSEIDON_ERR_STATE, "early input broadcast needs an SFB layer");
  if (!V || ldV < L->N) return fail(POSEIDON_ERR_INVALID_ARG, "V is NULL or ldV < N");
  if (L->v_posted) return fail(POSEIDON_ERR_STATE, "V already posted for this sync");
  cudaStream_t ps = reinterpret_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, ps)) != POSEIDON_OK) return st;
  st = producer_guard(c, *L, ps);   // the previous sync's K1 no longer reads the gather buffers
  if (st) return st;
  const int P = c->world;
  const bool round = (L->recon == POSEIDON_RECON_TF32);
  float* v_slot = L->Vg + (size_t)c->rank * slot_v(*L);
  cudaError_t err = L->mn ? cudaMemcpy2DAsync(v_slot, (size_t)L->N * 4, V, (size_t)ldV * 4, (size_t)L->N * 4,
                                              (size_t)L->K, cudaMemcpyDeviceToDevice, ps)
                          : launch_pack_t(V, ldV, v_slot, L->ldk, L->K, L->N, round, nullptr, ps);
  if (err != cudaSuccess) return cuda_fail(err, "pack V launch");
  EvSet& e = L->ev[c->iter % RING];
  CU_TRY(evrec(c, e.vready, ps));
  if (P > 1) {
    IterRecord& r = open_record(c);
    const size_t vcount = slot_v(*L);
    CU_TRY(evwait(c, c->comm_stream, e.vready));
    FZ(c->comm_stream);
    if (L->bcast) {
      const size_t vb = (size_t)((char*)L->Vg - (char*)L->symm);
      err = launch_sfb_bcast_nvls(c->nvls, L->win, 0, 0, vb + (size_t)c->rank * vcount * 4, (int64_t)vcount, 0, 0,
                                  kNvlsBlocks, c->comm_stream);
      if (err != cudaSuccess) return cuda_fail(err, "early V broadcast launch");
    } else {
      NC_TRY(ncclAllGather(L->Vg + (size_t)c->rank * vcount, L->Vg, vcount, ncclFloat32, c->comm, c->comm_stream));
    }
    r.sent += (uint64_t)vcount * 4u;
    r.recv += (uint64_t)vcount * 4u * (uint64_t)(P - 1);
    CU_TRY(evrec(c, e.vgath, c->comm_stream));
  } else {
    CU_TRY(evrec(c, e.vgath, ps));
  }
  L->v_posted = true;
  L->v_iter = c->iter;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_sync_ps(poseidon_ctx_t c, int32_t id, float* grad, float* W, int64_t n, float lr,
                                   poseidon_stream_t producer) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme != POSEIDON_SCHEME_PS) return fail(POSEIDON_ERR_STATE, "layer is not a PS layer");
  if (L->bucket >= 0 && (grad != nullptr && grad != L->grad))
    return fail(POSEIDON_ERR_STATE, "a bucketed PS layer syncs its arena buffers (pass NULL buffers)");
  if (L->bucket >= 0) grad = W = nullptr;
  if (grad || W) {
    if (!grad || !W) return fail(POSEIDON_ERR_INVALID_ARG, "pass both grad and W, or neither");
    if (grad != L->grad || W != L->Wps || n != L->n) {
      st = poseidon_bind_ps_buffers(c, id, grad, W, n, L->ps_flags);
      if (st) return st;
    }
  }
  if (!L->grad) return fail(POSEIDON_ERR_STATE, "no PS buffers given or bound");
  if ((st = note_capture(c, reinterpret_cast<cudaStream_t>(producer))) != POSEIDON_OK) return st;
  if (n != L->n) return fail(POSEIDON_ERR_SHAPE, "n does not match the bound buffers");
  cudaStream_t ps = reinterpret_cast<cudaStream_t>(producer);
  EvSet& e = L->ev[c->iter % RING];
  CU_TRY(evrec(c, e.ready, ps));
  L->last_iter = c->iter;
  if (c->ssp) {
    float* g = (L->in_arena && L->gsets.size() > 1) ? L->gsets[(size_t)next_set(c, *L)] : L->grad;
    return ssp_hook(c, id, *L, L->Wps, nullptr, g, lr);
  }
  if (L->bucket >= 0) {
    // bucketed: the bucket syncs once every member's gradient is ready (hooks fire in the same order
    // on every rank, so the bucket's collectives are issued at the same point everywhere)
    Layer& B = c->buckets[(size_t)L->bucket];
    if (++B.members_ready < B.members.size()) return POSEIDON_OK;
    B.members_ready = 0;
    const int32_t bid = MAX_LAYERS + L->bucket;
    for (int32_t m : B.members)
      if (m != id) CU_TRY(evwait(c, c->comm_stream, c->layers[(size_t)m].ev[c->iter % RING].ready));
    CU_TRY(evrec(c, B.ev[c->iter % RING].ready, ps));
    B.last_iter = c->iter;
    if (c->flags & POSEIDON_FLAG_DWBP_OFF) {
      B.pending = true;
      B.pending_lr = lr;
      B.pending_grad = B.grad;
      B.pending_W = B.Wps;
      c->pending_order.push_back(bid);
      open_record(c);
      return POSEIDON_OK;
    }
    return launch_ps_comm(c, bid, B, B.grad, B.Wps, lr, B.ev[c->iter % RING].ready);
  }
  if (c->flags & POSEIDON_FLAG_DWBP_OFF) {
    L->pending = true;
    L->pending_lr = lr;
    L->pending_grad = L->grad;
    L->pending_W = L->Wps;
    c->pending_order.push_back(id);
    open_record(c);
    return POSEIDON_OK;
  }
  return launch_ps_comm(c, id, *L, L->grad, L->Wps, lr, e.ready);
}

poseidon_status_t poseidon_backprop_hook(poseidon_ctx_t c, int32_t id, poseidon_stream_t stream) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (L->scheme == POSEIDON_SCHEME_PS) return poseidon_sync_ps(c, id, nullptr, nullptr, L->n, c->lr, stream);
  // SFB: the caller wrote its factors into the staging slot (poseidon_sfb_slot); pack them
  if (!L->W) return fail(POSEIDON_ERR_STATE, "SFB layer has no bound W (poseidon_bind_sfb_params)");
  if (!L->stU) return fail(POSEIDON_ERR_STATE, "SFB layer has no staging slot (call poseidon_sfb_slot first)");
  cudaStream_t ps = reinterpret_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, ps)) != POSEIDON_OK) return st;
  st = producer_guard(c, *L, ps);
  if (st) return st;
  st = pack_sfb(c, *L, L->stU, L->M, L->stV, L->N, ps);
  if (st) return st;
  return sfb_after_pack(c, id, *L, L->W, L->bias, c->lr, ps);
}

poseidon_status_t poseidon_flush(poseidon_ctx_t c, poseidon_stream_t stream) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (!c->ssp) return POSEIDON_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != POSEIDON_OK) return st;
  IterRecord& r = open_record(c);
  for (int32_t id = 0; id < (int32_t)c->layers.size(); ++id) {   // same order on every rank
    Layer& L = c->layers[id];
    if (!L.registered || L.pend.empty()) continue;
    EvSet& e = L.ev[c->iter % RING];
    CU_TRY(evrec(c, e.ready, s));
    CU_TRY(evwait(c, c->comm_stream, e.ready));
    CU_TRY(evrec(c, e.start, c->comm_stream));
    e.g_eff = e.ks_eff = e.start;
    while (!L.pend.empty()) {   // oldest first: every deferred update, in iteration order
      const Layer::Pend q = L.pend.front();
      L.pend.pop_front();
      const EvSet& src = L.ev[q.iter % RING];
      st = (L.scheme == POSEIDON_SCHEME_SFB) ? sfb_update(c, L, q.set, q.W, q.bias, q.lr, src.g_eff, e.ready, e)
                                             : ps_update_local(c, L, q.grad, L.Wps, q.lr, src.g_eff, e.ready, e);
      if (st) return st;
    }
    L.last_iter = c->iter;
    r.layers.push_back(id);
  }
  // the flush is an iteration of its own (its events live in ring slot c->iter): close and advance,
  // so hooks that follow a flush record into a fresh slot and the statistics never count a sync twice
  CU_TRY(evrec(c, r.bwd_end, s));
  r.closed = true;
  c->iter += 1;
  return POSEIDON_OK;
}

poseidon_status_t poseidon_wait_layer(poseidon_ctx_t c, int32_t id, poseidon_stream_t consumer) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if ((st = check_async(c)) != POSEIDON_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(consumer);
  if ((st = note_capture(c, cs)) != POSEIDON_OK) return st;
  if (c->flags & POSEIDON_FLAG_DWBP_OFF) {
    // traditional BP (Fig. dwbp (a)): the next iteration waits for every layer
    const IterRecord& r = c->rec[(c->iter + RING - 1) % RING];
    if (r.iter == c->iter - 1)
      for (int32_t lid : r.layers) CU_TRY(evwait(c, cs, resolve(c, lid).ev[r.iter % RING].done));
    return POSEIDON_OK;
  }
  const Layer& D = (L->bucket >= 0) ? c->buckets[(size_t)L->bucket] : *L;
  if (D.last_iter >= 0) CU_TRY(evwait(c, cs, D.ev[D.last_iter % RING].done));
  return POSEIDON_OK;
}

poseidon_status_t poseidon_iteration_end(poseidon_ctx_t c, poseidon_stream_t compute, poseidon_iter_stats_t* out) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if ((st = check_async(c)) != POSEIDON_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(compute);
  if ((st = note_capture(c, cs)) != POSEIDON_OK) return st;
  IterRecord& r = open_record(c);
  CU_TRY(evrec(c, r.bwd_end, cs));
  if (c->flags & POSEIDON_FLAG_DWBP_OFF) {
    // deferred syncs in the order the hooks fired, all after the whole backward
    for (int32_t id : c->pending_order) {
      Layer& L = resolve(c, id);
      if (!L.pending) continue;
      L.pending = false;
      st = (L.scheme != POSEIDON_SCHEME_PS)
               ? launch_factor_sync(c, id, L, L.pending_W, L.pending_bias, L.pending_lr, r.bwd_end)
               : launch_ps_comm(c, id, L, L.pending_grad, L.pending_W, L.pending_lr, r.bwd_end);
      if (st) return st;
    }
    c->pending_order.clear();
  }
  if (c->cap_id) {
    // captured step: the library's streams that joined the capture rejoin the caller's stream here (a graph
    // launch then covers every sync of the iteration; the next launch is ordered after all of them)
    cudaStream_t lib[2] = {c->comm_stream, c->recon_stream};
    for (int k = 0; k < 2; ++k) {
      cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
      unsigned long long id = 0;
      if (cudaStreamGetCaptureInfo(lib[k], &cst, &id) == cudaSuccess && cst == cudaStreamCaptureStatusActive &&
          id == c->cap_id) {
        CU_TRY(cudaEventRecord(c->join_ev[k], lib[k]));
        CU_TRY(cudaStreamWaitEvent(cs, c->join_ev[k], 0));
      }
    }
  }
  r.closed = true;
  c->iter += 1;
  if (out && c->cap_id) return fail(POSEIDON_ERR_STATE, "statistics of a captured iteration: read them after a replay");
  if (out) return poseidon_get_iter_stats(c, 0, out);
  return POSEIDON_OK;
}

poseidon_status_t poseidon_get_iter_stats(poseidon_ctx_t c, int32_t ago, poseidon_iter_stats_t* out) {
  poseidon_status_t st = check_ctx(c);
  if (st) return st;
  if (!out) return fail(POSEIDON_ERR_INVALID_ARG, "out is NULL");
  if (ago < 0 || ago >= RING - 1) return fail(POSEIDON_ERR_INVALID_ARG, "ago out of range");
  const int64_t it = c->iter - 1 - ago;
  if (it < 0) return fail(POSEIDON_ERR_STATE, "no such iteration");
  IterRecord& r = c->rec[it % RING];
  if (r.iter != it || !r.closed) return fail(POSEIDON_ERR_STATE, "iteration record overwritten");
  memset(out, 0, sizeof(*out));
  CU_TRY(cudaEventSynchronize(r.bwd_end));
  float exposed = 0.f, first_ready = 0.f;
  for (int32_t id : r.layers) {
    Layer& L = resolve(c, id);
    EvSet& e = L.ev[it % RING];
    CU_TRY(cudaEventSynchronize(e.done));
    exposed = std::max(exposed, elapsed(r.bwd_end, e.done));
    first_ready = std::max(first_ready, elapsed(e.ready, r.bwd_end));
    out->sync_total_ms += elapsed(e.start, e.done);
    out->queue_ms += elapsed(e.ready, e.start);
    if (L.scheme != POSEIDON_SCHEME_PS)
      out->recon_ms += elapsed(e.ks_eff, e.ke_eff);
    else
      out->ps_update_ms += elapsed(e.ks_eff, e.ke_eff);
  }
  out->exposed_ms = exposed;
  out->first_ready_to_bwd_end_ms = first_ready;
  out->nccl_bytes_sent = r.sent;
  out->nccl_bytes_recv = r.recv;
  out->n_layers = (int32_t)r.layers.size();
  out->iteration = (int32_t)it;
  return check_async(c);
}

poseidon_status_t poseidon_get_layer_stats(poseidon_ctx_t c, int32_t ago, int32_t id, poseidon_layer_stats_t* out) {
  Layer* L;
  poseidon_status_t st = check_layer(c, id, &L);
  if (st) return st;
  if (!out) return fail(POSEIDON_ERR_INVALID_ARG, "out is NULL");
  if (ago < 0 || ago >= RING - 1) return fail(POSEIDON_ERR_INVALID_ARG, "ago out of range");
  const int64_t it = c->iter - 1 - ago;
  if (it < 0) return fail(POSEIDON_ERR_STATE, "no such iteration");
  IterRecord& r = c->rec[it % RING];
  if (r.iter != it || !r.closed) return fail(POSEIDON_ERR_STATE, "iteration record overwritten");
  memset(out, 0, sizeof(*out));
  out->scheme = L->scheme;
  // a bucketed layer reports its bucket's sync (the same numbers for every member)
  const int32_t rid = (L->bucket >= 0) ? MAX_LAYERS + L->bucket : id;
  Layer* D = (L->bucket >= 0) ? &c->buckets[(size_t)L->bucket] : L;
  bool found = false;
  for (int32_t lid : r.layers) found |= (lid == rid);
  if (!found) return POSEIDON_OK;
  EvSet& e = D->ev[it % RING];
  CU_TRY(cudaEventSynchronize(e.done));
  CU_TRY(cudaEventSynchronize(r.bwd_end));
  out->launched = 1;
  out->ready_to_start_ms = elapsed(e.ready, e.start);
  out->comm_ms = elapsed(e.start, e.g_eff);
  out->kernel_ms = elapsed(e.ks_eff, e.ke_eff);
  out->start_to_done_ms = elapsed(e.start, e.done);
  out->done_after_bwd_end_ms = elapsed(r.bwd_end, e.done);
  out->pack_ms = e.packed ? elapsed(e.pstart, e.pack_async ? e.pend : e.ready) : 0.f;
  return POSEIDON_OK;
}

// ------------------------------------------- kernel-level entry points ----
poseidon_status_t poseidon_sfb_simulated(const float* U_all, const float* V_all, int32_t P, int64_t K, int64_t M,
                                         int64_t N, float* W, float* bias, float lr, int32_t recon,
                                         poseidon_stream_t stream) {
  if (!U_all || !V_all || !W || P < 1 || K < 0 || M <= 0 || N <= 0)
    return fail(POSEIDON_ERR_INVALID_ARG, "sfb_simulated: bad arguments");
  if (recon != POSEIDON_RECON_TF32 && recon != POSEIDON_RECON_FP32) return fail(POSEIDON_ERR_INVALID_ARG, "bad recon");
  if (!aligned16(W)) return fail(POSEIDON_ERR_ALIGNMENT, "W must be 16-byte aligned");
  if (K == 0) return POSEIDON_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t ldk = round_up(K, 4);
  const size_t ub = (size_t)P * M * ldk * 4, vb = (size_t)P * N * ldk * 4, bb = (size_t)P * M * 4;
  float *Ug = nullptr, *Vg = nullptr, *Bs = nullptr;
  CU_TRY(cudaMallocAsync(&Ug, ub, s));
  CU_TRY(cudaMallocAsync(&Vg, vb, s));
  CU_TRY(cudaMallocAsync(&Bs, bb, s));
  if (ldk != K) {
    CU_TRY(cudaMemsetAsync(Ug, 0, ub, s));
    CU_TRY(cudaMemsetAsync(Vg, 0, vb, s));
  }
  const bool round = recon == POSEIDON_RECON_TF32;
  cudaError_t err = cudaSuccess;
  for (int p = 0; p < P && err == cudaSuccess; ++p) {
    err = launch_pack_uv(U_all + (size_t)p * K * M, M, Ug + (size_t)p * M * ldk, M, Bs + (size_t)p * M,
                         V_all + (size_t)p * K * N, N, Vg + (size_t)p * N * ldk, N, ldk, K, round, s);
  }
  const float alpha = -lr / (float)P;
  if (err == cudaSuccess) {
    if (round && recon_tcgen05_supported(Ug, Vg, ldk, M, N, W))
      err = launch_recon_tcgen05(Ug, Vg, P, K, ldk, M, N, W, alpha, 1.0f, s);
    else
      err = launch_recon_simt(Ug, Vg, P, K, ldk, M, N, W, alpha, 1.0f, s);
  }
  if (err == cudaSuccess && bias) err = launch_bias_update(Bs, M, P, bias, M, alpha, s);
  cudaFreeAsync(Ug, s);
  cudaFreeAsync(Vg, s);
  cudaFreeAsync(Bs, s);
  if (err != cudaSuccess) return cuda_fail(err, "sfb_simulated launch");
  return POSEIDON_OK;
}

poseidon_status_t poseidon_ps_simulated(const float* grads, int32_t P, float* W, int64_t n, float lr,
                                        poseidon_stream_t stream) {
  if (!grads || !W || P < 1 || n < 0) return fail(POSEIDON_ERR_INVALID_ARG, "ps_simulated: bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t b, e, padded;
  poseidon_shard_range(n, P, 0, &b, &e, &padded);
  const float alpha = -lr / (float)P;
  for (int r = 0; r < P; ++r) {
    poseidon_shard_range(n, P, r, &b, &e, &padded);
    cudaError_t err = launch_ps_sim_update(grads + b, padded, P, W + b, e - b, alpha, s);
    if (err != cudaSuccess) return cuda_fail(err, "ps_simulated launch");
  }
  return POSEIDON_OK;
}

poseidon_status_t poseidon_ps_shard_update(const float* g, float* W, int64_t count, float alpha, float* stats,
                                           poseidon_stream_t stream) {
  if (!g || !W || count < 0) return fail(POSEIDON_ERR_INVALID_ARG, "ps_shard_update: bad arguments");
  cudaError_t err = launch_ps_shard_update(g, W, count, alpha, stats, reinterpret_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "ps_shard_update launch");
  return POSEIDON_OK;
}

poseidon_status_t poseidon_reconstruct_sgd(const float* Ug, const float* Vg, int32_t P, int64_t K, int64_t ldk,
                                           int64_t M, int64_t N, float* W, float alpha, int32_t recon,
                                           poseidon_stream_t stream) {
  if (!Ug || !Vg || !W || P < 1 || K < 0 || M <= 0 || N <= 0 || ldk < K)
    return fail(POSEIDON_ERR_INVALID_ARG, "reconstruct_sgd: bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t err;
  if (recon == POSEIDON_RECON_TF32) {
    if (!recon_tcgen05_supported(Ug, Vg, ldk, M, N, W))
      return fail(POSEIDON_ERR_ALIGNMENT, "tcgen05 path needs 16-B aligned buffers and ldk, N multiples of 4");
    err = launch_recon_tcgen05(Ug, Vg, P, K, ldk, M, N, W, alpha, 1.0f, s);
  } else if (recon == POSEIDON_RECON_FP32) {
    err = launch_recon_simt(Ug, Vg, P, K, ldk, M, N, W, alpha, 1.0f, s);
  } else {
    return fail(POSEIDON_ERR_INVALID_ARG, "bad recon");
  }
  if (err != cudaSuccess) return cuda_fail(err, "reconstruct_sgd launch");
  return POSEIDON_OK;
}

poseidon_status_t poseidon_reconstruct_sgd_mn(const float* U, int64_t ldu, int64_t ublk, const float* V, int64_t ldv,
                                              int64_t vblk, int32_t P, int64_t K, int64_t M, int64_t N, float* W,
                                              float alpha, poseidon_stream_t stream) {
  if (!U || !V || !W || P < 1 || K < 0 || M <= 0 || N <= 0 || ldu < M || ldv < N)
    return fail(POSEIDON_ERR_INVALID_ARG, "reconstruct_sgd_mn: bad arguments");
  if (K == 0) return POSEIDON_OK;
  if (!recon_tcgen05_mn_supported(U, ldu, ublk, V, ldv, vblk, P, K, M, N, W))
    return fail(POSEIDON_ERR_ALIGNMENT, "reconstruct_sgd_mn: 16-B aligned buffers, ldu/ldv/N (and block strides) "
                                        "multiples of 4, block strides >= K*ld");
  cudaError_t err = launch_recon_tcgen05_mn(U, ldu, ublk, V, ldv, vblk, P, K, M, N, W, alpha, 1.0f,
                                            reinterpret_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "reconstruct_sgd_mn launch");
  return POSEIDON_OK;
}

poseidon_status_t poseidon_reconstruct_sgd_rows(const float* Ug, const float* Vg, int32_t P, int64_t K,
                                                int64_t ldk, int64_t M, int64_t m0, int64_t m1, int64_t N,
                                                float* W, float alpha, int32_t recon, poseidon_stream_t stream) {
  if (!Ug || !Vg || !W || P < 1 || K < 0 || M <= 0 || N <= 0 || ldk < K || m0 < 0 || m1 < m0 || m1 > M)
    return fail(POSEIDON_ERR_INVALID_ARG, "reconstruct_sgd_rows: bad arguments");
  if (m1 == m0 || K == 0) return POSEIDON_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float* Ub = Ug + (size_t)m0 * ldk;
  float* Wb = W + (size_t)m0 * N;
  cudaError_t err;
  if (recon == POSEIDON_RECON_TF32) {
    if (!recon_tcgen05_supported(Ub, Vg, ldk, m1 - m0, N, Wb))
      return fail(POSEIDON_ERR_ALIGNMENT, "tcgen05 path needs 16-B aligned row blocks and ldk, N multiples of 4");
    err = launch_recon_tcgen05(Ub, Vg, P, K, ldk, m1 - m0, N, Wb, alpha, 1.0f, s, nullptr, M);
  } else if (recon == POSEIDON_RECON_FP32) {
    err = launch_recon_simt(Ub, Vg, P, K, ldk, m1 - m0, N, Wb, alpha, 1.0f, s, M);
  } else {
    return fail(POSEIDON_ERR_INVALID_ARG, "bad recon");
  }
  if (err != cudaSuccess) return cuda_fail(err, "reconstruct_sgd_rows launch");
  return POSEIDON_OK;
}

poseidon_status_t poseidon_pack_factors(const float* U, int64_t ldU, int64_t M, const float* V, int64_t ldV,
                                        int64_t N, int64_t K, int64_t ldk, int32_t round_tf32, float* u_dst,
                                        float* v_dst, float* colsum, poseidon_stream_t stream) {
  if (!U || !u_dst || M <= 0 || K < 0 || ldk < K || ldU < M || (V && (!v_dst || N <= 0 || ldV < N)))
    return fail(POSEIDON_ERR_INVALID_ARG, "pack_factors: bad arguments");
  if (K == 0) return POSEIDON_OK;
  cudaError_t err = launch_pack_uv(U, ldU, u_dst, M, colsum, V, ldV, v_dst, V ? N : 0, ldk, K, round_tf32 != 0,
                                   reinterpret_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "pack_factors launch");
  return POSEIDON_OK;
}

}  // extern "C"
