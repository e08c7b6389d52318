/*
 * poseidon.h — C ABI of libposeidon.so, a B200-native (sm_100a) implementation
 * of Poseidon's per-layer gradient synchronisation (Zhang et al., arXiv
 * 1512.06216): SACP (Alg. 3), sufficient-factor broadcasting (SFB, Sec. 4.3.1),
 * sharded parameter-server sync (PS, Alg. 1 master / Alg. 3 lines 1-3) and
 * distributed wait-free backprop scheduling (DWBP, Alg. 2).
 *
 * Citations "P:Lnnn" are lines of the paper's LaTeX source; readings
 * "Zn" are listed in DESIGN.md §3.
 *
 * General conventions
 *  - Every function returns poseidon_status_t (0 == POSEIDON_OK) unless stated.
 *    On failure nothing has been enqueued and poseidon_last_error() returns a
 *    thread-local message.  No C++ exception crosses this boundary.
 *  - All float pointers passed to sync/kernel entry points are fp32 DEVICE
 *    pointers on the context's device, 16-byte aligned, contiguous, row-major.
 *    The caller owns them; the library never frees caller memory.
 *  - Streams are CUDA runtime streams (cudaStream_t), passed as
 *    poseidon_stream_t; NULL means the legacy default stream.
 *  - Asynchrony: sync_* / backprop_hook / kernel entry points only ENQUEUE work
 *    and return immediately.  Results are valid after poseidon_wait_layer() on
 *    the consuming stream (or after synchronising the stream passed in).
 *  - A context is used from one host thread.  Collectives are issued in call
 *    order, which must be identical on every rank (top -> bottom layer order).
 *  - FC layer shapes follow the paper: W is M x N with M = output dim (length
 *    of the error message E_{i+1}) and N = input dim (reading Z8).
 *  - The update is plain SGD with the worker mean: W <- W + alpha * sum,
 *    alpha = -lr / P (readings Z1-Z4).
 */
#ifndef POSEIDON_H_
#define POSEIDON_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* poseidon_stream_t;

typedef enum {
  POSEIDON_OK = 0,
  POSEIDON_ERR_INVALID_ARG = -1,
  POSEIDON_ERR_NOT_INITIALIZED = -2,
  POSEIDON_ERR_CUDA = -3,
  POSEIDON_ERR_NCCL = -4,
  POSEIDON_ERR_SHAPE = -5,
  POSEIDON_ERR_ALIGNMENT = -6,
  POSEIDON_ERR_UNSUPPORTED = -7,
  POSEIDON_ERR_STATE = -8
} poseidon_status_t;

/* PS: full-gradient parameter server (Alg. 3 lines 1-3; also the rule's else-branch, reading Z7).
 * SFB: sufficient-factor broadcasting (Alg. 3 lines 6-8).
 * SFPS: the rule's else-branch executed literally (Alg. 3 lines 9-11, Adam-style
 *       P:L335): factors go to the master of each row block (rank q masters the output rows
 *       poseidon_shard_range(M, P, q)), the master reconstructs and updates its rows only, and the
 *       workers synchronise A_i from the masters (reading Z20).  Never returned by
 *       poseidon_choose_scheme; selected by scheme_override = 2 or POSEIDON_FLAG_SFPS. */
typedef enum { POSEIDON_SCHEME_PS = 0, POSEIDON_SCHEME_SFB = 1, POSEIDON_SCHEME_SFPS = 2 } poseidon_scheme_t;
typedef enum { POSEIDON_LAYER_CONV = 0, POSEIDON_LAYER_FC = 1 } poseidon_layer_kind_t;

/* Reconstruction kernel of the SFB path (step 3 of P:L331).
 *  TF32: K1, tcgen05.mma kind::tf32, TMA-fed, TMEM accumulators, fused SGD
 *        epilogue; factors rounded to TF32 (RN) when packed (reading Z12).
 *        Tolerance 2e-3 (Z13 metric).
 *  FP32: K1r, CUDA-core fp32 FMA tiles, fused SGD epilogue.  Tolerance 1e-5. */
typedef enum { POSEIDON_RECON_TF32 = 0, POSEIDON_RECON_FP32 = 1 } poseidon_recon_t;

/* Float counts of Alg. 3's cost rule, exact in 64 bits:
 *  sfb     = (P-1)^2 K (M+N)
 *  sf_ps   = P K (M+N) + P M N
 *  full_ps = 2 P M N           (reported only, never decides) */
typedef struct { uint64_t sfb, sf_ps, full_ps; } poseidon_costs_t;

/* Topology of one process/GPU.  nccl_id is the 128-byte ncclUniqueId created
 * by rank 0 with poseidon_get_unique_id() and broadcast by the caller (e.g.
 * torch.distributed); ignored when world == 1.  flags: POSEIDON_FLAG_*. */
typedef struct {
  int32_t rank, world, device;
  uint8_t nccl_id[128];
  uint32_t flags;
} poseidon_topology_t;

#define POSEIDON_FLAG_DWBP_OFF 0x1u   /* ablation: sync starts only at iteration_end (Fig. dwbp (a)) */
#define POSEIDON_FLAG_NO_PRIORITY 0x2u /* sync streams at default instead of highest priority */
#define POSEIDON_FLAG_NVLS_PS 0x4u     /* PS layers in the arena sync with one fused NVLink-SHARP kernel */
#define POSEIDON_FLAG_SYMM_SFB 0x8u    /* SFB gather buffers in NCCL symmetric windows (NCCL's symmetric-memory
                                         all-gather kernels); registration is collective, so every rank must
                                         register the same layers in the same order */
#define POSEIDON_FLAG_NVLS_SFB 0x10u   /* SFB factor "broadcast" by the library's own kernel on symmetric
                                         gather buffers instead of an NCCL all-gather (implies
                                         POSEIDON_FLAG_SYMM_SFB): LSA barrier, this rank's slots stored into
                                         every peer's buffers over NVLink (default) or as one NVLink-SHARP
                                         multicast store (env POSEIDON_SFB_BCAST=mc), LSA barrier */
#define POSEIDON_FLAG_SSP1 0x20u       /* stale synchronous parallel with staleness s = 1 (
                                         reading Z19): the update of a layer's sync t is applied at the
                                         layer's hook of iteration t+1, after that backward has read W, so
                                         forward t+1 reads every update of iterations <= t-1.  Gradient and
                                         factor buffers are double-buffered; PS layers need the arena.
                                         s = 2..5: poseidon_set_staleness (s + 1 buffer sets, update of t
                                         applied at hook t+s).  Incompatible with POSEIDON_FLAG_DWBP_OFF. */
#define POSEIDON_FLAG_SFPS 0x40u       /* FC layers the rule sends to the server (Alg. 3 else-branch) run as
                                         sharded SF-PS (POSEIDON_SCHEME_SFPS) instead of full-gradient PS.
                                         Not combined with POSEIDON_FLAG_SSP1. */
#define POSEIDON_FLAG_EARLY_V 0x80u    /* enables poseidon_sfb_post_input: an SFB layer's input factors V may be
                                         broadcast during the forward pass (BSP with DWBP only: not combined
                                         with POSEIDON_FLAG_SSP1 or POSEIDON_FLAG_DWBP_OFF) */
#define POSEIDON_FLAG_INPLACE_FACTORS 0x100u /* round 2 (BSP with DWBP, SFB layers): the library reads U and V of
                                         poseidon_sync_fc_sfb in place, asynchronously on its own streams, so no
                                         factor work stays on the caller's (backward's) stream: the pack (K3) runs
                                         on the stream the sync continues on (comm at world > 1, recon at 1).  The
                                         CALLER then keeps U and V unchanged until the layer's sync is done: e.g.
                                         it holds them until poseidon_wait_layer has ordered its stream after the
                                         sync (what the glue does).  (A torch caller could also record_stream the
                                         tensors on both poseidon_stream()s, but the caching allocator then defers
                                         and re-allocates blocks: measured step collapses.) */
#define POSEIDON_FLAG_INPLACE_MN 0x200u /* with POSEIDON_FLAG_INPLACE_FACTORS, for SFB layers with M and N multiples
                                         of 4 (TF32): no K3 pack.  At world == 1 (16-B aligned U / V) K1 consumes U
                                         and V MN-major where they are; at world > 1 the gather buffers are
                                         MN-major [P][K][M] / [P][K][N], this rank's slot is filled by a
                                         copy-engine memcpy and K1 reads them MN-major.  K1 forms the bias sums
                                         itself; the tensor core reads the fp32 factors as TF32 (13 low mantissa
                                         bits dropped) instead of the pack's RN rounding (reading Z12').  Set at
                                         init; a layer switched to POSEIDON_RECON_FP32 keeps the K-major pack. */

typedef struct poseidon_ctx* poseidon_ctx_t;

/* Per-iteration statistics from device events (milliseconds).
 *  exposed_ms    = max(0, max_i t(done_i) - t(bwd_end))  (sync time not hidden by backward)
 *  sync_total_ms = sum_i (t(done_i) - t(start_i))
 *  queue_ms      = sum_i (t(start_i) - t(ready_i))
 *  recon_ms      = sum of K1/K1r (+bias) kernel times; ps_update_ms = sum of K2 times
 *  first_ready_to_bwd_end_ms = t(bwd_end) - min_i t(ready_i)
 *  nccl_bytes_*  = bytes this rank handed to / received from NCCL */
typedef struct {
  float exposed_ms, sync_total_ms, queue_ms, recon_ms, ps_update_ms, first_ready_to_bwd_end_ms;
  uint64_t nccl_bytes_sent, nccl_bytes_recv;
  int32_t n_layers;
  int32_t iteration;
} poseidon_iter_stats_t;

/* Per-layer statistics of one iteration (milliseconds, device events).  pack_ms: the K3 factor pack
 * of a factor layer on the producer stream (0 for PS layers). */
typedef struct {
  float ready_to_start_ms, comm_ms, kernel_ms, start_to_done_ms, done_after_bwd_end_ms;
  int32_t scheme;
  int32_t launched;
  float pack_ms;
} poseidon_layer_stats_t;

/* ======================= the five named entry points ======================= */

/* Create a context for this process's GPU: one of the paper's P workers ("in a distributed setting with P
 * workers"; Alg. 2 "at iteration t on worker p"), one process per GPU.  world must equal
 * topo->world.
 * world > 1 creates an NCCL communicator from topo->nccl_id (collective over
 * all ranks) and requires single-node all-pairs peer access between the GPUs
 * the ranks actually use (their PCI bus ids are all-gathered through the new
 * communicator and checked with cudaDeviceCanAccessPeer; a peer GPU not visible
 * to this process is reached by NCCL through CUDA IPC).  Two ranks on one GPU or
 * a pair without peer access -> POSEIDON_ERR_UNSUPPORTED (there is no other
 * backend). */
poseidon_status_t poseidon_init(int32_t world, const poseidon_topology_t* topo, poseidon_ctx_t* out);

/* SACP decision, Alg. 3: kind != FC -> PS; FC -> SFB iff
 * (P-1)^2 K(M+N) <= PK(M+N) + PMN (tie -> SFB, Z5), else PS (the else branch
 * is executed as full-gradient PS, Z7).  Pure host integer code: needs no
 * context and no GPU.  Returns the scheme (>= 0) or a negative status for
 * M, N, K < 0, P < 1 or u64 overflow.  costs may be NULL. */
int32_t poseidon_choose_scheme(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                               poseidon_costs_t* costs);

/* SFB sync of one registered FC layer (Alg. 3 lines 6-8).
 *  U: K x M, row k = worker's error message E_{i+1} of sample k (dl/dy of the
 *     mean loss; the library never rescales by K, Z2).
 *  V: K x N, row k = layer input a_i of sample k.
 *  W: M x N (NULL -> bound W), bias: M (NULL -> bound bias or none).
 * Enqueues on `producer`: pack of U, V into this rank's slot of the gather
 * buffers (transposed to K-major, + per-worker bias column sums, TF32 RN
 * rounding on the TF32 path).  Then on
 * the library's streams: all-gather of all ranks' factors (NCCL, skipped at
 * P == 1) and the fused reconstruction + SGD  W += alpha * Ug^T Vg,
 * b += alpha * sum_rows Ug.  U and V may be reused after the producer stream
 * passes this point (with POSEIDON_FLAG_INPLACE_FACTORS at world == 1: only once
 * the layer's sync is done, see the flag).  K must equal the registered K.
 * SF-PS layers (POSEIDON_SCHEME_SFPS) take the same call: after the pack, each
 * rank sends its U rows of master q's block to q (NCCL send/recv) and all-gathers
 * V and the bias sums; master r runs K1 on its rows [rb, re) only
 * (W[rb:re] += alpha * sum_p U_p[:, rb:re]^T V_p); every master then broadcasts
 * its updated rows (ncclBroadcast, root q, in place) and every rank applies the
 * same bias update.  W must be the same-shaped replica on every rank. */
poseidon_status_t poseidon_sync_fc_sfb(poseidon_ctx_t ctx, int32_t layer_id, const float* U,
                                       const float* V, float* W, float* bias, float lr,
                                       poseidon_stream_t producer);

/* PS sync of one layer's flat buffer (Alg. 1 master P:L208-211, Alg. 3 lines
 * 1-3): grad and W are padded flat buffers of padded_n = P*S floats
 * (poseidon_shard_range) holding the layer's W row-major then bias, n real
 * elements, zero padding in grad.  In place: reduce-scatter(sum) of grad,
 * this rank's shard W[b,e) += alpha * gsum[b,e) (K2), all-gather of W.
 * grad/W NULL -> bound buffers.  After the call grad holds partial sums; it is
 * zeroed by the library iff the buffers were bound with POSEIDON_PS_ZERO_GRAD. */
poseidon_status_t poseidon_sync_ps(poseidon_ctx_t ctx, int32_t layer_id, float* grad, float* W,
                                   int64_t n, float lr, poseidon_stream_t producer);

/* DWBP trigger (Alg. 2 line 9): "layer `layer_id`'s gradient inputs
 * are complete on `stream`".  PS layers sync their bound buffers; SFB layers
 * sync the factors the caller wrote into the staging slot of
 * poseidon_sfb_slot() (packed like sync_fc_sfb does).  Starts the layer's
 * sync on the library streams right away (or at iteration_end under
 * POSEIDON_FLAG_DWBP_OFF). */
poseidon_status_t poseidon_backprop_hook(poseidon_ctx_t ctx, int32_t layer_id, poseidon_stream_t stream);

/* Early input broadcast (POSEIDON_FLAG_EARLY_V; DWBP's "start its communication once its gradients are
 * generated", applied to the half of the sufficient factors that exists before the backward): V, the
 * layer input a_i of Eq. 5 (K x N, row stride ldV >= N, device), is final
 * once the forward pass has produced it, so it is packed into this rank's slot on `stream` and its
 * broadcast (all-gather / broadcast kernel, whichever wire the layer uses) starts on the comm stream right
 * away, overlapping the rest of the forward and the backward.  The layer's next sync (sync_fc_sfb or
 * backprop_hook) then packs and broadcasts only U and the bias sums and reconstructs from the early V; its
 * V argument is ignored.  The result is bit-identical to the plain sync (the same values in the same gather
 * layout).  SFB layers only (ERR_STATE otherwise); at most one post per sync (ERR_STATE). */
poseidon_status_t poseidon_sfb_post_input(poseidon_ctx_t ctx, int32_t layer_id, const float* V, int64_t ldV,
                                          poseidon_stream_t stream);

/* Hardware figures for the measured-cost model (GB/s, TFLOP/s, microseconds). */
typedef struct {
  double nvlink_gbps;           /* per-direction peer bandwidth, e.g. 770 (measured peer copy) */
  double hbm_gbps;              /* e.g. 6543.7 (round-1 MEASURED_PEAKS.json; the binding's default) */
  double tensor_tflops;         /* TF32 dense, e.g. 669.6 (round-1 sustained; the binding's default) */
  double collective_latency_us; /* per collective launch + sync, e.g. 10 */
} poseidon_hw_t;

/* Measured-cost SACP variant, reported BESIDE the paper's rule, never used by it:
 * predicted per-rank times of the SFB execution (pack + all-gather + K1) and of the PS execution
 * (local dW GEMM + reduce-scatter + K2 + all-gather) from an alpha-beta NVLink model and the
 * HBM / tensor rooflines; returns the faster scheme (non-FC -> PS) or a negative status.
 * Pure host code.  t_sfb_us / t_ps_us may be NULL. */
int32_t poseidon_choose_scheme_model(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                                     const poseidon_hw_t* hw, double* t_sfb_us, double* t_ps_us);
/* The same model with SF-PS (Alg. 3's else-branch executed literally, reading Z20) as a third execution:
 * pack + V all-gather + U rows to their masters + K1 on the largest master's rows + row push.  Returns the
 * predicted-fastest POSEIDON_SCHEME_* (non-FC -> PS) or a negative status; pure host code; outputs
 * nullable. */
int32_t poseidon_choose_scheme_model3(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                                      const poseidon_hw_t* hw, double* t_sfb_us, double* t_ps_us,
                                      double* t_sfps_us);

/* ================================ helpers ================================= */

/* ncclGetUniqueId into out[128] (call on rank 0 only). */
poseidon_status_t poseidon_get_unique_id(uint8_t out[128]);

/* Shard map of the PS path (Alg. 1: the master "updates the part of model parameters for which a
 * corresponding gradient is received"; one shard per rank, reading Z11): S = 32*ceil(n/(32P)),
 * padded_n = P*S, rank r owns
 * [min(rS,n), min((r+1)S,n)) (possibly empty).  Pure host code. */
poseidon_status_t poseidon_shard_range(int64_t n, int32_t P, int32_t rank, int64_t* begin,
                                       int64_t* end, int64_t* padded_n);

/* Register layer `layer_id` (0 <= id < 4096): kind, M x N weight, per-worker
 * batch K, has_bias; the SACP decision of Alg. 3 is taken here, once
 * per layer.  scheme_override: -1 -> SACP rule, else the scheme to use
 * (C2 forces PS; 2 = SF-PS, FC only).  chosen_scheme may be NULL.  With
 * POSEIDON_FLAG_SFPS an FC layer the rule sends to PS is registered as SF-PS.
 * SFB and SF-PS layers get library-owned
 * gather buffers, rank-major with K-major blocks (the tensor cores consume
 * TF32 operands K-major): Ug [P][M][ldk], Vg [P][N][ldk], Bs [P][M] (per-worker
 * column sums of U for the bias), ldk = roundup(K,4), padding zero.
 * Re-registering a layer waits for its previous sync. */
poseidon_status_t poseidon_register_layer(poseidon_ctx_t ctx, int32_t layer_id, int32_t kind,
                                          int64_t M, int64_t N, int64_t K, int32_t has_bias,
                                          int32_t scheme_override, int32_t* chosen_scheme);

/* Staging slot of an SFB / SF-PS layer for poseidon_backprop_hook: library-owned
 * device buffers U [K x M] (*ld_u = M) and V [K x N] (*ld_v = N), row-major,
 * allocated on first call.  The caller writes the factors there (ordered
 * before the hook's stream), then calls poseidon_backprop_hook.  Errors: ERR_STATE (a PS layer), ERR_CUDA
 * (allocation). */
poseidon_status_t poseidon_sfb_slot(poseidon_ctx_t ctx, int32_t layer_id, float** U_slot,
                                    int64_t* ld_u, float** V_slot, int64_t* ld_v);

#define POSEIDON_PS_ZERO_GRAD 0x1u
/* Bind a PS layer's padded flat buffers: grad and W caller-owned device buffers of padded_n floats each
 * (poseidon_shard_range), 16-byte aligned, holding W row-major then the bias (n = M*N, + M with bias).
 * flags: POSEIDON_PS_ZERO_GRAD -> the library zeroes grad (padding included) after each sync.  Errors:
 * ERR_STATE (unregistered or not a PS layer), ERR_INVALID_ARG (NULL), ERR_ALIGNMENT, ERR_SHAPE (n). */
poseidon_status_t poseidon_bind_ps_buffers(poseidon_ctx_t ctx, int32_t layer_id, float* grad,
                                           float* W, int64_t n, uint32_t flags);
/* Bind an SFB / SF-PS layer's parameters for poseidon_backprop_hook: W caller-owned M x N row-major
 * device buffer (16-byte aligned), bias M floats or NULL.  Errors: ERR_STATE (a PS layer),
 * ERR_INVALID_ARG (W NULL, or a bias for a layer registered without one). */
poseidon_status_t poseidon_bind_sfb_params(poseidon_ctx_t ctx, int32_t layer_id, float* W, float* bias);

/* PS arena (collective over all ranks when world > 1): allocates ONE padded
 * gradient buffer and ONE parameter buffer holding every registered PS layer
 * (each layer's segment padded_n floats, 4 KB aligned), zero-filled, and binds
 * each PS layer to its segments with POSEIDON_PS_ZERO_GRAD.  The caller copies
 * its initial parameters in (poseidon_ps_layer_buffers) and makes its tensors
 * views of them.  With POSEIDON_FLAG_NVLS_PS the arenas are NCCL symmetric
 * windows (ncclMemAlloc + ncclCommWindowRegister) and each PS sync becomes ONE
 * kernel: multimem.ld_reduce of the shard across all ranks (NVSwitch sum) ->
 * SGD -> multimem.st of the updated shard to every rank -> zero the local
 * gradient.  *nvls_active (nullable) = 1 if that path is active;
 * otherwise the arena is plain device memory and the NCCL path is used. */
poseidon_status_t poseidon_ps_arena(poseidon_ctx_t ctx, int32_t* nvls_active);
/* PS layer bucketing (BSP only): call before poseidon_ps_arena, identically on every rank.
 * Runs of consecutive PS layers (layer-id order) whose 128-B aligned sizes add up to at most
 * bucket_bytes share one contiguous arena span and sync as ONE flat buffer (one fused NVLS kernel, or
 * one reduce-scatter / K2 / all-gather) once the last member's hook has fired; a run of one layer
 * stays unbucketed.  Members' stats report the bucket's sync.  0 (default) disables bucketing. */
poseidon_status_t poseidon_set_ps_buckets(poseidon_ctx_t ctx, int64_t bucket_bytes);
/* A PS layer's arena segments: *grad = the gradient buffer the layer's NEXT sync reduces (with
 * POSEIDON_FLAG_SSP1 the s + 1 buffers rotate: re-point the parameters' gradients after every
 * iteration), *W = its parameters, *padded_n = segment length in floats. */
poseidon_status_t poseidon_ps_layer_buffers(poseidon_ctx_t ctx, int32_t layer_id, float** grad, float** W,
                                            int64_t* padded_n);
/* How SFB layer `layer_id` moves its factors at world > 1: 0 = NCCL all-gather on plain device
 * buffers, 1 = NCCL all-gather on symmetric-window buffers (FLAG_SYMM_SFB), 2 = the library's
 * broadcast kernel (FLAG_NVLS_SFB), 3 = SF-PS layer (NCCL send/recv of U row blocks, all-gather of V, broadcast of
 * the masters' W rows).  Negative status for a bad id or a PS layer. */
int32_t poseidon_sfb_path(poseidon_ctx_t ctx, int32_t layer_id);

/* The library's streams (cudaStream_t as poseidon_stream_t), e.g. for the caller's allocator to order
 * buffer reuse after in-place factor reads (POSEIDON_FLAG_INPLACE_FACTORS).  NULL for a bad ctx / which. */
#define POSEIDON_STREAM_COMM 0
#define POSEIDON_STREAM_RECON 1
poseidon_stream_t poseidon_stream(poseidon_ctx_t ctx, int32_t which);
/* Human-readable state of the fused NVLS PS path ("active", "not requested", or the NCCL error). */
const char* poseidon_nvls_status(poseidon_ctx_t ctx);

/* lr (the stepsize epsilon of Eq. 3) used by poseidon_backprop_hook from the next hook on
 * (sync_* take theirs as an argument).
 * ERR_NOT_INITIALIZED for a NULL context. */
poseidon_status_t poseidon_set_lr(poseidon_ctx_t ctx, float lr);

/* Lambda of Eq. 3 / Alg. 3 line 8, applied once at the aggregation point
 * (oracle O4m):  g = (1/P) sum_p grad_p;  v = mu v + lr (g + weight_decay * w);
 * w -= v, for every parameter (weights and biases).  Velocity buffers are library-owned and
 * zero-initialised on first use: SFB layers keep a replicated M x N (+ M) velocity (on the TF32 path
 * K1's epilogue streams W and the velocity once and applies both, 16 B / element; the fp32 K1r path
 * updates the velocity and a second elementwise pass applies it); PS layers keep only the velocity of this
 * rank's shard (the shard owner is the only one that updates it).  layer_id -1 = every registered
 * layer; mu = weight_decay = 0 returns the layer to plain SGD.  0 <= mu < 1, weight_decay >= 0. */
poseidon_status_t poseidon_set_momentum(poseidon_ctx_t ctx, int32_t layer_id, float mu, float weight_decay);
/* Reconstruction kernel of a factor layer (POSEIDON_RECON_TF32: K1 on tcgen05, POSEIDON_RECON_FP32: K1r),
 * layer_id -1 = every layer.  Takes effect at the layer's next pack (the TF32 path rounds the factors when
 * packing).  Errors: ERR_INVALID_ARG (bad recon), ERR_STATE (unregistered layer). */
poseidon_status_t poseidon_set_recon(poseidon_ctx_t ctx, int32_t layer_id /* -1: all */, int32_t recon);

/* SSP (POSEIDON_FLAG_SSP1): apply every layer's deferred update now (in layer-id order, identical on
 * every rank: collective).  Call it on all ranks after the last iteration (and before reading the
 * parameters); afterwards poseidon_wait_layer orders a consumer after the updates.  The flush is an
 * iteration record of its own: it closes and advances the iteration counter (its statistics are
 * poseidon_get_iter_stats(ago = 0)), so training may continue after it.  No-op without SSP. */
poseidon_status_t poseidon_flush(poseidon_ctx_t ctx, poseidon_stream_t stream);

/* SSP staleness s ("a worker at iteration t reads parameters that contain all updates of iterations
 * <= t - s - 1"), round 2: a context created with POSEIDON_FLAG_SSP1 runs s = 1; this call sets
 * 1 <= s <= 5 before any layer is registered and before poseidon_ps_arena.  Each layer then keeps s + 1 gather /
 * gradient sets used round robin, and the update of iteration t - s is applied at the layer's hook of
 * iteration t (poseidon_flush applies every deferred one).  Errors: STATE (no SSP context, layers or arena
 * already set up), INVALID_ARG (s out of range). */
poseidon_status_t poseidon_set_staleness(poseidon_ctx_t ctx, int32_t s);

/* Next-forward barrier: `consumer` waits until layer_id's latest sync is done
 * (under DWBP_OFF: until every layer's sync of the last iteration is done).  DWBP "allows partial
 * parameter updating on the layer": the next forward of layer i waits for layer i's sync only. */
poseidon_status_t poseidon_wait_layer(poseidon_ctx_t ctx, int32_t layer_id, poseidon_stream_t consumer);

/* Mark the end of backward on `compute` (the end of Alg. 2's loop over layers; records bwd_end; under DWBP_OFF
 * launches the deferred syncs), close the iteration and, if out != NULL,
 * block until its syncs are done and fill the statistics.
 * CUDA graphs (round 2): a whole training step may be captured by stream capture on the caller's stream
 * (BSP with DWBP; e.g. torch.cuda.graph around forward, backward and this call).  Every entry point that
 * takes a stream notices the capture; the library's streams then fork from and join the capture through
 * internal event twins, its statistics events become event-record nodes (valid after each replay:
 * poseidon_get_iter_stats(ago = 0) describes the latest replay), waits on earlier iterations are dropped
 * (graph launches on one stream are ordered as a whole), and here the library's streams rejoin `compute`,
 * so one replay is one complete iteration.  out must be NULL while capturing (POSEIDON_ERR_STATE). */
poseidon_status_t poseidon_iteration_end(poseidon_ctx_t ctx, poseidon_stream_t compute, poseidon_iter_stats_t* out);

/* Statistics of a finished iteration, `ago` iterations back (0 = the last one
 * closed by iteration_end; at most 31).  Blocks on that iteration's events. */
poseidon_status_t poseidon_get_iter_stats(poseidon_ctx_t ctx, int32_t ago, poseidon_iter_stats_t* out);
poseidon_status_t poseidon_get_layer_stats(poseidon_ctx_t ctx, int32_t ago, int32_t layer_id,
                                           poseidon_layer_stats_t* out);

/* Number of library kernels launched so far by this process (all contexts). */
uint64_t poseidon_launch_count(void);

/* Frees everything the context owns (collective at world > 1: ncclCommDestroy).  A CUDA graph that captured
 * this context's NCCL collectives (stream capture of a step, see poseidon_iteration_end) must be destroyed
 * first: NCCL keeps the communicator's persistent resources alive for it, and the destroy would wait. */
poseidon_status_t poseidon_finalize(poseidon_ctx_t ctx);
const char* poseidon_last_error(void);
int32_t poseidon_version(void);

/* ============ kernel-level entry points (tests, microbenchmarks) ============
 * These run the hot-path kernels on caller buffers without a communicator:
 * "simulated workers" lay the P workers' data rank-major in one buffer, the
 * way the all-gather leaves it, so multi-worker arithmetic is exercised on
 * one GPU.  No context needed. */

/* SFB (P:L328-331 steps (1)-(3), Alg. 3 lines 6-8) with P_sim simulated workers on one GPU: U_all [P_sim*K x M] and
 * V_all [P_sim*K x N] (worker p = rows [pK,(p+1)K)), W [M x N], bias [M]|NULL.
 * Packs each worker block (K3, column sums, rounding for TF32) into scratch
 * gather buffers, then runs the reconstruction (K1 or K1r) and the bias
 * update with alpha = -lr / P_sim.  Scratch is owned by the library. */
poseidon_status_t poseidon_sfb_simulated(const float* U_all, const float* V_all, int32_t P_sim,
                                         int64_t K, int64_t M, int64_t N, float* W, float* bias,
                                         float lr, int32_t recon, poseidon_stream_t stream);

/* PS (Alg. 1 master P:L208-211, Alg. 3 lines 1-3) with P_sim simulated workers: grads [P_sim x padded_n] (padded flat
 * buffers), W [padded_n].  For every shard r of the map, W[b_r,e_r) +=
 * alpha * sum_p grads[p][b_r,e_r) summed in worker order (the fused
 * reduce + K2 a single GPU can do for all shards), alpha = -lr / P_sim. */
poseidon_status_t poseidon_ps_simulated(const float* grads, int32_t P_sim, float* W, int64_t n,
                                        float lr, poseidon_stream_t stream);

/* K2 alone (the master's update of its part of the parameters, Alg. 1):
 * W[i] = fmaf(alpha, g[i], W[i]) for i in [0,count); if stats !=
 * NULL (2 floats, device, caller-zeroed) accumulates sum((alpha g)^2) and the
 * count of non-finite updates via warp-shuffle reductions. */
poseidon_status_t poseidon_ps_shard_update(const float* g, float* W, int64_t count, float alpha,
                                           float* stats, poseidon_stream_t stream);

/* Reconstruction alone (K1 / K1r; SFB step (3), Alg. 3 line 8) on already-gathered, already-rounded
 * buffers in the gather layout: W[M x N] += alpha * sum_p sum_k<K
 * Ug[p][m][k] Vg[p][n][k], Ug [P][M][ldk], Vg [P][N][ldk], ldk >= K.  The
 * TF32 path needs ldk and N multiples of 4 and 16-byte aligned buffers. */
poseidon_status_t poseidon_reconstruct_sgd(const float* Ug, const float* Vg, int32_t P, int64_t K, int64_t ldk,
                                           int64_t M, int64_t N, float* W, float alpha, int32_t recon,
                                           poseidon_stream_t stream);

/* Reconstruction alone on the factors in the layer's own (MN-major) layout, no pack (round 2, step (3) of
 * SFB P:L331, Eq. 5): W[M x N] += alpha * sum_p sum_k<K U[p][k][m] V[p][k][n], where worker block p
 * of U starts at U + p*ublk and its row k at + k*ldu (M contiguous: the error messages dl/dy [K x M] exactly
 * as the backward wrote them), V alike with ldv / vblk (the layer input [K x N]).  tcgen05 only
 * (POSEIDON_RECON_TF32 semantics; the tensor core reads fp32 operands as TF32, i.e. drops their 13 low
 * mantissa bits, reading Z12'); needs U, V, W 16-byte aligned, ldu >= M, ldv >= N, ldu, ldv, N multiples of
 * 4 and, for P > 1, ublk >= K*ldu and vblk >= K*ldv multiples of 4 (ignored at P = 1).  Nothing is
 * allocated; errors: INVALID_ARG, ALIGNMENT (a layout the TMA maps cannot express), CUDA. */
poseidon_status_t poseidon_reconstruct_sgd_mn(const float* U, int64_t ldu, int64_t ublk, const float* V, int64_t ldv,
                                              int64_t vblk, int32_t P, int64_t K, int64_t M, int64_t N, float* W,
                                              float alpha, poseidon_stream_t stream);

/* The SF-PS master's reconstruction (reading Z20): rows [m0, m1) only of the above,
 * W[m][n] += alpha * sum_p sum_k<K Ug[p][m][k] Vg[p][n][k] for m0 <= m < m1 and every n, with
 * Ug [P][M][ldk] the full gather buffer (M rows per worker block) and W the full M x N matrix;
 * rows outside [m0, m1) are not touched.  0 <= m0 <= m1 <= M.  TF32 path: as above, and
 * W + m0*N, Ug + m0*ldk must stay 16-byte aligned (N, ldk multiples of 4). */
poseidon_status_t poseidon_reconstruct_sgd_rows(const float* Ug, const float* Vg, int32_t P, int64_t K,
                                                int64_t ldk, int64_t M, int64_t m0, int64_t m1, int64_t N,
                                                float* W, float alpha, int32_t recon, poseidon_stream_t stream);

/* K3 alone (step (1) of SFB: "decouple grad W_p into two vectors u_p and v_p", Eq. 5): pack
 * worker factors into the gather layout the reconstruction consumes.
 *   U: K x M (row stride ldU >= M), V: K x N (row stride ldV >= N; NULL -> U only), device, fp32.
 *   u_dst: M x ldk, v_dst: N x ldk (ldk >= K, multiple of 4), u_dst[m*ldk + k] = U[k*ldU + m] (likewise V);
 *   columns k in [K, ldk) are NOT written.  round_tf32 != 0: the packed values are rounded to TF32 with
 *   round-to-nearest, ties away from zero (cvt.rna, reading Z12).  colsum (M floats or NULL): sum_k U[k][m]
 *   of the UNROUNDED values in fp32 (the bias gradient, reading Z9), in a fixed order (deterministic).
 * One launch for U and V.  Errors: ERR_INVALID_ARG (NULL U / u_dst, K < 0, ldk < K, ld < cols). */
poseidon_status_t poseidon_pack_factors(const float* U, int64_t ldU, int64_t M, const float* V, int64_t ldV,
                                        int64_t N, int64_t K, int64_t ldk, int32_t round_tf32, float* u_dst,
                                        float* v_dst, float* colsum, poseidon_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* POSEIDON_H_ */
