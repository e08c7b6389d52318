"""Poseidon fp64 CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this module.  The product path
(``paper_1512_06216_b200`` + ``libposeidon.so``) never imports it, and this
module never imports the product: the two share no code.  The only shared
module is ``synthetic`` (seeded random inputs, none of the method's arithmetic).

Everything here is the plain definition of what Poseidon's gradient
synchronisation computes, written out in float64 (numpy) in the paper's order
and notation.  Citations are to ``PAPER.md`` lines (P:Lnnn) of arXiv 1512.06216
and to the readings Z1..Z18 recorded in DESIGN.md §3.

Conventions:
  * an FC layer's weight ``W`` is M x N with M = output dim, N = input dim
    ("E_{i+1}, which is an M dimensional vector").
  * worker p's sufficient factors are the K rows of ``U_p`` (K x M, the
    per-sample error messages E_{i+1}) and of ``V_p`` (K x N, the per-sample
    layer inputs a_i), so  grad W_p = sum_k U_p[k]^T V_p[k]  (Eq. 5).
  * aggregation over workers is a mean: alpha = -lr / P (reading Z1), descent
    sign (Z3), Lambda = 0 (Z4).

Parity status of every function is pinned by ``tests/test_oracle.py``; no
function here is "parity unpinned".
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

LAYER_CONV = 0
LAYER_FC = 1
SCHEME_PS = 0
SCHEME_SFB = 1
SHARD_ALIGN = 32  # elements (128 B) — reading Z11


# --------------------------------------------------------------------------
# O1 — SACP cost model and decision (Alg. 3; costs P:L333)
# --------------------------------------------------------------------------
def cost_sfb(M: int, N: int, K: int, P: int) -> int:
    """SFB float volume "(P-1)^2 K(M+N)" verbatim from P:L333 (reading Z6)."""
    return (P - 1) ** 2 * K * (M + N)


def cost_sf_ps(M: int, N: int, K: int, P: int) -> int:
    """Adam-style SF-via-PS volume "PK(M+N) + PMN"."""
    return P * K * (M + N) + P * M * N


def cost_full_ps(M: int, N: int, K: int, P: int) -> int:
    """Full-matrix PS volume "2PMN".  Reported only, never decides."""
    return 2 * P * M * N


def costs(M: int, N: int, K: int, P: int) -> Tuple[int, int, int]:
    """(C_sfb, C_sf_ps, C_full) of P:L333 / P:L335 as exact Python integers."""
    return cost_sfb(M, N, K, P), cost_sf_ps(M, N, K, P), cost_full_ps(M, N, K, P)


def choose_scheme(kind: int, M: int, N: int, K: int, P: int) -> int:
    """Alg. 3: non-FC layers go to the parameter server
    (P:L359-361); an FC layer broadcasts its sufficient factors iff
    (P-1)^2 K(M+N) <= PK(M+N) + PMN (tie -> SFB, reading Z5),
    otherwise it is synchronised server-side (executed as full-gradient PS,
    reading Z7)."""
    if kind != LAYER_FC:
        return SCHEME_PS
    return SCHEME_SFB if cost_sfb(M, N, K, P) <= cost_sf_ps(M, N, K, P) else SCHEME_PS


# --------------------------------------------------------------------------
# O2 — shard map of a PS layer's flat buffer (reading Z11; paper silent,
# single "master node" P:L207-212)
# --------------------------------------------------------------------------
def shard_size(n: int, P: int) -> int:
    """S(n, P) = 32 * ceil(n / (32 P)): one shard of the PS layer per rank (the master of Alg. 1,
    P:L208-211, split over the P ranks; reading Z11)."""
    return SHARD_ALIGN * (-(-n // (SHARD_ALIGN * P)))


def shard_range(n: int, P: int, rank: int) -> Tuple[int, int, int]:
    """Rank ``rank`` owns [min(rS, n), min((r+1)S, n)); returns (begin, end, padded_n) (reading Z11;
    the master "updates the part of model parameters for which a corresponding gradient is
    received")."""
    S = shard_size(n, P)
    return min(rank * S, n), min((rank + 1) * S, n), P * S


# --------------------------------------------------------------------------
# The FC layer + softmax cross-entropy used by the brute-force pins (O3, O7)
# --------------------------------------------------------------------------
def fc_forward(W: np.ndarray, b: np.ndarray, X: np.ndarray) -> np.ndarray:
    """y = W x + b for every row x of X (K x N) -> K x M: the FC layer of P:L322-324 (W is M x N,
    E_{i+1} is M-dimensional, a_i N-dimensional)."""
    return X @ W.T + b[None, :]


def softmax(z: np.ndarray) -> np.ndarray:
    """Row-wise softmax: the loss layer on top of the FC layer in the brute-force pins (the paper's
    models end in a softmax classifier, P:L436 / P:L481)."""
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


def mean_ce_loss(W: np.ndarray, b: np.ndarray, X: np.ndarray, labels: np.ndarray) -> float:
    """l = (1/#samples) * sum_samples -log softmax(W x + b)[label]: the loss l of Alg. 2,
    a mean over the batch (reading Z2)."""
    y = fc_forward(W, b, X)
    y = y - y.max(axis=1, keepdims=True)
    logp = y - np.log(np.exp(y).sum(axis=1, keepdims=True))
    return float(-logp[np.arange(len(labels)), labels].mean())


def error_messages(W: np.ndarray, b: np.ndarray, X: np.ndarray, labels: np.ndarray,
                   denom: int) -> np.ndarray:
    """Per-sample E_{i+1} = dl/dy (the error message of P:L324) for the mean CE loss with ``denom``
    samples: (softmax(y) - onehot(label)) / denom  (K x M)."""
    s = softmax(fc_forward(W, b, X))
    s[np.arange(len(labels)), labels] -= 1.0
    return s / float(denom)


def fd_gradient(W: np.ndarray, b: np.ndarray, X: np.ndarray, labels: np.ndarray,
                h: float = 1e-6) -> Tuple[np.ndarray, np.ndarray]:
    """O3: dl/dW and dl/db by central finite differences, element by element (brute force; for tiny
    layers only): the gradient that Eq. 5 claims the factors reconstruct exactly."""
    gW = np.zeros_like(W)
    gb = np.zeros_like(b)
    for i in range(W.shape[0]):
        for j in range(W.shape[1]):
            Wp = W.copy(); Wp[i, j] += h
            Wm = W.copy(); Wm[i, j] -= h
            gW[i, j] = (mean_ce_loss(Wp, b, X, labels) - mean_ce_loss(Wm, b, X, labels)) / (2 * h)
    for i in range(b.shape[0]):
        bp = b.copy(); bp[i] += h
        bm = b.copy(); bm[i] -= h
        gb[i] = (mean_ce_loss(W, bp, X, labels) - mean_ce_loss(W, bm, X, labels)) / (2 * h)
    return gW, gb


# --------------------------------------------------------------------------
# Eq. 5: gradient reconstruction from sufficient factors
# --------------------------------------------------------------------------
def reconstruct_loops(U: np.ndarray, V: np.ndarray) -> np.ndarray:
    """sum_k u_k v_k^T with explicit loops k -> m -> n (Eq. 5).
    Pure-Python loops: tiny inputs only."""
    K, M = U.shape
    N = V.shape[1]
    G = np.zeros((M, N), dtype=np.float64)
    for k in range(K):
        for m in range(M):
            u = float(U[k, m])
            for n in range(N):
                G[m, n] += u * float(V[k, n])
    return G


def reconstruct(U: np.ndarray, V: np.ndarray) -> np.ndarray:
    """sum_k u_k v_k^T = U^T V (Eq. 5), one library matmul in float64."""
    return np.asarray(U, dtype=np.float64).T @ np.asarray(V, dtype=np.float64)


# --------------------------------------------------------------------------
# O4 — the synchronous step, by definition (Eq. 4 P:L146 with readings Z1-Z4)
# --------------------------------------------------------------------------
def sync_step(W: np.ndarray, b, Us: Sequence[np.ndarray], Vs: Sequence[np.ndarray],
              lr: float) -> Tuple[np.ndarray, np.ndarray]:
    """Eq. 4 with readings Z1-Z4: W' = W - lr * (1/P) * sum_p G_p,
    G_p = sum_k U_p[k]^T V_p[k] (Eq. 5); b' = b - lr * (1/P) * sum_p sum_k U_p[k].  Workers p = 0..P-1
    in order."""
    P = len(Us)
    W = np.asarray(W, dtype=np.float64)
    G = np.zeros_like(W)
    gb = np.zeros(W.shape[0], dtype=np.float64)
    for p in range(P):
        G += reconstruct(Us[p], Vs[p])
        gb += np.asarray(Us[p], dtype=np.float64).sum(axis=0)
    W1 = W - lr * (1.0 / P) * G
    b1 = None if b is None else np.asarray(b, dtype=np.float64) - lr * (1.0 / P) * gb
    return W1, b1


# --------------------------------------------------------------------------
# O5 — SFB simulated: all-gather then one reconstruction (Alg. 3
# lines 366-368)
# --------------------------------------------------------------------------
def sfb_simulated(W, b, Us, Vs, lr):
    """SFB: every worker receives the rank-major concatenation [U_1..U_P], [V_1..V_P]
    (the broadcast, step 2) and applies the reconstructed update locally (step 3; Alg. 3 lines 6-8,
    P:L366-368).  Returns the replica of worker 0 (all replicas are identical)."""
    P = len(Us)
    Ug = np.concatenate([np.asarray(u, np.float64) for u in Us], axis=0)
    Vg = np.concatenate([np.asarray(v, np.float64) for v in Vs], axis=0)
    W1 = np.asarray(W, np.float64) + (-lr / P) * (Ug.T @ Vg)
    b1 = None if b is None else np.asarray(b, np.float64) + (-lr / P) * Ug.sum(axis=0)
    return W1, b1


# --------------------------------------------------------------------------
# O6 — PS simulated over the sharded flat buffer (Alg. 1 master P:L208-211,
# Alg. 3, reading Z7/Z11)
# --------------------------------------------------------------------------
def flatten_params(W: np.ndarray, b) -> np.ndarray:
    """Flat layout of a PS layer: W row-major, then bias (the buffer Alg. 1's master updates by parts,
    P:L210; reading Z11)."""
    parts = [np.asarray(W, np.float64).reshape(-1)]
    if b is not None:
        parts.append(np.asarray(b, np.float64).reshape(-1))
    return np.concatenate(parts)


def ps_step_flat(w: np.ndarray, grads: Sequence[np.ndarray], lr: float) -> np.ndarray:
    """Alg. 1's master loop (collect gradients, update the part of the parameters they
    cover, push the parameters back) on a flat buffer of n elements from P workers' flat gradients:
    each shard r is collected (summed over workers), updated by alpha = -lr/P, and pushed back
    (concatenated).  Each index must be owned by exactly one shard."""
    P = len(grads)
    n = w.shape[0]
    out = np.empty(n, dtype=np.float64)
    owned = np.zeros(n, dtype=np.int64)
    for r in range(P):
        lo, hi, _ = shard_range(n, P, r)
        s = np.zeros(hi - lo, dtype=np.float64)
        for p in range(P):
            s += np.asarray(grads[p], np.float64)[lo:hi]
        out[lo:hi] = np.asarray(w, np.float64)[lo:hi] + (-lr / P) * s
        owned[lo:hi] += 1
    if not np.all(owned == 1):
        raise AssertionError("shard map does not cover [0, n) exactly once")
    return out


def ps_simulated(W, b, Us, Vs, lr):
    """Alg. 3 lines 1-3: workers form their full gradients (G_p, gb_p) locally, "send
    them to the master node" and "synchronize" the updated layer (the sharded server of ps_step_flat)."""
    grads = [flatten_params(reconstruct(u, v), np.asarray(u, np.float64).sum(axis=0)
                            if b is not None else None) for u, v in zip(Us, Vs)]
    w1 = ps_step_flat(flatten_params(W, b), grads, lr)
    M, N = np.asarray(W).shape
    W1 = w1[:M * N].reshape(M, N)
    b1 = None if b is None else w1[M * N:]
    return W1, b1


# --------------------------------------------------------------------------
# O11 — SF-via-PS, the literal else-branch of Alg. 3 ("Send u, v
# to the master node; Synchronize A_i from the master node"; Adam-style,
# P:L335), with the master sharded by rows (reading Z20): worker r is the
# master of the output rows [lo_r, hi_r) = O2's shard_range(M, P, r).
# --------------------------------------------------------------------------
def row_shard_range(M: int, P: int, rank: int) -> Tuple[int, int]:
    """Output rows mastered by ``rank``: O2's shard map applied to the M rows (reading Z20 of the
    "master node" of P:L370-371)."""
    lo, hi, _ = shard_range(M, P, rank)
    return lo, hi


def sf_ps_simulated(W, b, Us, Vs, lr):
    """Alg. 3's else-branch: every worker p sends its sufficient factors to the masters: to master r
    the entries of its error messages for r's rows (columns [lo_r, hi_r) of
    U_p) and all of its inputs V_p.  Master r reconstructs its rows of
    sum_p U_p^T V_p, applies W[lo_r:hi_r] += (-lr/P) * (.) (and the bias rows),
    and every worker synchronises A_i from the masters (the row blocks,
    concatenated).  Each row must be mastered exactly once.

    Returns (W', b', floats) where ``floats`` counts the floats that cross
    between distinct workers (factor messages + the pushed row blocks)."""
    P = len(Us)
    W = np.asarray(W, np.float64)
    M, N = W.shape
    W1 = np.empty_like(W)
    b1 = None if b is None else np.empty(M, dtype=np.float64)
    owned = np.zeros(M, dtype=np.int64)
    floats = 0
    for r in range(P):
        lo, hi = row_shard_range(M, P, r)
        G = np.zeros((hi - lo, N), dtype=np.float64)
        gb = np.zeros(hi - lo, dtype=np.float64)
        for p in range(P):
            u = np.asarray(Us[p], np.float64)[:, lo:hi]      # message p -> r: K x (hi-lo)
            v = np.asarray(Vs[p], np.float64)                # and K x N
            if p != r:
                floats += u.size + v.size
            for k in range(u.shape[0]):                      # Eq. 5: sum of outer products
                G += np.outer(u[k], v[k])
            gb += u.sum(axis=0)
        W1[lo:hi] = W[lo:hi] + (-lr / P) * G
        if b1 is not None:
            b1[lo:hi] = np.asarray(b, np.float64)[lo:hi] + (-lr / P) * gb
        # "synchronize A_i": the updated rows (and bias entries) go to the P-1 others
        floats += (P - 1) * (hi - lo) * (N + (0 if b is None else 1))
        owned[lo:hi] += 1
    if not np.all(owned == 1):
        raise AssertionError("row shards do not cover [0, M) exactly once")
    return W1, b1, floats


# --------------------------------------------------------------------------
# O7 — one SGD step of single-worker softmax regression on the concatenated
# batch ("converges to the same objective value as a single machine")
# --------------------------------------------------------------------------
def concat_batch_sgd(W, b, X_all: np.ndarray, labels_all: np.ndarray, lr: float):
    """P:L24 ("converges to the same objective value as a single machine"): single worker, all P*K
    samples, mean CE loss: W' = W - lr dl/dW with dl/dW = sum_samples E a^T (Eq. 5) and
    E = (softmax - onehot)/(PK)."""
    W = np.asarray(W, np.float64)
    b = np.asarray(b, np.float64)
    X = np.asarray(X_all, np.float64)
    E = error_messages(W, b, X, labels_all, denom=X.shape[0])
    return W - lr * reconstruct(E, X), b - lr * E.sum(axis=0)


def worker_factors(W, b, X_all, labels_all, P: int):
    """Data parallelism (worker p computes on its own batch D_p): split the concatenated
    batch contiguously rank-major (reading Z14) and let every worker form its mean-loss factors
    U_p = (softmax-onehot)/K (E_{i+1}), V_p = X_p (a_i)."""
    X = np.asarray(X_all, np.float64)
    K = X.shape[0] // P
    Us, Vs = [], []
    for p in range(P):
        Xp = X[p * K:(p + 1) * K]
        Us.append(error_messages(np.asarray(W, np.float64), np.asarray(b, np.float64),
                                 Xp, labels_all[p * K:(p + 1) * K], denom=K))
        Vs.append(Xp)
    return Us, Vs


# --------------------------------------------------------------------------
# Error metric of reading Z13 (gate on the update, not on W')
# --------------------------------------------------------------------------
def update_error(W0, W1_test, W1_ref) -> float:
    """Reading Z13 (the north_star tolerances are stated on the update): max_i |dW_test,i - dW_ref,i|
    / max_i |dW_ref,i| with dW = W' - W0, computed in float64.  Returns 0 when the reference update is all zero and
    the test update equals it."""
    W0 = np.asarray(W0, np.float64)
    d_t = np.asarray(W1_test, np.float64) - W0
    d_r = np.asarray(W1_ref, np.float64) - W0
    denom = float(np.max(np.abs(d_r))) if d_r.size else 0.0
    num = float(np.max(np.abs(d_t - d_r))) if d_r.size else 0.0
    if denom == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / denom


def update_error_fp32(W0, W1_test, W1_ref) -> float:
    """Z13 metric for a result STORED in fp32 (reading Z13b): the deviation of
    each element beyond one fp32 ulp of the reference value W'_ref (the
    unavoidable rounding of the stored result, which is not arithmetic error
    of the update) is normalised by max |dW_ref|.  With the test updates much
    larger than one ulp of W, a wrong scale or sign still reads ~1."""
    W0 = np.asarray(W0, np.float64)
    t = np.asarray(W1_test, np.float64)
    r = np.asarray(W1_ref, np.float64)
    if r.size == 0:
        return 0.0
    ulp = np.spacing(np.abs(r).astype(np.float32)).astype(np.float64)
    dev = np.maximum(np.abs(t - r) - ulp, 0.0)
    denom = float(np.max(np.abs(r - W0)))
    num = float(np.max(dev))
    if denom == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / denom


def ulp_excuse(W0, W1_ref) -> float:
    """What update_error_fp32 forgives, relative to its normaliser: max_i ulp_fp32(W'_ref,i) /
    max_i |dW_ref,i| (reading Z13b).  A parity case is only as tight as its gate if this is well
    below the gate (the tests require <= 0.1 x gate): with |W| >> |dW| one ulp of W' is a large
    fraction of the update and the fp32 metric would pass an error of that size."""
    W0 = np.asarray(W0, np.float64)
    r = np.asarray(W1_ref, np.float64)
    if r.size == 0:
        return 0.0
    ulp = np.spacing(np.abs(r).astype(np.float32)).astype(np.float64)
    denom = float(np.max(np.abs(r - W0)))
    return math.inf if denom == 0.0 else float(np.max(ulp)) / denom


def sync_step_rows(W_rows, b_rows, Us, Vs, lr, rows):
    """O4 (Eq. 4; Eq. 5) restricted to a subset of output rows m (each row of W'
    depends only on column m of every U_p), so full-size layers can be checked one sampled row at a
    time."""
    rows = np.asarray(rows)
    P = len(Us)
    G = np.zeros((len(rows), np.asarray(Vs[0]).shape[1]), dtype=np.float64)
    gb = np.zeros(len(rows), dtype=np.float64)
    for p in range(P):
        Up = np.asarray(Us[p], np.float64)[:, rows]
        G += Up.T @ np.asarray(Vs[p], np.float64)
        gb += Up.sum(axis=0)
    W1 = np.asarray(W_rows, np.float64) - lr * (1.0 / P) * G
    b1 = None if b_rows is None else np.asarray(b_rows, np.float64) - lr * (1.0 / P) * gb
    return W1, b1


# --------------------------------------------------------------------------
# O4m — the synchronous step with Lambda = momentum + weight decay (Eq. 3 / Eq. 4
# "Lambda(A^{t-1}) contains regularization and momentums"; Alg. 3 line 8
# "A_i <- A_i + sum_j u v^T + Lambda(A_i)"; reading Z4b: applied once at the
# aggregation point; Caffe's SGD solver semantics, decay on every parameter)
# --------------------------------------------------------------------------
def sync_step_momentum(W, b, VW, Vb, Us, Vs, lr: float, mu: float, wd: float):
    """Lambda of Eq. 3 / Alg. 3 line 8 (reading Z4b): g = (1/P) sum_p G_p;
    V' = mu V + lr (g + wd W);  W' = W - V'   (same for the bias).  Returns (W', b', VW', Vb')."""
    P = len(Us)
    W = np.asarray(W, np.float64)
    G = np.zeros_like(W)
    gb = np.zeros(W.shape[0], dtype=np.float64)
    for p in range(P):
        G += reconstruct(Us[p], Vs[p])
        gb += np.asarray(Us[p], dtype=np.float64).sum(axis=0)
    G /= P
    gb /= P
    VW1 = mu * np.asarray(VW, np.float64) + lr * (G + wd * W)
    W1 = W - VW1
    if b is None:
        return W1, None, VW1, None
    b = np.asarray(b, np.float64)
    Vb1 = mu * np.asarray(Vb, np.float64) + lr * (gb + wd * b)
    return W1, b - Vb1, VW1, Vb1


def ps_step_flat_momentum(w, v, grads: Sequence[np.ndarray], lr: float, mu: float, wd: float):
    """Alg. 1's master step with Lambda = momentum/decay (reading Z4b) on a flat
    buffer: each shard owner keeps the velocity of its own shard only.  Returns (w', v')."""
    P = len(grads)
    w = np.asarray(w, np.float64)
    v = np.asarray(v, np.float64)
    w1 = np.empty_like(w)
    v1 = np.empty_like(v)
    for r in range(P):
        lo, hi, _ = shard_range(w.shape[0], P, r)
        s = np.zeros(hi - lo)
        for p in range(P):
            s += np.asarray(grads[p], np.float64)[lo:hi]
        v1[lo:hi] = mu * v[lo:hi] + lr * (s / P + wd * w[lo:hi])
        w1[lo:hi] = w[lo:hi] - v1[lo:hi]
    return w1, v1


# --------------------------------------------------------------------------
# O10 — stale synchronous parallel with staleness s ("if a worker reads from server at
# iteration t, it is guaranteed to receive all updates from all workers computed at and before
# iteration t-s-1"), read at the staleness bound (reading Z19): the parameters a
# worker's forward of iteration t uses contain exactly the updates of iterations <= t-s-1.
# --------------------------------------------------------------------------
def ssp_visible_weights(W0, b0, steps, lr: float, s: int = 1):
    """SSP at the staleness bound (reading Z19).  steps[t] = (Us, Vs): the
    sufficient factors every worker produces at iteration t (fixed
    inputs, independent of the parameters).  Returns vis with vis[t] = (W, b) the forward of
    iteration t reads, for t = 0 .. len(steps) + s (the last entries are what remains after all
    updates have been applied, i.e. after a flush)."""
    applied = [(np.asarray(W0, np.float64), None if b0 is None else np.asarray(b0, np.float64))]
    for Us, Vs in steps:                      # applied[k] = parameters after the updates of 0..k-1
        W, b = applied[-1]
        applied.append(sync_step(W, b, Us, Vs, lr))
    T = len(steps)
    return [applied[min(max(0, t - s), T)] for t in range(T + s + 1)]
