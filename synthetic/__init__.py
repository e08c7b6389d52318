"""Seeded synthetic inputs shared by the tests, the oracle and bench.py.

This module holds NO arithmetic of the method (no reconstruction, no update,
no cost rule): it only draws random numbers with the shapes and value
distributions of the paper's workloads (recipe in DESIGN.md §4).  It is the
one module both the CUDA path's callers and the oracle may use.

All arrays are float32 (the exact values the GPU sees); the oracle widens them
to float64 itself.
"""
from __future__ import annotations

import math
from typing import List, Tuple

import numpy as np

WEIGHT_SEED = 6216          # identical weights on every rank
DATA_SEED_BASE = 1512       # + rank


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def fc_weights(M: int, N: int, seed: int = WEIGHT_SEED, with_bias: bool = True):
    """W ~ U(-r, r), r = sqrt(6 / (fan_in + fan_out)) (Xavier); b = 0."""
    g = rng(seed)
    r = math.sqrt(6.0 / (M + N))
    W = g.uniform(-r, r, size=(M, N)).astype(np.float32)
    b = np.zeros(M, dtype=np.float32) if with_bias else None
    return W, b


def fc_weights_randbias(M: int, N: int, seed: int = WEIGHT_SEED):
    """Like fc_weights but with a non-zero bias, so bias updates are visible."""
    g = rng(seed)
    r = math.sqrt(6.0 / (M + N))
    W = g.uniform(-r, r, size=(M, N)).astype(np.float32)
    b = g.uniform(-r, r, size=(M,)).astype(np.float32)
    return W, b


def hidden_factors(M: int, N: int, K: int, P: int, seed: int = DATA_SEED_BASE
                   ) -> Tuple[List[np.ndarray], List[np.ndarray]]:
    """Per-worker sufficient factors of a hidden FC layer: U_p ~ N(0,1)/K
    (error messages of a mean loss), V_p = max(0, N(0,1)) (post-ReLU inputs,
    ~50% zeros).  Worker p uses seed + p."""
    Us, Vs = [], []
    for p in range(P):
        g = rng(seed + p)
        Us.append((g.standard_normal((K, M)) / K).astype(np.float32))
        Vs.append(np.maximum(g.standard_normal((K, N)), 0.0).astype(np.float32))
    return Us, Vs


def integer_factors(M: int, N: int, K: int, P: int, seed: int = 7):
    """Integer variant: U in {-3..3}, V in {0..3},
    W = k * 2^-10 with |k| < 2^10, b likewise, lr = 2^-7.  Every path
    (fp32 SIMT, TF32 tensor core, NCCL sums) is exact on these when
    P*K*9 < 2^24 and P is a power of two."""
    g = rng(seed)
    Us = [g.integers(-3, 4, size=(K, M)).astype(np.float32) for _ in range(P)]
    Vs = [g.integers(0, 4, size=(K, N)).astype(np.float32) for _ in range(P)]
    W = (g.integers(-1023, 1024, size=(M, N)) * 2.0 ** -10).astype(np.float32)
    b = (g.integers(-1023, 1024, size=(M,)) * 2.0 ** -10).astype(np.float32)
    return W, b, Us, Vs, 2.0 ** -7


def integer_grads(n: int, P: int, seed: int = 11):
    """Integer-valued flat gradients for the PS path (|g| <= 64)."""
    g = rng(seed)
    return [g.integers(-64, 65, size=(n,)).astype(np.float32) for _ in range(P)]


def dense_grads(n: int, P: int, seed: int = 13, scale: float = 1e-2):
    """Random flat gradients for the PS path: N(0, scale^2)."""
    out = []
    for p in range(P):
        g = rng(seed + p)
        out.append((g.standard_normal(n) * scale).astype(np.float32))
    return out


def softmax_batch(N: int, n_classes: int, n_samples: int, seed: int = DATA_SEED_BASE):
    """Inputs and labels for the softmax-regression pins: x ~ U[0,1)^N,
    labels uniform over classes."""
    g = rng(seed)
    X = g.random((n_samples, N)).astype(np.float32)
    labels = g.integers(0, n_classes, size=(n_samples,))
    return X, labels


def images(batch: int, channels: int, hw: int, seed: int):
    """Synthetic images U[0,1) and uniform labels."""
    g = rng(seed)
    x = g.random((batch, channels, hw, hw), dtype=np.float32)
    return x
