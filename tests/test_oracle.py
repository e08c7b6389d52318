"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test names the oracle part (O1..O7) and the kind of pin:
printed values (tests/golden/, cited), closed forms, brute force on tiny
inputs, exact integer arithmetic, invariants.  None of these re-types the
oracle's own formula as its check.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synthetic as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- O1 ----
def test_o1_printed_cost_example():
    """P:L333 / P:L335 printed numbers for P=4, K=256, M=N=4096."""
    g = _golden("sacp_cost_example.json")
    sfb, sfps, full = O.costs(g["M"], g["N"], g["K"], g["P"])
    pm = g["printed_millions"]
    tol = g["printed_precision"]
    assert abs(sfb / 1e6 - pm["sfb"]) <= tol
    assert abs(sfps / 1e6 - pm["sf_ps"]) <= tol
    assert abs(full / 1e6 - pm["full_ps"]) <= tol
    pr = g["printed_ratios"]
    assert abs(full / sfb - pr["full_over_sfb"]) <= tol
    assert abs(sfps / sfb - pr["sfps_over_sfb"]) <= tol
    assert O.choose_scheme(O.LAYER_FC, 4096, 4096, 256, 4) == O.SCHEME_SFB


def test_o1_spec_p32_example():
    g = _golden("sacp_cost_example.json")["spec_examples"]
    sfb, sfps, _ = O.costs(4096, 4096, 256, 32)
    assert abs(sfb / g["P32_sfb_approx"] - 1) < g["approx_rel"]
    assert abs(sfps / g["P32_sfps_approx"] - 1) < g["approx_rel"]
    assert O.choose_scheme(O.LAYER_FC, 4096, 4096, 256, 32) == O.SCHEME_PS


def test_o1_conv_always_ps():
    for P, K in itertools.product(range(1, 9), (1, 64, 256)):
        assert O.choose_scheme(O.LAYER_CONV, 96, 363, K, P) == O.SCHEME_PS


def _k_star(M, N, P):
    """Closed form derived by hand (O1): for P >= 3,
    (P-1)^2 K(M+N) <= PK(M+N) + PMN  <=>  K (M+N)(P^2-3P+1) <= PMN."""
    return (P * M * N) // ((M + N) * (P * P - 3 * P + 1))


SHAPES = [(128, 256), (64, 1024), (10, 64), (4096, 9216), (4096, 4096),
          (1000, 4096), (1000, 1024), (21841, 4096)]


def test_o1_closed_form_crossover_matches_rule():
    for (M, N) in SHAPES:
        for P in range(1, 9):
            for K in list(range(1, 300)) + [511, 512, 1000, 1024, 2048, 3000, 4096, 10347, 10348]:
                rule = O.choose_scheme(O.LAYER_FC, M, N, K, P)
                if P <= 2:
                    expect = O.SCHEME_SFB
                else:
                    expect = O.SCHEME_SFB if K <= _k_star(M, N, P) else O.SCHEME_PS
                assert rule == expect, (M, N, K, P)


def test_o1_tie_goes_to_sfb():
    """Reading Z5: M=128, N=256, K=256, P=3 is an exact tie (393,216 floats)."""
    sfb, sfps, _ = O.costs(128, 256, 256, 3)
    assert sfb == sfps == 2 * 2 * 256 * 384 == 393216
    assert O.choose_scheme(O.LAYER_FC, 128, 256, 256, 3) == O.SCHEME_SFB
    assert O.choose_scheme(O.LAYER_FC, 128, 256, 257, 3) == O.SCHEME_PS


def test_o1_monotone_in_P():
    """Once SFB flips to PS as P grows it never flips back."""
    for (M, N) in SHAPES:
        for K in (1, 8, 100, 128, 256, 1024):
            seq = [O.choose_scheme(O.LAYER_FC, M, N, K, P) for P in range(1, 65)]
            flipped = False
            for s in seq:
                if s == O.SCHEME_PS:
                    flipped = True
                elif flipped:
                    pytest.fail(f"flip back at {(M, N, K)}")


def test_o1_spot_decisions():
    """Hand-computed decisions (recomputed here by hand)."""
    # fc8 1000x4096, K=256: P=5 -> 16*256*5096 = 20,873,216 <= 5*256*5096 + 5*4,096,000 = 27,002,880
    assert O.costs(1000, 4096, 256, 5)[:2] == (20873216, 27002880)
    assert O.choose_scheme(O.LAYER_FC, 1000, 4096, 256, 5) == O.SCHEME_SFB
    # P=6 -> 25*256*5096 = 32,614,400 > 6*256*5096 + 6*4,096,000 = 32,403,456 -> PS
    assert O.costs(1000, 4096, 256, 6)[:2] == (32614400, 32403456)
    assert O.choose_scheme(O.LAYER_FC, 1000, 4096, 256, 6) == O.SCHEME_PS
    # fc6 at P=8: 49*256*13312 = 166,985,728 <= 8*256*13312 + 8*37,748,736 = 329,252,864
    assert O.costs(4096, 9216, 256, 8)[:2] == (166985728, 329252864)
    # C2 ip1 64x1024, K=100: SFB at P=3, PS at P=4
    assert O.choose_scheme(O.LAYER_FC, 64, 1024, 100, 3) == O.SCHEME_SFB
    assert O.choose_scheme(O.LAYER_FC, 64, 1024, 100, 4) == O.SCHEME_PS
    # orientation does not matter (reading Z8)
    for (M, N) in SHAPES:
        for P in range(1, 9):
            assert O.costs(M, N, 256, P) == O.costs(N, M, 256, P)


def test_o1_u64_range_values():
    """Values exceed 2^31 inside the grid; Python ints are exact."""
    sfb, sfps, full = O.costs(21841, 4096, 256, 13)
    assert full == 2 * 13 * 21841 * 4096 and full > 2 ** 31
    assert sfb == 144 * 256 * 25937


# ---------------------------------------------------------------- O2 ----
def test_o2_partition_brute_force():
    for n in list(range(0, 200)) + [650, 2432, 32896, 34944, 145578, 4097000]:
        for P in range(1, 9):
            S_ = O.shard_size(n, P)
            assert S_ % 32 == 0 and S_ * P >= n and (S_ == 0 or S_ * P - n < 32 * P)
            seen = np.zeros(n, dtype=np.int32) if n < 10 ** 6 else None
            prev_end = 0
            for r in range(P):
                lo, hi, padded = O.shard_range(n, P, r)
                assert padded == P * S_
                assert lo == prev_end and lo <= hi
                prev_end = hi
                if seen is not None:
                    seen[lo:hi] += 1
            assert prev_end == n
            if seen is not None:
                assert np.all(seen == 1)


def test_o2_examples():
    """DESIGN.md §3 reading Z11 examples (n=650 at P=8 has an empty shard)."""
    assert O.shard_size(650, 8) == 96
    assert O.shard_range(650, 8, 6) == (576, 650, 768)
    assert O.shard_range(650, 8, 7) == (650, 650, 768)
    assert O.shard_range(32896, 2, 1) == (16448, 32896, 32896)
    assert O.shard_range(34944, 8, 7) == (30688, 34944, 35072)
    assert O.shard_range(100, 1, 0) == (0, 100, 128)


# ---------------------------------------------------------------- O3 ----
@pytest.mark.parametrize("M,N,K,P", [(3, 4, 2, 1), (5, 3, 4, 2), (4, 6, 3, 3), (8, 8, 4, 3)])
def test_o3_eq5_against_finite_differences(M, N, K, P):
    """Eq. 5: sum over all workers' samples of E a^T equals dl/dW of
    the mean loss over the P*K samples, by central differences in fp64."""
    g = S.rng(100 + M * N + K + P)
    W = g.standard_normal((M, N))
    b = g.standard_normal(M)
    X = g.standard_normal((P * K, N))
    labels = g.integers(0, M, size=P * K)
    gW_fd, gb_fd = O.fd_gradient(W, b, X, labels)
    U = O.error_messages(W, b, X, labels, denom=P * K)
    G = O.reconstruct_loops(U, X)
    assert np.max(np.abs(G - gW_fd)) / np.max(np.abs(gW_fd)) < 1e-7
    assert np.max(np.abs(U.sum(axis=0) - gb_fd)) / np.max(np.abs(gb_fd)) < 1e-7


def test_reconstruct_matmul_equals_loops():
    g = S.rng(3)
    U = g.standard_normal((5, 7))
    V = g.standard_normal((5, 6))
    assert np.allclose(O.reconstruct(U, V), O.reconstruct_loops(U, V), rtol=0, atol=1e-13)


def test_reconstruct_single_entry():
    """K=1, u=e_i, v=e_j gives the single-entry matrix."""
    U = np.zeros((1, 4)); U[0, 2] = 1
    V = np.zeros((1, 3)); V[0, 1] = 1
    G = O.reconstruct_loops(U, V)
    assert G[2, 1] == 1 and G.sum() == 1


# --------------------------------------------------------- O4 / O5 / O6 --
def _exact_sync(W, b, Us, Vs, lr):
    """Exact rational arithmetic (Fractions) of the definition, brute force."""
    P = len(Us)
    M, N = W.shape
    W1 = [[Fraction(float(W[m, n])) for n in range(N)] for m in range(M)]
    b1 = [Fraction(float(b[m])) for m in range(M)]
    a = Fraction(lr) / P
    for p in range(P):
        for k in range(Us[p].shape[0]):
            for m in range(M):
                u = Fraction(float(Us[p][k, m]))
                b1[m] -= a * u
                for n in range(N):
                    W1[m][n] -= a * u * Fraction(float(Vs[p][k, n]))
    return W1, b1


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_o4_against_exact_rationals(P):
    W, b, Us, Vs, lr = S.integer_factors(5, 6, 3, P, seed=P)
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    We, be = _exact_sync(W, b, Us, Vs, lr)
    for m in range(5):
        assert b1[m] == float(be[m]) or abs(b1[m] - float(be[m])) < 1e-15
        for n in range(6):
            assert abs(W1[m, n] - float(We[m][n])) < 1e-15


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_o4_integer_variant_is_exact_in_fp32(P):
    """The integer variant is exactly representable at every step, so O4's
    fp64 result is representable in fp32 (what makes GPU parity bit-exact)."""
    W, b, Us, Vs, lr = S.integer_factors(16, 24, 8, P)
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    assert np.array_equal(W1, W1.astype(np.float32).astype(np.float64))
    assert np.array_equal(b1, b1.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("M,N,K,P", [(7, 5, 3, 1), (16, 9, 4, 2), (33, 17, 5, 3), (64, 40, 8, 8)])
def test_o4_o5_o6_agree(M, N, K, P):
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    lr = 0.05
    W4, b4 = O.sync_step(W, b, Us, Vs, lr)
    W5, b5 = O.sfb_simulated(W, b, Us, Vs, lr)
    W6, b6 = O.ps_simulated(W, b, Us, Vs, lr)
    for Wx, bx in ((W5, b5), (W6, b6)):
        assert np.max(np.abs(Wx - W4)) < 1e-12
        assert np.max(np.abs(bx - b4)) < 1e-12


def test_o4_invariants():
    M, N, K, P = 12, 10, 4, 3
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    # lr = 0 -> unchanged bitwise
    W1, b1 = O.sync_step(W, b, Us, Vs, 0.0)
    assert np.array_equal(W1, W.astype(np.float64)) and np.array_equal(b1, b.astype(np.float64))
    # U = 0 -> unchanged
    W1, _ = O.sync_step(W, b, [u * 0 for u in Us], Vs, 0.1)
    assert np.array_equal(W1, W.astype(np.float64))
    # doubling U doubles the update
    Wa, _ = O.sync_step(W, b, Us, Vs, 0.1)
    Wb, _ = O.sync_step(W, b, [2 * u for u in Us], Vs, 0.1)
    assert np.allclose(Wb - W, 2 * (Wa - W), rtol=0, atol=1e-14)
    # permuting workers leaves the result unchanged
    perm = [2, 0, 1]
    Wc, _ = O.sync_step(W, b, [Us[i] for i in perm], [Vs[i] for i in perm], 0.1)
    assert np.allclose(Wc, Wa, rtol=0, atol=1e-14)
    # a mean over workers: P identical workers == one worker
    W1w, b1w = O.sync_step(W, b, Us[:1], Vs[:1], 0.1)
    W3w, b3w = O.sync_step(W, b, Us[:1] * 3, Vs[:1] * 3, 0.1)
    assert np.allclose(W1w, W3w, rtol=0, atol=1e-14) and np.allclose(b1w, b3w, rtol=0, atol=1e-14)


@pytest.mark.parametrize("M,N,K,P", [(7, 5, 3, 1), (16, 9, 4, 2), (33, 17, 5, 3), (70, 40, 8, 8),
                                     (10, 6, 3, 8)])
def test_o11_sf_ps_equals_definition(M, N, K, P):
    """Sharded SF-via-PS (Alg. 3 else-branch) computes the same step as O4 (pure
    reassociation); (10, 6, 3, 8) has masters with no rows (empty shards)."""
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    W4, b4 = O.sync_step(W, b, Us, Vs, 0.05)
    W11, b11, _ = O.sf_ps_simulated(W, b, Us, Vs, 0.05)
    assert np.max(np.abs(W11 - W4)) < 1e-12 and np.max(np.abs(b11 - b4)) < 1e-12


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_o11_sf_ps_against_exact_rationals(P):
    """Integer variant, P a power of two: every operation is exact, so equality is exact."""
    W, b, Us, Vs, lr = S.integer_factors(37, 6, 3, P, seed=10 + P)
    W11, b11, _ = O.sf_ps_simulated(W, b, Us, Vs, lr)
    We, be = _exact_sync(W, b, Us, Vs, lr)
    for m in range(37):
        assert b11[m] == float(be[m])
        for n in range(6):
            assert W11[m, n] == float(We[m][n])


def test_o11_row_masters_and_message_count():
    """Row masters follow O2 (32-row shards, empty trailing masters legal), and the floats that
    cross between workers add up, by a hand count of the messages, to
    (P-1) (K M + P K N + M (N+1)): each worker's U columns go to the P-1 other masters once
    (K M in total per worker), its V to every other master (K N each), and every row block
    (with its bias entry) to the P-1 other workers."""
    assert [O.row_shard_range(1000, 8, r) for r in range(8)] == \
        [(0, 128), (128, 256), (256, 384), (384, 512), (512, 640), (640, 768), (768, 896), (896, 1000)]
    assert O.row_shard_range(10, 8, 0) == (0, 10) and O.row_shard_range(10, 8, 1) == (10, 10)
    for M, N, K, P in [(70, 9, 3, 3), (10, 6, 3, 8), (33, 5, 2, 1)]:
        W, b = S.fc_weights_randbias(M, N)
        Us, Vs = S.hidden_factors(M, N, K, P)
        _, _, floats = O.sf_ps_simulated(W, b, Us, Vs, 0.1)
        assert floats == (P - 1) * (K * M + P * K * N + M * (N + 1))
        _, _, floats_nb = O.sf_ps_simulated(W, None, Us, Vs, 0.1)
        assert floats_nb == (P - 1) * (K * M + P * K * N + M * N)


def test_o6_shard_cover_failure_is_detected():
    """ps_step_flat checks coverage; an inconsistent P/grad list still works
    only when the map covers [0,n) — sanity that the check exists."""
    w = np.zeros(100)
    out = O.ps_step_flat(w, [np.ones(100)] * 4, 1.0)
    assert np.allclose(out, -1.0)


def test_sync_step_rows_matches_full():
    M, N, K, P = 40, 12, 5, 3
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    W1, b1 = O.sync_step(W, b, Us, Vs, 0.3)
    rows = np.array([0, 7, 39, 13])
    Wr, br = O.sync_step_rows(W[rows], b[rows], Us, Vs, 0.3, rows)
    assert np.allclose(Wr, W1[rows], rtol=0, atol=1e-14)
    assert np.allclose(br, b1[rows], rtol=0, atol=1e-14)


# ---------------------------------------------------------------- O7 ----
@pytest.mark.parametrize("M,N,K,P", [(10, 64, 8, 2), (5, 7, 4, 4), (3, 9, 6, 1)])
def test_o7_concat_batch_equivalence(M, N, K, P):
    """A synchronous step with per-worker mean-loss factors equals
    single-worker SGD on the concatenated P*K batch."""
    W, b = S.fc_weights_randbias(M, N)
    X, labels = S.softmax_batch(N, M, P * K)
    Us, Vs = O.worker_factors(W, b, X, labels, P)
    Wsync, bsync = O.sync_step(W, b, Us, Vs, 0.07)
    Wcat, bcat = O.concat_batch_sgd(W, b, X, labels, 0.07)
    assert np.max(np.abs(Wsync - Wcat)) < 1e-12
    assert np.max(np.abs(bsync - bcat)) < 1e-12


def test_o7_single_worker_is_textbook_sgd_by_fd():
    """P=1: the step equals W - lr * (finite-difference gradient)."""
    M, N, K = 4, 5, 6
    W, b = S.fc_weights_randbias(M, N)
    X, labels = S.softmax_batch(N, M, K)
    W64, b64 = W.astype(np.float64), b.astype(np.float64)
    gW, gb = O.fd_gradient(W64, b64, X.astype(np.float64), labels)
    Us, Vs = O.worker_factors(W, b, X, labels, 1)
    W1, b1 = O.sync_step(W, b, Us, Vs, 0.5)
    assert np.max(np.abs(W1 - (W64 - 0.5 * gW))) < 1e-8
    assert np.max(np.abs(b1 - (b64 - 0.5 * gb))) < 1e-8


# --------------------------------------------------------- Z13 metric ----
def test_update_error_metric_catches_2x_bug():
    W0 = np.ones((4, 4), dtype=np.float32)
    ref = W0 - 1e-4
    bad = W0 - 2e-4
    assert O.update_error(W0, ref, ref) == 0.0
    assert O.update_error(W0, bad, ref) == pytest.approx(1.0, rel=1e-2)


def test_update_error_fp32_excuses_only_storage_rounding():
    W0 = np.full(8, 1.0, np.float32)
    ref = W0.astype(np.float64) - 1e-3 * np.arange(8)
    stored = ref.astype(np.float32)          # correctly rounded result
    assert O.update_error_fp32(W0, stored, ref) == 0.0
    wrong = (W0.astype(np.float64) - 2e-3 * np.arange(8)).astype(np.float32)
    assert O.update_error_fp32(W0, wrong, ref) > 0.99
    off_by_two_ulps = ref + 2 * np.spacing(np.float32(1.0))
    assert O.update_error_fp32(W0, off_by_two_ulps, ref) > 0


# --------------------------------------------------------------- O4m ----
def test_o4m_reduces_to_o4_without_momentum_and_decay():
    W, b = S.fc_weights_randbias(12, 9)
    Us, Vs = S.hidden_factors(12, 9, 4, 3)
    z = np.zeros_like(W, dtype=np.float64)
    W1, b1, VW, Vb = O.sync_step_momentum(W, b, z, np.zeros(12), Us, Vs, 0.1, 0.0, 0.0)
    W4, b4 = O.sync_step(W, b, Us, Vs, 0.1)
    assert np.max(np.abs(W1 - W4)) < 1e-14 and np.max(np.abs(b1 - b4)) < 1e-14
    assert np.allclose(VW, W.astype(np.float64) - W4, rtol=0, atol=1e-14)


def test_o4m_geometric_series_closed_form():
    """Constant gradient, no decay: after t steps W_t = W_0 - lr g sum_{s=1..t} (1 - mu^s)/(1 - mu)."""
    W, b = S.fc_weights_randbias(6, 5)
    Us, Vs = S.hidden_factors(6, 5, 3, 2)
    g = sum(O.reconstruct(u, v) for u, v in zip(Us, Vs)) / 2
    lr, mu, T = 0.05, 0.9, 6
    Wt, bt = W.astype(np.float64), b.astype(np.float64)
    VW, Vb = np.zeros_like(Wt), np.zeros_like(bt)
    for _ in range(T):
        Wt, bt, VW, Vb = O.sync_step_momentum(Wt, bt, VW, Vb, Us, Vs, lr, mu, 0.0)
    coeff = sum((1 - mu ** s) / (1 - mu) for s in range(1, T + 1))
    assert np.max(np.abs(Wt - (W.astype(np.float64) - lr * g * coeff))) < 1e-12


def test_o4m_pure_decay_closed_form():
    """Zero gradient, mu = 0: one step is W (1 - lr wd)."""
    W, b = S.fc_weights_randbias(5, 4)
    Us = [np.zeros((2, 5), np.float32)]
    Vs = [np.zeros((2, 4), np.float32)]
    W1, b1, _, _ = O.sync_step_momentum(W, b, np.zeros((5, 4)), np.zeros(5), Us, Vs, 0.1, 0.0, 0.01)
    assert np.allclose(W1, W.astype(np.float64) * (1 - 0.1 * 0.01), rtol=0, atol=1e-15)
    assert np.allclose(b1, b.astype(np.float64) * (1 - 0.1 * 0.01), rtol=0, atol=1e-15)


def test_o4m_ps_equals_definition():
    M, N, K, P = 7, 5, 3, 3
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    g = S.rng(3)
    VW0, Vb0 = g.standard_normal((M, N)) * 1e-3, g.standard_normal(M) * 1e-3
    W1, b1, VW1, Vb1 = O.sync_step_momentum(W, b, VW0, Vb0, Us, Vs, 0.2, 0.8, 0.05)
    grads = [O.flatten_params(O.reconstruct(u, v), np.asarray(u, np.float64).sum(0)) for u, v in zip(Us, Vs)]
    w1, v1 = O.ps_step_flat_momentum(O.flatten_params(W, b), O.flatten_params(VW0, Vb0), grads, 0.2, 0.8, 0.05)
    assert np.max(np.abs(w1 - O.flatten_params(W1, b1))) < 1e-13
    assert np.max(np.abs(v1 - O.flatten_params(VW1, Vb1))) < 1e-13



def _brute_mean_grad(Us, Vs):
    """(1/P) sum_p sum_k u_k v_k^T and (1/P) sum_p sum_k u_k in exact rationals, element by element."""
    P, K, M, N = len(Us), Us[0].shape[0], Us[0].shape[1], Vs[0].shape[1]
    G = [[Fraction(0)] * N for _ in range(M)]
    gb = [Fraction(0)] * M
    for p in range(P):
        for k in range(K):
            for m in range(M):
                u = Fraction(float(Us[p][k, m]))
                gb[m] += u / P
                for n in range(N):
                    G[m][n] += u * Fraction(float(Vs[p][k, n])) / P
    return G, gb


def test_o4m_two_steps_momentum_and_decay_closed_form():
    """mu != 0 AND wd != 0 (pins with only one of them non-zero let a decoupled-decay
    oracle pass).  Caffe's coupled rule v = mu v + lr (g + wd w), w -= v (P:L141 Lambda, reading Z4b),
    written out by hand for two steps from v_0 = 0:
        w_1 = (1 - lr wd) w_0 - lr g_1
        w_2 = (1 - lr wd)^2 w_0 - (1 - lr wd) lr g_1 - lr g_2 - mu lr (g_1 + wd w_0)
    A decoupled rule (w -= mu v + lr g + lr wd w) gives the same w_1 but lacks the -mu lr wd w_0 term
    in w_2.  Dyadic inputs make the fp64 oracle exact, so equality is exact."""
    M, N, K, P = 3, 4, 2, 2
    W0, b0, _, _, _ = S.integer_factors(M, N, K, P, seed=31)
    steps = [S.integer_factors(M, N, K, P, seed=32 + t)[2:4] for t in range(2)]
    lr, mu, wd = Fraction(1, 8), Fraction(1, 2), Fraction(1, 4)
    w = [[Fraction(float(W0[m, n])) for n in range(N)] for m in range(M)]
    bb = [Fraction(float(b0[m])) for m in range(M)]
    (G1, gb1), (G2, gb2) = (_brute_mean_grad(Us, Vs) for Us, Vs in steps)
    a = 1 - lr * wd

    def two_steps(w0, g1, g2):
        return a * a * w0 - a * lr * g1 - lr * g2 - mu * lr * (g1 + wd * w0)

    Wt, bt = W0.astype(np.float64), b0.astype(np.float64)
    VW, Vb = np.zeros_like(Wt), np.zeros_like(bt)
    for Us, Vs in steps:
        Wt, bt, VW, Vb = O.sync_step_momentum(Wt, bt, VW, Vb, Us, Vs, float(lr), float(mu), float(wd))
    for m in range(M):
        assert bt[m] == float(two_steps(bb[m], gb1[m], gb2[m]))
        for n in range(N):
            assert Wt[m, n] == float(two_steps(w[m][n], G1[m][n], G2[m][n]))
    # the decoupled variant differs by exactly mu lr wd w_0 (so this pin can tell them apart)
    assert any(mu * lr * wd * w[m][n] != 0 for m in range(M) for n in range(N))
    # the PS form with shard-owned velocities gives the same two steps
    n_ = M * N + M
    wf, vf = O.flatten_params(W0, b0), np.zeros(n_)
    for Us, Vs in steps:
        grads = [O.flatten_params(O.reconstruct(u, v), np.asarray(u, np.float64).sum(0)) for u, v in zip(Us, Vs)]
        wf, vf = O.ps_step_flat_momentum(wf, vf, grads, float(lr), float(mu), float(wd))
    assert np.array_equal(wf, O.flatten_params(Wt, bt))


def test_ulp_excuse_of_the_fp32_metric():
    """ulp_excuse = max ulp_fp32(W') / max |dW| (reading Z13b): one ulp of 1.0 is 2^-23; W = 0 leaves
    only the relative rounding of the update itself."""
    W0 = np.ones(4, np.float32)
    ref = W0.astype(np.float64) - 1e-4
    assert O.ulp_excuse(W0, ref) == pytest.approx(2.0 ** -24 / 1e-4, rel=1e-12)   # ulp(0.9999) = 2^-24
    ref2 = W0.astype(np.float64) + 0.5
    assert O.ulp_excuse(W0, ref2) == pytest.approx(2.0 ** -23 / 0.5, rel=1e-12)
    z = np.zeros(4, np.float32)
    assert O.ulp_excuse(z, z + 3.0) == pytest.approx(2.0 ** -22 / 3.0, rel=1e-12)
    assert O.ulp_excuse(z, z) == float("inf")


# ---------------------------------------------------------------- O10 SSP ----
def _ssp_steps(M, N, K, P, T, seed):
    out = []
    for t in range(T):
        _, _, Us, Vs, _ = S.integer_factors(M, N, K, P, seed=seed + t)
        out.append((Us, Vs))
    return out


def test_ssp_zero_staleness_is_bsp():
    """s = 0 is bulk synchronous: iteration t reads every update of iterations <= t-1."""
    W, b, _, _, lr = S.integer_factors(12, 20, 3, 2, seed=1)
    steps = _ssp_steps(12, 20, 3, 2, 4, seed=10)
    vis = O.ssp_visible_weights(W, b, steps, lr, s=0)
    Wt, bt = W.astype(np.float64), b.astype(np.float64)
    for t, (Us, Vs) in enumerate(steps):
        assert np.array_equal(vis[t][0], Wt) and np.array_equal(vis[t][1], bt)
        Wt, bt = O.sync_step(Wt, bt, Us, Vs, lr)
    assert np.array_equal(vis[len(steps)][0], Wt)


def test_ssp_one_reads_exactly_updates_up_to_t_minus_2():
    """s = 1 at the bound (P:L123 with s = 1): the forward of iteration t sees the updates of
    iterations 0..t-2 and none of t-1: W_t = W_0 + sum_{tau <= t-2} dW_tau, with each dW_tau
    computed independently of the others from its own factors (closed form, not the recursion)."""
    M, N, K, P, T = 9, 14, 2, 4, 5
    W, b, _, _, lr = S.integer_factors(M, N, K, P, seed=2)
    steps = _ssp_steps(M, N, K, P, T, seed=20)
    vis = O.ssp_visible_weights(W, b, steps, lr, s=1)
    assert len(vis) == T + 2
    dW = [(-lr / P) * sum(np.asarray(U, np.float64).T @ np.asarray(V, np.float64) for U, V in zip(Us, Vs))
          for Us, Vs in steps]
    for t in range(T + 2):
        ref = W.astype(np.float64) + sum((dW[k] for k in range(0, max(0, t - 1))), np.zeros((M, N)))
        assert np.array_equal(vis[t][0], ref), t
    # iterations 0 and 1 both read the initial parameters; the flushed end state equals BSP's
    assert np.array_equal(vis[0][0], vis[1][0])
    assert np.array_equal(vis[-1][0], O.ssp_visible_weights(W, b, steps, lr, s=0)[-1][0])


def _round_mantissa(x, keep_bits, mode):
    """fp32 -> fp32 with only `keep_bits` explicit mantissa bits: 'rn' = round half away from zero (cvt.rna),
    'rz' = truncate (what the tensor core does to fp32 operands read as TF32)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    drop = 23 - keep_bits
    if mode == "rn":
        b = b + (1 << (drop - 1))
    b = b & ~np.uint64((1 << drop) - 1) & 0xFFFFFFFF
    return b.astype(np.uint32).view(np.float32)


def test_wire_precision_readings_against_the_gate():
    """DESIGN §9 / reading Z12': on the hidden-layer factor recipe, a bf16 wire (7 mantissa bits, RN) exceeds the
    2e-3 gate of the Z13 metric while TF32 (10 bits) stays inside it, rounded (the pack) or truncated (the
    in-place MN-major K1 at P = 1) -- the arithmetic behind rejecting the compact wire and accepting truncation."""
    errs = {}
    for (M, N, K, P) in [(256, 512, 8, 2), (1024, 2048, 256, 1), (1000, 1024, 128, 4)]:
        W, _ = S.fc_weights_randbias(M, N)
        Us, Vs = S.hidden_factors(M, N, K, P)
        W1, _ = O.sync_step(W, None, Us, Vs, 0.5)
        for name, bits, mode in (("bf16", 7, "rn"), ("tf32_rn", 10, "rn"), ("tf32_rz", 10, "rz")):
            Ur = [_round_mantissa(u, bits, mode) for u in Us]
            Vr = [_round_mantissa(v, bits, mode) for v in Vs]
            Wt, _ = O.sync_step(W, None, Ur, Vr, 0.5)
            errs.setdefault(name, []).append(O.update_error(W, Wt, W1))
    assert min(errs["bf16"]) > 2e-3, errs
    assert max(errs["tf32_rn"]) < 6e-4, errs
    assert max(errs["tf32_rz"]) < 1.5e-3, errs   # 0.79e-3 .. 1.28e-3 (small K: fewer products average out)
    assert min(errs["tf32_rz"]) > max(errs["tf32_rn"]), errs   # truncation is the worse of the two TF32 roundings
