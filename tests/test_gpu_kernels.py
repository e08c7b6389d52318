"""GPU parity of the hot-path kernels against the fp64 oracle (all through the
C ABI).  Tolerances (BASELINE.json north_star, metric of reading Z13):
  * integer variant: bit-exact on every path;
  * fp32 CUDA-core paths (K1r, K2): max-normalised update error <= 1e-5;
  * TF32 tensor-core path (K1): <= 2e-3.
"""
import numpy as np
import pytest

import oracle as O
import synthetic as S
from parity import check_update, w0_like

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-5
TOL_TF32 = 2e-3


@pytest.fixture(scope="module")
def pz():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1512_06216_b200 as pz
    return pz


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ K2 ----
@pytest.mark.parametrize("count", [1, 3, 4, 5, 31, 1023, 1027, 4096, 65536 + 7, 1_000_003])
def test_k2_integer_bit_exact(pz, count):
    g = S.rng(count)
    W = (g.integers(-1023, 1024, size=count) * 2.0 ** -10).astype(np.float32)
    gr = g.integers(-64, 65, size=count).astype(np.float32)
    alpha = -(2.0 ** -7)
    Wd, gd = dev(W), dev(gr)
    pz.ps_shard_update(gd, Wd, count, alpha)
    ref = W.astype(np.float64) + alpha * gr.astype(np.float64)
    assert np.array_equal(host(Wd).astype(np.float64), ref)


def test_k2_unaligned_and_random(pz):
    n = 100_001
    gr = S.dense_grads(n + 1, 1, seed=6)[0]
    W = w0_like(S.dense_grads(n + 1, 1, seed=5, scale=1.0)[0], 0.01 * gr)
    Wd, gd = dev(W), dev(gr)
    # offset by one float -> not 16-byte aligned -> scalar path
    pz.ps_shard_update(gd[1:], Wd[1:], n, -0.01)
    out = host(Wd)
    ref = W.astype(np.float64)
    ref[1:] += -0.01 * gr[1:].astype(np.float64)
    assert out[0] == W[0]
    check_update(W, out, ref, TOL_FP32)


def test_k2_stats_warp_reduction(pz):
    n = 50_000
    gr = S.dense_grads(n, 1, seed=9)[0]
    gr[123] = np.inf
    gr[40000] = np.nan
    W = np.zeros(n, np.float32)
    st = torch.zeros(2, device="cuda")
    pz.ps_shard_update(dev(gr), dev(W), n, 0.5, stats=st)
    s = host(st)
    fin = np.isfinite(gr)
    assert s[1] == 2.0
    # sum of squares over the finite updates is reported only when all are finite; check separately
    st2 = torch.zeros(2, device="cuda")
    gr2 = np.where(fin, gr, 0).astype(np.float32)
    pz.ps_shard_update(dev(gr2), dev(W), n, 0.5, stats=st2)
    s2 = host(st2)
    ref = float(np.sum((0.5 * gr2.astype(np.float64)) ** 2))
    assert s2[1] == 0.0 and abs(s2[0] - ref) / ref < 1e-5


def test_k2_zero_count_is_noop(pz):
    W = dev(np.ones(8, np.float32))
    pz.ps_shard_update(W, W, 0, 1.0)
    assert np.all(host(W) == 1.0)


# --------------------------------------------------------- PS simulated ----
@pytest.mark.parametrize("n,P", [(650, 8), (2432, 8), (34944, 8), (145578, 3), (32896, 2), (100, 1), (37, 4)])
def test_ps_simulated_integer_bit_exact(pz, n, P):
    _, _, padded = O.shard_range(n, P, 0)
    g = S.rng(n + P)
    W = (g.integers(-1023, 1024, size=padded) * 2.0 ** -10).astype(np.float32)
    grads = np.zeros((P, padded), np.float32)
    for p, gp in enumerate(S.integer_grads(n, P, seed=n)):
        grads[p, :n] = gp
    lr = 2.0 ** -7 * (P if P in (1, 2, 4, 8) else 1)
    Wd = dev(W)
    pz.ps_simulated(dev(grads), P, Wd, n, lr)
    out = host(Wd)
    ref = O.ps_step_flat(W[:n], [grads[p, :n] for p in range(P)], lr)
    if P in (1, 2, 4, 8):
        assert np.array_equal(out[:n].astype(np.float64), ref)
    else:
        check_update(W[:n], out[:n], ref, TOL_FP32)
    assert np.array_equal(out[n:], W[n:])  # padding untouched


def test_ps_simulated_random(pz):
    n, P = 1_000_000, 8
    _, _, padded = O.shard_range(n, P, 0)
    grads = np.zeros((P, padded), np.float32)
    for p, gp in enumerate(S.dense_grads(n, P, seed=2)):
        grads[p, :n] = gp
    W = np.zeros(padded, np.float32)
    W[:n] = w0_like(S.dense_grads(n, 1, seed=1, scale=0.05)[0], 0.01 / P * grads[:, :n].sum(0, dtype=np.float64))
    Wd = dev(W)
    pz.ps_simulated(dev(grads), P, Wd, n, 0.01)
    out = host(Wd)
    ref = O.ps_step_flat(W[:n], [grads[p, :n] for p in range(P)], 0.01)
    check_update(W[:n], out[:n], ref, TOL_FP32)


# -------------------------------------------------------- SFB simulated ----
SFB_CASES = [
    # (M, N, K, P)   C1; ragged tiles; C2 ip2 (M not /4, N < 256); odd everything; tiny
    (128, 256, 8, 2),
    (1000, 1024, 16, 3),
    (10, 64, 100, 2),
    (333, 260, 7, 3),
    (1, 4, 1, 1),
    (130, 516, 33, 2),
    (640, 4096, 32, 4),
]


@pytest.mark.parametrize("recon", ["fp32", "tf32"])
@pytest.mark.parametrize("M,N,K,P", SFB_CASES)
def test_sfb_simulated_vs_oracle(pz, recon, M, N, K, P):
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    lr = 0.5
    Wd, bd = dev(W), dev(b)
    pz.sfb_simulated(dev(np.concatenate(Us)), dev(np.concatenate(Vs)), P, K, M, N, Wd, bd, lr,
                     recon=pz.RECON_FP32 if recon == "fp32" else pz.RECON_TF32)
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    tol = TOL_FP32 if recon == "fp32" else TOL_TF32
    check_update(W, host(Wd), W1, tol)
    # the bias uses the unrounded fp32 column sums on both paths
    check_update(b, host(bd), b1, TOL_FP32)


@pytest.mark.parametrize("recon", ["fp32", "tf32"])
@pytest.mark.parametrize("M,N,K,P", [(128, 256, 8, 2), (1000, 1024, 64, 4), (10, 64, 100, 2),
                                     (300, 520, 40, 8), (256, 512, 256, 8)])
def test_sfb_integer_bit_exact(pz, recon, M, N, K, P):
    W, b, Us, Vs, lr = S.integer_factors(M, N, K, P, seed=M + N)
    Wd, bd = dev(W), dev(b)
    pz.sfb_simulated(dev(np.concatenate(Us)), dev(np.concatenate(Vs)), P, K, M, N, Wd, bd, lr,
                     recon=pz.RECON_FP32 if recon == "fp32" else pz.RECON_TF32)
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    assert np.array_equal(host(Wd).astype(np.float64), W1)
    assert np.array_equal(host(bd).astype(np.float64), b1)


def test_sfb_sfb_equals_ps_on_same_layer(pz):
    """Cross-path check (SURVEY 8(c) K2 numerics): SFB (TF32) and PS (fp32)
    land within the TF32 gate of each other; PS within 1e-5 of the oracle."""
    M, N, K, P = 256, 384, 32, 4
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    lr = 0.3
    Wd = dev(W)
    pz.sfb_simulated(dev(np.concatenate(Us)), dev(np.concatenate(Vs)), P, K, M, N, Wd, None, lr)
    n = M * N
    _, _, padded = O.shard_range(n, P, 0)
    grads = np.zeros((P, padded), np.float32)
    for p in range(P):
        grads[p, :n] = (Us[p].astype(np.float64).T @ Vs[p].astype(np.float64)).astype(np.float32).reshape(-1)
    Wps = np.zeros(padded, np.float32)
    Wps[:n] = W.reshape(-1)
    Wpsd = dev(Wps)
    pz.ps_simulated(dev(grads), P, Wpsd, n, lr)
    W1, _ = O.sync_step(W, None, Us, Vs, lr)
    sfb_out = host(Wd)
    ps_out = host(Wpsd)[:n].reshape(M, N)
    check_update(W, sfb_out, W1, TOL_TF32)
    check_update(W, ps_out, W1, TOL_FP32)
    check_update(W, sfb_out, ps_out, TOL_TF32)


def test_reconstruct_zero_rows_noop(pz):
    W = dev(np.ones((8, 8), np.float32))
    U = dev(np.ones((8, 8), np.float32))
    pz.reconstruct_sgd(U, U, 1, 0, 8, 8, 8, W, 1.0)
    assert np.all(host(W) == 1.0)
    pz.reconstruct_sgd(U, U, 1, 0, 8, 8, 8, W, 1.0, recon=pz.RECON_FP32)
    assert np.all(host(W) == 1.0)


@pytest.mark.parametrize("recon", ["fp32", "tf32"])
def test_reconstruct_sgd_gather_layout(pz, recon):
    """K1/K1r on buffers already in the gather layout ([P][M][ldk], ldk > K)."""
    M, N, K, P, ldk = 200, 300, 6, 3, 8
    g = S.rng(77)
    U = np.zeros((P, M, ldk), np.float32)
    V = np.zeros((P, N, ldk), np.float32)
    U[:, :, :K] = g.integers(-3, 4, size=(P, M, K))
    V[:, :, :K] = g.integers(0, 4, size=(P, N, K))
    W = (g.integers(-1023, 1024, size=(M, N)) * 2.0 ** -10).astype(np.float32)
    Wd = dev(W)
    pz.reconstruct_sgd(dev(U), dev(V), P, K, ldk, M, N, Wd, -(2.0 ** -9),
                       recon=pz.RECON_FP32 if recon == "fp32" else pz.RECON_TF32)
    ref = W.astype(np.float64) - 2.0 ** -9 * np.einsum("pmk,pnk->mn", U.astype(np.float64), V.astype(np.float64))
    assert np.array_equal(host(Wd).astype(np.float64), ref)


@pytest.mark.parametrize("recon", ["fp32", "tf32"])
@pytest.mark.parametrize("m0,m1", [(0, 200), (0, 96), (96, 200), (33, 161), (199, 200), (50, 50)])
def test_reconstruct_sgd_rows_master_block(pz, recon, m0, m1):
    """SF-PS master (reading Z20): K1/K1r on rows [m0, m1) of the gather buffer, integer variant bit-exact
    vs the oracle's O4 rows; every other row untouched.  (33, 161) spans tiles with a ragged start,
    (199, 200) is a one-row block, (50, 50) an empty master."""
    M, N, K, P, ldk = 200, 300, 6, 4, 8
    g = S.rng(78)
    U = np.zeros((P, M, ldk), np.float32)
    V = np.zeros((P, N, ldk), np.float32)
    U[:, :, :K] = g.integers(-3, 4, size=(P, M, K))
    V[:, :, :K] = g.integers(0, 4, size=(P, N, K))
    W = (g.integers(-1023, 1024, size=(M, N)) * 2.0 ** -10).astype(np.float32)
    lr = 2.0 ** -7
    Wd = dev(W)
    pz.reconstruct_sgd_rows(dev(U), dev(V), P, K, ldk, M, m0, m1, N, Wd, -lr / P,
                            recon=pz.RECON_FP32 if recon == "fp32" else pz.RECON_TF32)
    Us = [U[p, :, :K].T.copy() for p in range(P)]
    Vs = [V[p, :, :K].T.copy() for p in range(P)]
    W1, _ = O.sync_step(W, None, Us, Vs, lr)
    ref = W.astype(np.float64)
    ref[m0:m1] = W1[m0:m1]
    assert np.array_equal(host(Wd).astype(np.float64), ref)


# ------------------------------------------- full size, sampled rows ----
def _sampled_rows(M, n=48, seed=0):
    g = S.rng(seed)
    rows = np.unique(np.concatenate([[0, M - 1, M // 2, 127, 128], g.integers(0, M, size=n)]))
    return rows[rows < M]


@pytest.mark.parametrize("M,N,K,P", [(4096, 9216, 256, 8),     # C3 fc6 at P=8 (bench launch shape x8 rows)
                                     (4096, 9216, 256, 1),     # C3 fc6 at P=1 (bench N=1 launch)
                                     (21841, 4096, 256, 2),    # C5 softmax FC (M not a multiple of 4)
                                     (21841, 4096, 32, 8),     # C5 sweep: smallest K, P = 8 simulated workers
                                     (21841, 4096, 2048, 4)])  # C5 sweep: largest K (P*K = 8192)
def test_sfb_full_size_sampled_rows(pz, M, N, K, P):
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    lr = 0.5
    Wd, bd = dev(W), dev(b)
    pz.sfb_simulated(dev(np.concatenate(Us)), dev(np.concatenate(Vs)), P, K, M, N, Wd, bd, lr)
    out, outb = host(Wd), host(bd)
    rows = _sampled_rows(M)
    W1r, b1r = O.sync_step_rows(W[rows], b[rows], Us, Vs, lr, rows)
    check_update(W[rows], out[rows], W1r, TOL_TF32)
    check_update(b[rows], outb[rows], b1r, TOL_FP32)
    # property at any size: rows never sampled still moved only where factors are non-zero
    assert np.all(np.isfinite(out))


# ------------------------------------------------------------------ K3 ----
def _tf32_rna(a):
    """TF32 round-to-nearest, ties away from zero (cvt.rna): keep 10 mantissa bits, in sign-magnitude."""
    b = np.ascontiguousarray(a, np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def _tf32_bits(a):
    return (np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("M,N,K", [(4096, 9216, 256), (1000, 4096, 256), (10, 64, 100), (333, 260, 7),
                                   (21841, 4096, 2048), (5, 3, 513), (128, 256, 8)])
@pytest.mark.parametrize("round_tf32", [False, True])
def test_k3_pack_exact(pz, M, N, K, round_tf32):
    """K3: the packed slot is the exact transpose (and the exact TF32 RNA rounding of it), columns
    [K, ldk) untouched, U's column sums within fp32 summation error of the fp64 sums (any order), one
    launch for U and V; cluster split of K (cs = min(8, ceil(K/64))) covers K = 7 ... 2048."""
    ldk = (K + 3) // 4 * 4 + 4
    g = S.rng(M + K)
    U = (g.standard_normal((K, M)) / K).astype(np.float32)
    V = np.maximum(g.standard_normal((K, N)), 0).astype(np.float32)
    ud = torch.full((M, ldk), 7.0, device="cuda")
    vd = torch.full((N, ldk), 7.0, device="cuda")
    cs = torch.zeros(M, device="cuda")
    pz.pack_factors(dev(U), dev(V), K, ldk, ud, vd, cs, round_tf32=round_tf32)
    uo, vo, co = host(ud), host(vd), host(cs)
    rnd = _tf32_rna if round_tf32 else (lambda a: a)
    # (TF32 values are compared on their 19 significant bits: the tensor core reads no others)
    keep = _tf32_bits if round_tf32 else (lambda a: a)
    assert np.array_equal(keep(uo[:, :K]), rnd(U.T))
    assert np.array_equal(keep(vo[:, :K]), rnd(V.T))
    assert np.all(uo[:, K:] == 7.0) and np.all(vo[:, K:] == 7.0)
    ref = U.astype(np.float64).sum(0)
    bound = K * np.finfo(np.float32).eps * np.abs(U).astype(np.float64).sum(0) + 1e-30
    assert np.all(np.abs(co - ref) <= bound)


def test_k3_pack_deterministic_and_u_only(pz):
    K, M = 1024, 3000
    U = dev(S.rng(5).standard_normal((K, M)).astype(np.float32))
    outs = []
    for _ in range(3):
        ud = torch.zeros(M, K, device="cuda")
        cs = torch.zeros(M, device="cuda")
        pz.pack_factors(U, None, K, K, ud, None, cs)
        outs.append((host(ud).copy(), host(cs).copy()))
    assert all(np.array_equal(outs[0][1], o[1]) for o in outs[1:])   # fixed-order column sums
    assert np.array_equal(_tf32_bits(outs[0][0]), _tf32_rna(host(U).T))


# --------------------------------------- K1 on MN-major (in-place) factors ----
@pytest.mark.parametrize("M,N,K,P,ldu", [(200, 300, 6, 2, 200), (128, 256, 8, 1, 128), (1000, 1024, 37, 2, 1004),
                                         (300, 520, 64, 4, 304), (256, 512, 256, 1, 256), (4, 4, 1, 1, 4)])
def test_reconstruct_sgd_mn_integer_bit_exact(pz, M, N, K, P, ldu):
    """K1 reading the factors as the layer produced them (U [P][K][ldu], V [P][K][N], MN contiguous): integer
    variant bit-exact vs O4; ragged M / N / K tails, padded ldu, single-row K, tiny tiles."""
    g = S.rng(M + N + K)
    U = np.zeros((P, K, ldu), np.float32)
    U[:, :, :M] = g.integers(-3, 4, size=(P, K, M))
    U[:, :, M:] = 1e6                              # columns [M, ldu) must never be read
    V = g.integers(0, 4, size=(P, K, N)).astype(np.float32)
    W = (g.integers(-1023, 1024, size=(M, N)) * 2.0 ** -10).astype(np.float32)
    lr = 2.0 ** -7
    Wd = dev(W)
    pz.reconstruct_sgd_mn(dev(U), dev(V), P, K, M, N, Wd, -lr / P)
    W1, _ = O.sync_step(W, None, [U[p, :, :M] for p in range(P)], [V[p] for p in range(P)], lr)
    assert np.array_equal(host(Wd).astype(np.float64), W1)


@pytest.mark.parametrize("M,N,K,P", [(1000, 4096, 256, 1), (512, 1024, 100, 3)])
def test_reconstruct_sgd_mn_equals_kmajor(pz, M, N, K, P):
    """Same factors, two operand layouts: the MN-major and the K-major (transposed, zero-padded) K1 give
    bit-identical W (same accumulation order), random fp32 factors."""
    U = torch.randn(P, K, M, device="cuda") * 0.01
    V = torch.randn(P, K, N, device="cuda").relu()
    W = torch.randn(M, N, device="cuda")
    ldk = (K + 3) // 4 * 4
    Ug = torch.zeros(P, M, ldk, device="cuda")
    Vg = torch.zeros(P, N, ldk, device="cuda")
    Ug[:, :, :K] = U.transpose(1, 2)
    Vg[:, :, :K] = V.transpose(1, 2)
    Wa, Wb = W.clone(), W.clone()
    pz.reconstruct_sgd_mn(U, V, P, K, M, N, Wa, -1e-3)
    pz.reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, Wb, -1e-3)
    torch.cuda.synchronize()
    assert torch.equal(Wa, Wb)


def test_reconstruct_sgd_mn_random_vs_oracle(pz):
    """Random hidden-layer factors at the C3 fc6 shape, P = 1: within the TF32 gate of O4 (the tensor core
    reads the fp32 factors as TF32, truncating: reading Z12'), sampled rows."""
    M, N, K = 4096, 9216, 256
    W, _ = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, 1)
    lr = 0.5
    Wd = dev(W)
    pz.reconstruct_sgd_mn(dev(Us[0]), dev(Vs[0]), 1, K, M, N, Wd, -lr)
    rows = _sampled_rows(M, seed=5)
    W1r, _ = O.sync_step_rows(W[rows], None, Us, Vs, lr, rows)
    check_update(W[rows], host(Wd)[rows], W1r, TOL_TF32)


def test_reconstruct_sgd_mn_rejects_bad_layouts(pz):
    U = torch.zeros(2, 8, 6, device="cuda")    # ldu = 6: not a multiple of 4
    V = torch.zeros(2, 8, 16, device="cuda")
    W = torch.zeros(6, 16, device="cuda")
    with pytest.raises(pz.PoseidonError):
        pz.reconstruct_sgd_mn(U, V, 2, 8, 6, 16, W, 1.0)
