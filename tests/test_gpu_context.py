"""GPU tests of the context-level C ABI at world == 1 (P = 1: no collective;
SFB degenerates to K1 on local factors with alpha = -lr, PS to K2 over the
whole buffer — reading Z10), compared with the fp64 oracle."""
import numpy as np
import pytest

import oracle as O
from parity import check_update
import synthetic as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def test_context_sfps_world1(pz):
    """SF-PS at P = 1 (scheme_override = 2): the only master owns every row, so the step is K1 on the
    local factors (integer variant bit-exact vs O11); the bias follows the same update."""
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    M, N, K = 130, 64, 5
    assert ctx.register_layer(0, pz.LAYER_FC, M, N, K, scheme_override=pz.SCHEME_SFPS) == pz.SCHEME_SFPS
    assert ctx.sfb_path(0) == pz.SFB_PATH_SFPS
    with pytest.raises(pz.PoseidonError):
        ctx.register_layer(1, pz.LAYER_CONV, M, N, K, scheme_override=pz.SCHEME_SFPS)
    for recon in (pz.RECON_TF32, pz.RECON_FP32):
        ctx.set_recon(recon, 0)
        W, b, Us, Vs, lr = S.integer_factors(M, N, K, 1, seed=31)
        Wd, bd = dev(W), dev(b)
        ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
        ctx.wait_layer(0)
        st = ctx.iteration_end(stats=True)
        W1, b1, _ = O.sf_ps_simulated(W, b, Us, Vs, lr)
        assert np.array_equal(host(Wd).astype(np.float64), W1)
        assert np.array_equal(host(bd).astype(np.float64), b1)
        assert st["nccl_bytes_sent"] == 0 and st["n_layers"] == 1
    ctx.close()


def test_context_early_input_world1(pz):
    """FLAG_EARLY_V at P = 1: V posted at forward time, the sync's own V argument ignored (garbage here),
    integer variant bit-exact vs O4 over two syncs; misuse is refused."""
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device(), flags=pz.FLAG_EARLY_V)
    M, N, K = 70, 132, 6
    assert ctx.register_layer(0, pz.LAYER_FC, M, N, K) == pz.SCHEME_SFB
    ctx.register_layer(1, pz.LAYER_CONV, 8, 8, K)
    W, b, _, _, lr = S.integer_factors(M, N, K, 1, seed=41)
    Wd, bd = dev(W), dev(b)
    Wr, br = W.astype(np.float64), b.astype(np.float64)
    for t in range(2):
        _, _, Us, Vs, _ = S.integer_factors(M, N, K, 1, seed=50 + t)
        ctx.sfb_post_input(0, dev(Vs[0]))
        with pytest.raises(pz.PoseidonError):
            ctx.sfb_post_input(0, dev(Vs[0]))           # one post per sync
        ctx.sync_fc_sfb(0, dev(Us[0]), dev(np.full_like(Vs[0], 7.0)), Wd, bd, lr)
        ctx.wait_layer(0)
        ctx.iteration_end()
        Wr, br = O.sync_step(Wr, br, Us, Vs, lr)
        assert np.array_equal(host(Wd).astype(np.float64), Wr)
        assert np.array_equal(host(bd).astype(np.float64), br)
    with pytest.raises(pz.PoseidonError):
        ctx.sfb_post_input(1, dev(np.zeros((K, 8), np.float32)))   # not an SFB layer
    ctx.close()
    plain = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    plain.register_layer(0, pz.LAYER_FC, M, N, K)
    with pytest.raises(pz.PoseidonError):
        plain.sfb_post_input(0, dev(np.zeros((K, N), np.float32)))  # context without FLAG_EARLY_V
    plain.close()


def test_context_sfb_and_ps_world1(pz):
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    M, N, K = 128, 256, 8
    assert ctx.register_layer(0, pz.LAYER_FC, M, N, K) == pz.SCHEME_SFB
    assert ctx.register_layer(1, pz.LAYER_FC, M, N, K, scheme_override=pz.SCHEME_PS) == pz.SCHEME_PS
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, 1)
    lr = 0.25
    Wd, bd = dev(W), dev(b)
    ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
    # PS path of the same layer: flat buffer W||b and its gradient
    n = M * N + M
    _, _, padded = pz.shard_range(n, 1, 0)
    flatW = torch.zeros(padded, device="cuda")
    flatW[:n] = dev(O.flatten_params(W, b).astype(np.float32))
    G = Us[0].astype(np.float64).T @ Vs[0].astype(np.float64)
    flatG = torch.zeros(padded, device="cuda")
    flatG[:n] = dev(O.flatten_params(G, Us[0].astype(np.float64).sum(0)).astype(np.float32))
    ctx.bind_ps_buffers(1, flatG, flatW, n, pz.PS_ZERO_GRAD)
    ctx.sync_ps(1, flatG, flatW, n, lr)
    ctx.wait_layer(0)
    ctx.wait_layer(1)
    st = ctx.iteration_end(stats=True)
    assert st["n_layers"] == 2 and st["nccl_bytes_sent"] == 0
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    check_update(W, host(Wd), W1, 2e-3)
    check_update(b, host(bd), b1, 1e-5)
    out = host(flatW)
    check_update(W, out[:M * N].reshape(M, N), W1, 1e-5)
    check_update(b, out[M * N:n], b1, 1e-5)
    assert np.all(host(flatG) == 0)  # PS_ZERO_GRAD
    ls = ctx.layer_stats(0)
    assert ls["launched"] == 1 and ls["kernel_ms"] > 0
    ctx.close()


def test_context_hook_slot_path_and_dwbp_off(pz):
    for flags in (0, pz.FLAG_DWBP_OFF):
        ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device(), flags=flags)
        M, N, K = 1000, 1024, 16
        ctx.register_layer(3, pz.LAYER_FC, M, N, K)
        W, b = S.fc_weights_randbias(M, N)
        Us, Vs = S.hidden_factors(M, N, K, 1, seed=44)
        Wd, bd = dev(W), dev(b)
        ctx.bind_sfb_params(3, Wd, bd)
        ctx.set_lr(0.1)
        u_ptr, ldu, v_ptr, ldv = ctx.sfb_slot(3)
        assert ldu == 1000 and ldv == 1024
        # write the factors straight into the slot (zero-copy path)
        from paper_1512_06216_b200.binding import device_view
        device_view(u_ptr, (K, ldu)).copy_(dev(Us[0]))
        device_view(v_ptr, (K, ldv)).copy_(dev(Vs[0]))
        ctx.backprop_hook(3)
        st = ctx.iteration_end(stats=True)
        assert st["n_layers"] == 1
        ctx.wait_layer(3)
        W1, b1 = O.sync_step(W, b, Us, Vs, 0.1)
        check_update(W, host(Wd), W1, 2e-3)
        check_update(b, host(bd), b1, 1e-5)
        ctx.close()


def test_context_errors(pz):
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    with pytest.raises(pz.PoseidonError) as ei:
        ctx.backprop_hook(7)
    assert ei.value.code == -8  # not registered
    ctx.register_layer(7, pz.LAYER_CONV, 96, 363, 256)
    with pytest.raises(pz.PoseidonError):
        ctx.sync_fc_sfb(7, 1, 1, 1, None, 0.1)  # PS layer
    with pytest.raises(pz.PoseidonError):
        ctx.register_layer(8, pz.LAYER_CONV, 4, 4, 4, scheme_override=pz.SCHEME_SFB)
    g = torch.zeros(96 * 363 + 96 + 64, device="cuda")
    with pytest.raises(pz.PoseidonError):
        ctx.bind_ps_buffers(7, g, g, 12345)  # wrong n
    ctx.close()


@pytest.mark.parametrize("n", [1, 3, 5, 650, 4097, 100003])
def test_ps_zero_grad_odd_sizes(pz, n):
    """K2 with the fused gradient clear at P = 1: exact update of W[0, n), W padding untouched,
    the whole padded gradient buffer (garbage padding included) zero afterwards."""
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    ctx.register_layer(0, pz.LAYER_CONV, 1, n, 1, False)
    _, _, padded = pz.shard_range(n, 1, 0)
    g = S.integer_grads(n, 1, seed=n)[0]
    w0 = (S.rng(n + 1).integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
    gflat = torch.full((padded,), 5.0, device="cuda")
    gflat[:n] = dev(g)
    wflat = torch.full((padded,), -3.0, device="cuda")
    wflat[:n] = dev(w0)
    ctx.bind_ps_buffers(0, gflat, wflat, n, pz.PS_ZERO_GRAD)
    lr = 2.0 ** -7
    ctx.sync_ps(0, gflat, wflat, n, lr)
    ctx.wait_layer(0)
    ctx.iteration_end()
    torch.cuda.synchronize()
    out = host(wflat)
    assert np.array_equal(out[:n].astype(np.float64), O.ps_step_flat(w0, [g], lr))
    assert np.all(out[n:] == -3.0)
    assert np.all(host(gflat) == 0)
    ctx.close()


@pytest.mark.parametrize("bucket_kb", [0, 16, 256])
def test_ps_buckets_world1(pz, bucket_kb):
    """PS layers in buckets (one flat sync per bucket) give exactly O6 per layer, clear every gradient,
    and report the bucket's stats for each member."""
    from paper_1512_06216_b200.binding import device_view
    shapes = [(10, 65), (32, 64), (3, 1), (96, 363), (64, 1025), (500, 400)]   # n = M*N + M
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    for lid, (M, N) in enumerate(shapes):
        ctx.register_layer(lid, pz.LAYER_CONV, M, N, 1, True, pz.SCHEME_PS)
    ctx.set_ps_buckets(bucket_kb * 1024)
    ctx.ps_arena()
    lr = 2.0 ** -7
    ctx.set_lr(lr)
    refs, views = [], []
    for lid, (M, N) in enumerate(shapes):
        n = M * N + M
        gp, wp, padded = ctx.ps_layer_buffers(lid)
        g = S.integer_grads(n, 1, seed=lid)[0]
        w0 = (S.rng(100 + lid).integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
        wv, gv = device_view(wp, (padded,)), device_view(gp, (padded,))
        wv[:n] = dev(w0)
        gv[:n] = dev(g)
        refs.append(O.ps_step_flat(w0, [g], lr))
        views.append((wv, gv, n))
    torch.cuda.synchronize()
    for lid in reversed(range(len(shapes))):          # backward order
        ctx.backprop_hook(lid, torch.cuda.current_stream())
    for lid in range(len(shapes)):
        ctx.wait_layer(lid)
    st = ctx.iteration_end(stats=True)
    torch.cuda.synchronize()
    for (wv, gv, n), ref in zip(views, refs):
        assert np.array_equal(host(wv)[:n].astype(np.float64), ref)
        assert np.all(host(gv)[:n] == 0)
    if bucket_kb == 0:
        assert st["n_layers"] == len(shapes)
    else:
        assert st["n_layers"] < len(shapes)            # buckets count once
    for lid in range(len(shapes)):
        assert ctx.layer_stats(lid)["launched"] == 1
    ctx.close()


@pytest.mark.parametrize("mn", [False, True])
@pytest.mark.parametrize("M,N,K", [(128, 256, 8), (1000, 4096, 256), (100, 200, 37), (130, 256, 8)])
def test_context_inplace_factors_world1(pz, M, N, K, mn):
    """POSEIDON_FLAG_INPLACE_FACTORS at world 1: the pack reads U [K x M] and V [K x N] in place on the
    reconstruction stream; with POSEIDON_FLAG_INPLACE_MN K1 reads them itself (MN-major, no pack) and forms the
    bias sums.  Integer variant bit-exact vs O4 (W and bias); random factors within the TF32 / fp32 gates;
    M = 130 (not a multiple of 4) falls back to the pack; a second iteration reuses the layer; no pack time is
    reported for the MN in-place syncs."""
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device(),
                     flags=pz.FLAG_INPLACE_FACTORS | (pz.FLAG_INPLACE_MN if mn else 0))
    assert ctx.register_layer(0, pz.LAYER_FC, M, N, K, has_bias=True) == pz.SCHEME_SFB
    inplace = mn and M % 4 == 0
    # integer variant: bit-exact
    W, b, Us, Vs, lr = S.integer_factors(M, N, K, 1, seed=M + K)
    Wd, bd = dev(W), dev(b)
    Ud, Vd = dev(Us[0]), dev(Vs[0])
    ctx.sync_fc_sfb(0, Ud, Vd, Wd, bd, lr)
    ctx.wait_layer(0)
    ctx.iteration_end()
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    assert np.array_equal(host(Wd).astype(np.float64), W1)
    assert np.array_equal(host(bd).astype(np.float64), b1)
    assert (ctx.layer_stats(0)["pack_ms"] == 0) == inplace
    # random hidden-layer factors: gates
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, 1)
    lr = 0.5
    Wd, bd = dev(W), dev(b)
    ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
    ctx.wait_layer(0)
    ctx.iteration_end()
    W1, b1 = O.sync_step(W, b, Us, Vs, lr)
    check_update(W, host(Wd), W1, 2e-3)
    check_update(b, host(bd), b1, 1e-5)
    ctx.close()
