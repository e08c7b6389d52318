"""GPU parity of the f4 path (momentum + weight decay, the paper's Lambda) against the oracle's
O4m over several steps, through the context API at world == 1."""
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


@pytest.mark.parametrize("recon,tol,M,N,K", [("tf32", 2e-3, 300, 520, 16), ("fp32", 1e-5, 300, 520, 16),
                                             ("tf32", 2e-3, 4096, 4096, 384)])
def test_sfb_momentum_three_steps(pz, recon, tol, M, N, K):
    """Lambda fused into K1's epilogue (f4, O4m).  K = 384: 12 factor slabs per tile, the <4 stages, 2 W+V slots>
    configuration, and 256 tiles over 74 CTA pairs, so W slots are reused across tiles by both epilogue groups."""
    steps, lr, mu, wd = 3, 0.5, 0.9, 1e-2
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    ctx.register_layer(0, pz.LAYER_FC, M, N, K)
    ctx.set_recon(pz.RECON_TF32 if recon == "tf32" else pz.RECON_FP32, 0)
    ctx.set_momentum(0.9, wd, 0)
    W, b = S.fc_weights_randbias(M, N)
    Wd, bd = dev(W), dev(b)
    Wr, br = W.astype(np.float64), b.astype(np.float64)
    VW, Vb = np.zeros_like(Wr), np.zeros_like(br)
    for t in range(steps):
        Us, Vs = S.hidden_factors(M, N, K, 1, seed=100 + t)
        ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
        ctx.wait_layer(0)
        ctx.iteration_end()
        Wr, br, VW, Vb = O.sync_step_momentum(Wr, br, VW, Vb, Us, Vs, lr, mu, wd)
    torch.cuda.synchronize()
    check_update(W, Wd.cpu().numpy(), Wr, tol)
    check_update(b, bd.cpu().numpy(), br, 1e-5)
    # and switching back to plain SGD frees the velocity and follows O4
    ctx.set_momentum(0.0, 0.0, 0)
    W0 = Wd.cpu().numpy()
    Us, Vs = S.hidden_factors(M, N, K, 1, seed=7)
    ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
    ctx.wait_layer(0)
    W1, _ = O.sync_step(W0, None, Us, Vs, lr)
    torch.cuda.synchronize()
    check_update(W0, Wd.cpu().numpy(), W1, tol)
    ctx.close()


def test_ps_momentum_three_steps(pz):
    M, N, steps, lr, mu, wd = 64, 75, 3, 0.05, 0.9, 5e-3
    n = M * N + M
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    ctx.register_layer(0, pz.LAYER_CONV, M, N, 1)
    ctx.set_momentum(mu, wd, 0)
    _, _, padded = pz.shard_range(n, 1, 0)
    W, b = S.fc_weights_randbias(M, N)
    w0 = O.flatten_params(W, b)
    wflat = torch.zeros(padded, device="cuda")
    wflat[:n] = dev(w0.astype(np.float32))
    gflat = torch.zeros(padded, device="cuda")
    ctx.bind_ps_buffers(0, gflat, wflat, n, pz.PS_ZERO_GRAD)
    wr, vr = w0.copy(), np.zeros(n)
    for t in range(steps):
        g = S.dense_grads(n, 1, seed=30 + t, scale=1.0)[0]
        gflat[:n] = dev(g)
        ctx.sync_ps(0, gflat, wflat, n, lr)
        ctx.wait_layer(0)
        ctx.iteration_end()
        wr, vr = O.ps_step_flat_momentum(wr, vr, [g], lr, mu, wd)
    torch.cuda.synchronize()
    check_update(w0, wflat[:n].cpu().numpy(), wr, 1e-5)
    ctx.close()


def test_set_momentum_validation(pz):
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    ctx.register_layer(0, pz.LAYER_CONV, 4, 4, 1)
    for bad in ((1.0, 0.0), (-0.1, 0.0), (0.5, -1.0)):
        with pytest.raises(pz.PoseidonError):
            ctx.set_momentum(*bad)
    ctx.close()
