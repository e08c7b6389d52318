"""GPU parity of SSP with staleness 1 (POSEIDON_FLAG_SSP1, reading Z19) against the oracle's O10
(ssp_visible_weights), through the context API at world == 1, and a DWBP training run of CIFAR-10
quick against single-GPU SGD with the same one-iteration delay."""
import copy

import numpy as np
import pytest

import oracle as O
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


@pytest.mark.parametrize("recon,s", [("tf32", 1), ("fp32", 1), ("tf32", 2), ("tf32", 3), ("fp32", 3)])
def test_ssp_sfb_and_ps_integer_exact(pz, recon, s):
    """Staleness s (poseidon_set_staleness; s = 1 is FLAG_SSP1's default): after the hook of iteration t the
    parameters hold exactly the updates of iterations <= t - s (O10), for SFB and PS; s + 1 gradient sets used
    round robin; flush applies the rest."""
    from paper_1512_06216_b200.binding import device_view
    M, N, K, T = 72, 136, 8, 7
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device(), flags=pz.FLAG_SSP1)
    if s != 1:
        ctx.set_staleness(s)
    ctx.register_layer(0, pz.LAYER_FC, M, N, K)                          # SFB
    ctx.register_layer(1, pz.LAYER_CONV, M, N, K, True, pz.SCHEME_PS)    # PS (arena)
    ctx.set_recon(pz.RECON_TF32 if recon == "tf32" else pz.RECON_FP32, 0)
    ctx.ps_arena()
    W, b, _, _, lr = S.integer_factors(M, N, K, 1, seed=40)
    steps = []
    for t in range(T):
        _, _, Us, Vs, _ = S.integer_factors(M, N, K, 1, seed=50 + t)
        steps.append((Us, Vs))
    vis = O.ssp_visible_weights(W, b, steps, lr, s=s)
    Wd, bd = dev(W), dev(b)
    n = M * N + M
    _, wp, padded = ctx.ps_layer_buffers(1)
    wflat = device_view(wp, (padded,))
    wflat[:n] = dev(O.flatten_params(W, b).astype(np.float32))
    ctx.set_lr(lr)
    seen_g = set()
    for t, (Us, Vs) in enumerate(steps):
        ctx.sync_fc_sfb(0, dev(Us[0]), dev(Vs[0]), Wd, bd, lr)
        gp = ctx.ps_layer_buffers(1)[0]           # the buffer this sync reduces
        seen_g.add(gp)
        gflat = device_view(gp, (padded,))
        g = O.flatten_params(O.reconstruct(Us[0], Vs[0]), Us[0].astype(np.float64).sum(0))
        gflat[:n] = dev(g.astype(np.float32))
        ctx.backprop_hook(1, torch.cuda.current_stream())
        ctx.wait_layer(0)
        ctx.wait_layer(1)
        ctx.iteration_end()
        torch.cuda.synchronize()
        Wv, bv = vis[t + 1]                       # after hook t: updates of iterations <= t-s
        assert np.array_equal(Wd.cpu().numpy().astype(np.float64), Wv), f"SFB step {t}"
        assert np.array_equal(bd.cpu().numpy().astype(np.float64), bv)
        assert np.array_equal(wflat[:n].cpu().numpy().astype(np.float64), O.flatten_params(Wv, bv)), f"PS step {t}"
    assert len(seen_g) == s + 1                    # the s + 1 gradient buffers are used round robin
    ctx.flush()
    ctx.wait_layer(0)
    ctx.wait_layer(1)
    torch.cuda.synchronize()
    Wf, bf = vis[T + s]
    assert np.array_equal(Wd.cpu().numpy().astype(np.float64), Wf)
    assert np.array_equal(bd.cpu().numpy().astype(np.float64), bf)
    assert np.array_equal(wflat[:n].cpu().numpy().astype(np.float64), O.flatten_params(Wf, bf))
    for gp in seen_g:                              # both gradient buffers are clean again
        assert float(device_view(gp, (padded,)).abs().sum()) == 0.0
    ctx.close()


def test_ssp1_flag_validation(pz):
    with pytest.raises(pz.PoseidonError):
        pz.Context(rank=0, world=1, device=torch.cuda.current_device(),
                   flags=pz.FLAG_SSP1 | pz.FLAG_DWBP_OFF)


def test_set_staleness_validation(pz):
    c0 = pz.Context(rank=0, world=1, device=torch.cuda.current_device())
    with pytest.raises(pz.PoseidonError):
        c0.set_staleness(2)                       # no SSP context
    c0.close()
    c1 = pz.Context(rank=0, world=1, device=torch.cuda.current_device(), flags=pz.FLAG_SSP1)
    for bad in (0, 6):
        with pytest.raises(pz.PoseidonError):
            c1.set_staleness(bad)
    c1.register_layer(0, pz.LAYER_FC, 8, 8, 4)
    with pytest.raises(pz.PoseidonError):
        c1.set_staleness(2)                       # after a registration
    c1.close()


@pytest.mark.parametrize("s", [1, 2])
def test_ssp_cifar_training_matches_delayed_sgd(pz, s):
    """DWBP steps of CIFAR-10 quick with SSP staleness s (SFB for ip1/ip2, PS for the convs) + flush equal
    single-GPU SGD where the gradient of iteration t is applied after the backward of t+s."""
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CifarQuick
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(3)
    model = CifarQuick().cuda()
    ref = copy.deepcopy(model)
    lr, T, B = 0.05, 4, 16
    ctx = pz.Context(rank=0, world=1, device=torch.cuda.current_device(), flags=pz.FLAG_SSP1)
    if s != 1:
        ctx.set_staleness(s)
    sync = PoseidonSync(model, ctx, K=B, lr=lr, arena=True)
    g = torch.Generator(device="cuda").manual_seed(11)
    batches = [(torch.rand(B, 3, 32, 32, device="cuda", generator=g),
                torch.randint(0, 10, (B,), device="cuda", generator=g)) for _ in range(T)]
    pending = []
    for x, y in batches:
        F.cross_entropy(model(x), y).backward()
        sync.iteration_end()
        ref.zero_grad()
        F.cross_entropy(ref(x), y).backward()
        pending.append([p.grad.detach().clone() for p in ref.parameters()])
        with torch.no_grad():
            if len(pending) > s:                  # after the backward of t: apply the gradient of t - s
                for p, gr in zip(ref.parameters(), pending.pop(0)):
                    p -= lr * gr
    sync.flush()
    with torch.no_grad():
        for grads in pending:
            for p, gr in zip(ref.parameters(), grads):
                p -= lr * gr
    torch.cuda.synchronize()
    for (name, p), (_, q) in zip(model.named_parameters(), ref.named_parameters()):
        w0 = q.detach().cpu().numpy()
        err = np.max(np.abs(p.detach().cpu().numpy() - w0)) / max(1e-12, np.max(np.abs(w0)))
        assert err < 2e-3, (name, err)
    ctx.close()
