"""Parity of the full DWBP path in the launch configuration bench.py times
(C3 AlexNet, batch 256, P = 1, SACP auto): one training step through
PoseidonSync, then
  * fc6 / fc7 / fc8 (SFB, K1 tcgen05): W' vs the oracle's O4 on the captured
    sufficient factors (grad_out, input), on sampled output rows (TF32 gate);
  * conv1 .. conv5 (PS, K2): W' vs the oracle's PS step on the captured
    gradient, every element (fp32 gate);
  * the integer-exact property is covered by test_gpu_kernels; here the
    factors are the real backprop ones.
"""
import numpy as np
import pytest

import oracle as O
from parity import check_update

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1512_06216_b200 as pz
    return pz


@pytest.mark.parametrize("cfg,factors", [("C3", "async"), ("C3", "mn"), ("C3", "pack"), ("C5", "mn")])
def test_alexnet_step_matches_oracle(pz, cfg, factors):
    """factors="mn" is bench.py's N = 1 default (POSEIDON_FLAG_INPLACE_FACTORS | _INPLACE_MN: K1 reads grad_out
    and x in place, MN-major, no pack); "async" keeps the pack but runs it on the library's stream; "pack" the
    round-1 path (K3 on the backward's stream).  C5 = the ImageNet-22K AlexNet: its 21841-way fc8 (M not a
    multiple of 4) is packed even under "mn", fc6 / fc7 are read in place."""
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import AlexNet

    dev = torch.device("cuda", 0)
    torch.manual_seed(6216)
    classes = 21841 if cfg == "C5" else 1000
    model = AlexNet(n_classes=classes).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1512)
    x = torch.rand((256, 3, 227, 227), device=dev, generator=g)
    y = torch.randint(0, classes, (256,), device=dev, generator=g)
    # lr large enough that every layer's update is at least a quarter of its weights, so the fp32 gate
    # tests the update and not the storage rounding of W' (tests/parity.py: at lr = 0.05 the conv updates
    # are ~1e-4 of W and one ulp of W' would be most of the 1e-5 gate).  A plain torch backward of the same
    # batch (before the hooks exist) gives each layer's max|grad|.
    F.cross_entropy(model(x), y).backward()
    lr = max(float(p.detach().abs().max() / (4 * p.grad.abs().max())) for p in model.parameters())
    model.zero_grad(set_to_none=True)
    flags = {"async": pz.FLAG_INPLACE_FACTORS, "mn": pz.FLAG_INPLACE_FACTORS | pz.FLAG_INPLACE_MN, "pack": 0}[factors]
    ctx = pz.Context(rank=0, world=1, device=0, flags=flags)
    sync = PoseidonSync(model, ctx, K=256, lr=lr)
    plans = {p.name: p for p in sync.plans}
    fcs, convs = ("fc6", "fc7", "fc8"), ("conv1", "conv2", "conv3", "conv4", "conv5")
    assert all(plans[n].scheme == pz.SCHEME_SFB for n in fcs)
    assert all(plans[n].scheme == pz.SCHEME_PS for n in convs)

    captured = {}
    orig_sfb = sync.sfb_backward

    def sfb_capture(plan, grad_out, x, weight, bias):
        captured[plan.name] = (grad_out.detach().clone(), x.detach().clone())
        orig_sfb(plan, grad_out, x, weight, bias)

    sync.sfb_backward = sfb_capture
    grads = {}
    before = {n: (plans[n].module.weight.detach().clone(), plans[n].module.bias.detach().clone())
              for n in fcs + convs}
    # capture PS gradients: wrap the context's backprop_hook
    orig_hook = ctx.backprop_hook

    def hook_capture(layer_id, stream=None):
        for n in convs:
            if plans[n].layer_id == layer_id:
                m = plans[n].module
                grads[(n, "w")] = m.weight.grad.detach().clone()
                grads[(n, "b")] = m.bias.grad.detach().clone()
        orig_hook(layer_id, stream)

    ctx.backprop_hook = hook_capture

    loss = F.cross_entropy(model(x), y)
    loss.backward()
    sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()

    rng = np.random.default_rng(0)
    for name in fcs:
        G, X = (t.cpu().numpy() for t in captured[name])
        W0, b0 = (t.cpu().numpy() for t in before[name])
        W1 = plans[name].module.weight.detach().cpu().numpy()
        b1 = plans[name].module.bias.detach().cpu().numpy()
        M = W0.shape[0]
        rows = np.unique(np.concatenate([[0, M - 1], rng.integers(0, M, 40)]))
        Wr, br = O.sync_step_rows(W0[rows], b0[rows], [G], [X], lr, rows)
        check_update(W0[rows], W1[rows], Wr, 2e-3, name)
        check_update(b0[rows], b1[rows], br, 1e-5, name)
    for name in convs:
        W0, b0 = (t.cpu().numpy() for t in before[name])
        gw = grads[(name, "w")].cpu().numpy()
        gb = grads[(name, "b")].cpu().numpy()
        ref = O.ps_step_flat(O.flatten_params(W0, b0), [O.flatten_params(gw, gb)], lr)
        mod = plans[name].module
        out = O.flatten_params(mod.weight.detach().cpu().numpy(), mod.bias.detach().cpu().numpy())
        check_update(O.flatten_params(W0, b0), out, ref, 1e-5, name)
    ctx.close()
