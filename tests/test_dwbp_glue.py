"""Host-side checks of the DWBP glue (no GPU): the SFB Linear wrapper posts the layer input for the early
input broadcast only in a forward that will be backpropagated, hands (grad_out, input) to the library in
backward, and returns dX = grad_out @ W (Alg. 2 line 7) without forming dW.  The library context is a
recording stand-in; all arithmetic checked here is the wrapper's own dX."""
import pytest
import torch
import torch.nn as nn

from paper_1512_06216_b200 import binding as B
from paper_1512_06216_b200.dwbp import LayerPlan, PoseidonSync


class _RecordingCtx:
    def __init__(self):
        self.posted, self.synced = [], []

    def sfb_post_input(self, layer_id, V, stream=None):
        self.posted.append((layer_id, V.detach().clone()))

    def sync_fc_sfb(self, layer_id, U, V, W=None, bias=None, lr=0.0, producer=None):
        self.synced.append((layer_id, U.detach().clone(), V.detach().clone()))


@pytest.fixture
def wrapped(monkeypatch):
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a, **k: None)
    torch.manual_seed(0)
    mod = nn.Linear(6, 4)
    sync = PoseidonSync.__new__(PoseidonSync)   # no library context: only the wrapper is under test
    sync.ctx = _RecordingCtx()
    sync.lr = 0.1
    sync.early_v = True
    plan = LayerPlan(3, "fc", mod, B.LAYER_FC, 4, 6, 5, B.SCHEME_SFB, B.SCHEME_SFB, (0, 0, 0))
    sync._wrap_linear(mod, plan)
    return mod, sync


def test_forward_posts_input_and_backward_hands_factors(wrapped):
    mod, sync = wrapped
    x = torch.randn(5, 6, requires_grad=True)
    y = mod(x)
    assert torch.allclose(y, x @ mod.weight.t() + mod.bias)
    assert len(sync.ctx.posted) == 1 and sync.ctx.posted[0][0] == 3
    assert torch.equal(sync.ctx.posted[0][1], x.detach())
    g = torch.randn(5, 4)
    y.backward(g)
    (lid, U, V), = sync.ctx.synced
    assert lid == 3 and torch.equal(U, g) and torch.equal(V, x.detach())
    assert torch.allclose(x.grad, g @ mod.weight.detach())
    assert mod.weight.grad is None   # the local dW is never formed (Eq. 5: the factors travel instead)


def test_no_grad_forward_posts_nothing(wrapped):
    mod, sync = wrapped
    with torch.no_grad():
        mod(torch.randn(5, 6))
    assert sync.ctx.posted == []


def test_early_v_off_posts_nothing(wrapped):
    mod, sync = wrapped
    sync.early_v = False
    mod(torch.randn(5, 6, requires_grad=True))
    assert sync.ctx.posted == []


def test_describe_reports_rule_and_models():
    """describe() (bench.py's per-layer JSON) names the executed scheme, the paper's rule and both model picks."""
    class _Ctx:
        world = 4

    sync = PoseidonSync.__new__(PoseidonSync)
    sync.ctx = _Ctx()
    fc6 = LayerPlan(5, "fc6", None, B.LAYER_FC, 4096, 9216, 256, B.SCHEME_SFB, B.SCHEME_SFB,
                    B.choose_scheme(B.LAYER_FC, 4096, 9216, 256, 4)[1])
    big = LayerPlan(7, "fc8", None, B.LAYER_FC, 21841, 4096, 2048, B.SCHEME_SFPS, B.SCHEME_SFB,
                    B.choose_scheme(B.LAYER_FC, 21841, 4096, 2048, 4)[1])
    sync.plans = [fc6, big]
    d = {x["name"]: x for x in sync.describe()}
    assert d["fc6"]["scheme"] == "SFB" and d["fc6"]["rule"] == "SFB" and d["fc6"]["model3"] == "SFB"
    assert d["fc8"]["scheme"] == "SFPS" and d["fc8"]["model3"] == "SFPS"
    assert d["fc8"]["model_t_sfps_us"] < d["fc8"]["model_t_sfb_us"]


class _FakeContext:
    """Stands in for B.Context on the host: records the calls the glue makes, takes the paper's rule for the
    scheme (no library state, no device)."""

    def __init__(self, flags=0):
        self.world, self.rank, self.flags = 1, 0, flags
        self.calls = []

    def set_lr(self, lr):
        pass

    def register_layer(self, lid, kind, M, N, K, has_bias=True, scheme_override=-1):
        return scheme_override if scheme_override >= 0 else B.choose_scheme(kind, M, N, K, self.world)[0]

    def set_recon(self, recon, lid=-1):
        pass

    def bind_sfb_params(self, lid, W, bias):
        pass

    def bind_ps_buffers(self, lid, grad, W, n, flags=0):
        pass

    def backprop_hook(self, lid, stream=None):
        self.calls.append(("sync", lid))

    def sync_fc_sfb(self, lid, U, V, W=None, bias=None, lr=0.0, producer=None):
        self.calls.append(("sync", lid))

    def sfb_post_input(self, lid, V, stream=None):
        self.calls.append(("post", lid))

    def wait_layer(self, lid, stream=None):
        self.calls.append(("wait", lid))

    def iteration_end(self, stream=None, stats=False):
        self.calls.append(("end", -1))


def test_dwbp_hook_order_and_next_forward_barrier(monkeypatch):
    """Alg. 2 on the host side (SURVEY T4 enqueue order): within one backward every layer's sync is issued
    exactly once, top layer first (the order the collectives must have on every rank), SFB layers from the
    layer's own backward (their inputs posted in the forward when early V is on), PS layers once all their
    gradients have accumulated; the next forward of layer i waits for layer i's sync before it runs."""
    from drivers.cnn import CifarQuick
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a, **k: None)
    for flags in (0, B.FLAG_EARLY_V):
        torch.manual_seed(0)
        model = CifarQuick()
        ctx = _FakeContext(flags)
        sync = PoseidonSync(model, ctx, K=4, lr=0.1)
        ids = [p.layer_id for p in sync.plans]
        assert [p.name for p in sync.plans] == ["conv1", "conv2", "conv3", "ip1", "ip2"]
        sfb = [p.layer_id for p in sync.plans if p.scheme == B.SCHEME_SFB]
        assert sfb == [3, 4]   # the rule at P = 1: the FC layers broadcast their factors
        for it in range(2):
            ctx.calls.clear()
            x, y = torch.rand(4, 3, 32, 32), torch.randint(0, 10, (4,))
            out = model(x)
            torch.nn.functional.cross_entropy(out, y).backward()
            sync.iteration_end()
            waits = [lid for c, lid in ctx.calls if c == "wait"]
            posts = [lid for c, lid in ctx.calls if c == "post"]
            syncs = [lid for c, lid in ctx.calls if c == "sync"]
            assert waits == ids                         # next-forward barrier, in forward order
            assert posts == (sfb if flags else [])      # early V: in the forward, SFB layers only
            assert syncs == ids[::-1]                   # DWBP: top -> bottom, once each
            first_sync = min(i for i, c in enumerate(ctx.calls) if c[0] == "sync")
            assert all(i < first_sync for i, c in enumerate(ctx.calls) if c[0] in ("wait", "post"))
            assert ctx.calls[-1] == ("end", -1)


@pytest.mark.parametrize("shape", [(4, 6), (6, 6), (5, 7), (5, 2, 3)])
def test_sfb_layer_refuses_batch_other_than_registered_K(wrapped, shape):
    """the library reads the factors with the registered K; a partial last batch, a
    larger batch or a >2-D input must fail loudly before anything reaches the C ABI."""
    mod, sync = wrapped
    with pytest.raises(ValueError, match="registered per-GPU batch K"):
        mod(torch.randn(*shape, requires_grad=True))
    assert sync.ctx.posted == [] and sync.ctx.synced == []


def test_binding_refuses_factor_shapes_other_than_registered():
    """The binding's factor check (argument marshalling: shapes against the registration) runs before
    the C call; a context stand-in carries the registered (M, N, K)."""
    c = B.Context.__new__(B.Context)
    c._shapes = {0: (4, 6, 5)}
    c._check_factor(0, "U", torch.zeros(5, 4), 4)
    c._check_factor(0, "V", torch.zeros(5, 6), 6)
    for bad in [(4, 4), (5, 5), (6, 4), (5, 2, 2)]:
        with pytest.raises(ValueError, match="registered K"):
            c._check_factor(0, "U", torch.zeros(*bad), 4)


def test_inplace_factors_are_held_until_the_next_wait(monkeypatch):
    """POSEIDON_FLAG_INPLACE_FACTORS: the library reads an SFB layer's grad_out and input where they are, on its
    own streams, so the glue keeps both tensors alive from the layer's backward until the layer's next
    pre-forward hook has called wait_layer (or until wait_all), and drops them right after (no record_stream:
    plain stream-ordered reuse).  Without the flag, or with DWBP off, nothing is held."""
    from drivers.cnn import CifarQuick
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a, **k: None)
    for flags, expect in ((B.FLAG_INPLACE_FACTORS, True), (0, False),
                          (B.FLAG_INPLACE_FACTORS | B.FLAG_DWBP_OFF, False)):
        torch.manual_seed(0)
        model = CifarQuick()
        ctx = _FakeContext(flags)
        sync = PoseidonSync(model, ctx, K=4, lr=0.1)
        sfb = {p.layer_id for p in sync.plans if p.scheme == B.SCHEME_SFB}
        x, y = torch.rand(4, 3, 32, 32), torch.randint(0, 10, (4,))
        torch.nn.functional.cross_entropy(model(x), y).backward()
        sync.iteration_end()
        assert set(sync.held) == (sfb if expect else set())
        if expect:
            for lid in sfb:
                g, a = sync.held[lid]
                assert g.shape[0] == 4 and a.shape[0] == 4          # (K x M) error messages, (K x N) inputs
        # the next forward: each layer's hold ends at its own pre-forward hook, after its wait_layer
        waits_before = len([c for c in ctx.calls if c[0] == "wait"])
        model(x)
        assert sync.held == {}
        assert len([c for c in ctx.calls if c[0] == "wait"]) == waits_before + len(sync.plans)
        torch.nn.functional.cross_entropy(model(x), y).backward()
        sync.wait_all()
        assert sync.held == {}
