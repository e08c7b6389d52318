"""DWBP timing invariants (Alg. 2; "communication ... overlapped with the
backward of the layers below"), measured on the library's own device events at P = 1:

  * DWBP on: the sync of every layer above the first starts BEFORE the backward pass ends
    (t(start_i) < t(bwd_end)), i.e. it overlaps the backward of the layers below it;
  * DWBP off (traditional BP, Fig. dwbp (a)): every sync starts after the backward pass ended;
  * both give bit-identical parameters (scheduling only; O8).
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1512_06216_b200 as pz
    return pz


def _run(pz, dwbp_on):
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CifarQuick

    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    dev = torch.device("cuda", 0)
    ctx = pz.Context(rank=0, world=1, device=0, flags=0 if dwbp_on else pz.FLAG_DWBP_OFF)
    torch.manual_seed(6216)
    model = CifarQuick().to(dev)
    sync = PoseidonSync(model, ctx, K=256, lr=0.01)
    g = torch.Generator(device=dev)
    g.manual_seed(1512)
    for _ in range(4):
        x = torch.rand((256, 3, 32, 32), device=dev, generator=g)
        y = torch.randint(0, 10, (256,), device=dev, generator=g)
        F.cross_entropy(model(x), y).backward()
        sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()
    # start of layer i's sync relative to the end of the backward pass (ms; < 0: before it ended)
    rel = {p.name: ctx.layer_stats(p.layer_id, 0)["done_after_bwd_end_ms"] -
           ctx.layer_stats(p.layer_id, 0)["start_to_done_ms"] for p in sync.plans}
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
    ctx.close()
    return rel, flat


def test_dwbp_overlaps_backward_and_is_semantics_preserving(pz):
    rel_on, w_on = _run(pz, True)
    rel_off, w_off = _run(pz, False)
    # every layer but the first (whose gradient completes the backward pass) starts syncing while the
    # backward of the layers below is still running
    for name, t in rel_on.items():
        if name != "conv1":
            assert t < 0.0, (name, rel_on)
    # traditional BP: nothing starts before the whole backward has finished
    for name, t in rel_off.items():
        assert t >= -1e-3, (name, rel_off)
    assert torch.equal(w_on, w_off)


_FUZZ_CHILD = r"""
import sys, torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests")
import paper_1512_06216_b200 as pz
from test_gpu_dwbp import _run
rel, flat = _run(pz, {dwbp_on})
torch.save(flat, {out!r})
"""


@pytest.mark.parametrize("dwbp_on", [True, False])
def test_ordering_fuzz_changes_timing_not_results(pz, tmp_path, dwbp_on):
    """SURVEY §5 ordering fuzz: with POSEIDON_FUZZ_US every collective leg and update kernel is delayed by a
    pseudo-random sleep (up to 300 us) on its stream; a missing stream-order edge (e.g. a forward not waiting
    for its layer's update, a pack overwriting a buffer an update still reads) would change the parameters."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    _, ref = _run(pz, dwbp_on)
    out = str(tmp_path / "w.pt")
    env = dict(os.environ, POSEIDON_FUZZ_US="300")
    r = subprocess.run([sys.executable, "-c", _FUZZ_CHILD.format(root=root, dwbp_on=dwbp_on, out=out)],
                       env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert torch.equal(torch.load(out), ref)


def test_early_input_broadcast_is_bit_identical(pz):
    """FLAG_EARLY_V through the glue at P = 1: every SFB layer posts its input in the forward (counted), and
    the trained parameters equal the plain run bit for bit."""
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CifarQuick

    dev = torch.device("cuda", 0)
    out = {}
    for flags in (0, pz.FLAG_EARLY_V):
        ctx = pz.Context(rank=0, world=1, device=0, flags=flags)
        posts = []
        orig = ctx.sfb_post_input
        ctx.sfb_post_input = lambda lid, V, stream=None, _o=orig: (posts.append(lid), _o(lid, V, stream))
        torch.manual_seed(6216)
        model = CifarQuick().to(dev)
        sync = PoseidonSync(model, ctx, K=64, lr=0.01)
        g = torch.Generator(device=dev)
        g.manual_seed(1512)
        for _ in range(3):
            x = torch.rand((64, 3, 32, 32), device=dev, generator=g)
            y = torch.randint(0, 10, (64,), device=dev, generator=g)
            F.cross_entropy(model(x), y).backward()
            sync.iteration_end()
        with torch.no_grad():
            model(x)                     # an evaluation forward posts nothing
        sync.wait_all()
        torch.cuda.synchronize()
        n_sfb = sum(1 for p in sync.plans if p.scheme == pz.SCHEME_SFB)
        assert len(posts) == (3 * n_sfb if flags else 0), posts
        out[flags] = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
        ctx.close()
    assert torch.equal(out[0], out[pz.FLAG_EARLY_V])
