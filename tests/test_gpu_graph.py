"""CUDA-graph capture of a whole DWBP training step (round 2; bench.py --graph): the library sees the capture on
the caller's stream, forks its streams from it, records its statistics events as graph nodes and rejoins at
iteration_end.  A replayed step must compute exactly what an eager step computes (same kernels, same order of
every reduction; cuDNN deterministic), and the statistics read after a replay must describe that replay.

  * CIFAR-quick (C2 model, PS layers through K2), and the same net with its FC layers on SFB (K1; with and
    without POSEIDON_FLAG_INPLACE_FACTORS, and with momentum + weight decay fused into K1 / K2):
    4 eager steps == 2 eager + 2 replays, bit for bit;
  * after a replay: every layer's sync has a positive duration, starts after its ready event, and DWBP still
    overlaps the backward (every layer above the first starts its sync before the backward ends).
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


def _batches(dev, n):
    g = torch.Generator(device=dev)
    g.manual_seed(1512)
    return [(torch.rand((100, 3, 32, 32), device=dev, generator=g), torch.randint(0, 10, (100,), device=dev,
                                                                                   generator=g)) for _ in range(n)]


def _run(pz, scheme, flags, graph, mom=False):
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CifarQuick

    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    dev = torch.device("cuda", 0)
    ctx = pz.Context(rank=0, world=1, device=0, flags=flags)
    torch.manual_seed(6216)
    model = CifarQuick().to(dev)
    sync = PoseidonSync(model, ctx, K=100, lr=0.05, scheme=scheme)
    if mom:   # f4: velocities live in the library; the fused-momentum K1 / K2 variants are captured
        ctx.set_momentum(0.9, 5e-4)
    data = _batches(dev, 4)
    x = torch.empty_like(data[0][0])
    y = torch.empty_like(data[0][1])

    def step():
        F.cross_entropy(model(x), y).backward()
        sync.iteration_end()

    stats = None
    for i, (xb, yb) in enumerate(data):
        x.copy_(xb)
        y.copy_(yb)
        if graph and i == 2:
            sync.wait_all()
            torch.cuda.synchronize()
            gs = torch.cuda.Stream(device=dev)
            gs.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                step()
            torch.cuda.current_stream().wait_stream(gs)
        if graph and i >= 2:
            g.replay()
        else:
            step()
    sync.wait_all()
    torch.cuda.synchronize()
    if graph:
        stats = {p.name: ctx.layer_stats(p.layer_id, 0) for p in sync.plans}
        it = ctx.iter_stats(0)
        stats["_iter"] = it
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
    if graph:
        del g   # release the graph before the context (its NCCL work, if any, holds the communicator)
    ctx.close()
    return flat, stats


@pytest.mark.parametrize("scheme,flags", [("ps", 0), ("auto", 0), ("auto", "inplace"), ("auto", "momentum")])
def test_graph_replay_equals_eager(pz, scheme, flags):
    fl = (pz.FLAG_INPLACE_FACTORS | pz.FLAG_INPLACE_MN) if flags == "inplace" else 0
    mom = flags == "momentum"
    w_eager, _ = _run(pz, scheme, fl, False, mom)
    w_graph, stats = _run(pz, scheme, fl, True, mom)
    assert torch.equal(w_eager, w_graph)
    it = stats.pop("_iter")
    assert it["n_layers"] == len(stats) and it["sync_total_ms"] > 0
    for name, st in stats.items():
        assert st["start_to_done_ms"] > 0, (name, st)
        if name != "conv1":   # DWBP: the sync of every layer above the first overlaps the backward below it
            assert st["done_after_bwd_end_ms"] - st["start_to_done_ms"] < 0, (name, st)


def test_ssp_refuses_capture(pz):
    """SSP (staleness 1) carries host-side state from one iteration to the next (which gather / gradient set a
    sync uses): a captured step would replay one fixed assignment, so the library refuses the capture."""
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CifarQuick

    dev = torch.device("cuda", 0)
    ctx = pz.Context(rank=0, world=1, device=0, flags=pz.FLAG_SSP1)
    torch.manual_seed(6216)
    model = CifarQuick().to(dev)
    sync = PoseidonSync(model, ctx, K=100, lr=0.05, arena=True)
    x, y = _batches(dev, 1)[0]
    F.cross_entropy(model(x), y).backward()
    sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()
    gs = torch.cuda.Stream(device=dev)
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with pytest.raises(Exception):
        with torch.cuda.graph(g, stream=gs):
            F.cross_entropy(model(x), y).backward()
            sync.iteration_end()
    torch.cuda.synchronize()
    del g
    ctx.close()
