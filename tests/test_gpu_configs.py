"""Whole-config parity against the oracle at P = 1 in bench.py's launch configuration (channels_last,
per-GPU batch of BASELINE.json, DWBP on, SACP as bench runs it): one training step through PoseidonSync,
then EVERY parameterised layer's update is recomputed by the fp64 oracle from what the layer handed to
the library (tests/stepcheck.py): PS layers element by element (O6, 1e-5), factor layers on sampled rows
(O4, TF32 gate 2e-3), biases 1e-5.

  C2 cifar10_quick, batch 100, PS-only (BJ): 5 layers
  C4 bvlc_googlenet, batch 128, SACP auto: 57 conv layers PS + the 1024 x 1000 FC (SFB at P = 1)
  C3 and C5 (22K-way fc8) are covered by test_gpu_bench_path.py.  The context has bench.py's N = 1 flags
  (POSEIDON_FLAG_INPLACE_FACTORS | _INPLACE_MN: GoogLeNet's FC reads its factors in place); C2's CUDA-graph
  step equals the eager one bit for bit (test_gpu_graph.py).
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


@pytest.mark.parametrize("config,n_layers", [("C2", 5), ("C4", 58)])
def test_config_step_matches_oracle(pz, config, n_layers):
    import torch.nn.functional as F
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CONFIGS
    from stepcheck import StepCapture, oracle_check, safe_lr

    torch.backends.cudnn.deterministic = True
    cfg = CONFIGS[config]
    dev = torch.device("cuda", 0)
    torch.manual_seed(6216)
    model = cfg["model"]().to(dev).to(memory_format=torch.channels_last)
    g = torch.Generator(device=dev)
    g.manual_seed(1512)
    K = cfg["batch"]
    x = torch.rand((K, 3, cfg["hw"], cfg["hw"]), device=dev, generator=g).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, cfg["classes"], (K,), device=dev, generator=g)
    lr = safe_lr(model, lambda m: F.cross_entropy(m(x), y))
    ctx = pz.Context(rank=0, world=1, device=0, flags=pz.FLAG_INPLACE_FACTORS | pz.FLAG_INPLACE_MN)
    sync = PoseidonSync(model, ctx, K=K, lr=lr, scheme=cfg["scheme"])
    assert len(sync.plans) == n_layers
    cap = StepCapture(sync)
    cap.snapshot()
    F.cross_entropy(model(x), y).backward()
    sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()
    errs = oracle_check(cap, lr, 1)
    assert len(errs) == n_layers
    n_ps = sum(1 for p in sync.plans if p.scheme == pz.SCHEME_PS)
    assert n_ps == (5 if config == "C2" else 57)
    ctx.close()
