"""K1 in-step CTA timeline (diagnostics): run C3 DWBP steps at P = 1 with POSEIDON_K1_PROF=1 and print, for
the last fc6 K1 launch, when each CTA pair started / finished relative to the first start (globaltimer),
next to the same launch alone.  Tells late CTA starts (SMs held by the concurrent conv backward) from a
uniformly slower stream (HBM shared with the backward).

    POSEIDON_K1_PROF=1 python tools/k1_prof.py
"""
import ctypes
import os
import statistics
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402
from paper_1512_06216_b200 import binding as B  # noqa: E402
from paper_1512_06216_b200.dwbp import PoseidonSync  # noqa: E402
from drivers.cnn import AlexNet  # noqa: E402

assert os.environ.get("POSEIDON_K1_PROF") == "1"
fn = B.lib.poseidon_debug_k1_prof
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]


def stamps():
    buf = (ctypes.c_ulonglong * 2048)()
    n = fn(buf, 148)
    st = [buf[2 * i] for i in range(n)]
    en = [buf[2 * i + 1] for i in range(n)]
    t0 = min(st)
    return [(s - t0) / 1e3 for s in st], [(e - t0) / 1e3 for e in en]


def report(tag, st, en):
    st_s, en_s = sorted(st), sorted(en)
    print(f"{tag}: CTA start: min 0 / median {statistics.median(st):.1f} / p90 {st_s[int(0.9 * len(st))]:.1f} / "
          f"max {st_s[-1]:.1f} us;  end: min {en_s[0]:.1f} / median {statistics.median(en):.1f} / max {en_s[-1]:.1f} us;"
          f"  busy per CTA median {statistics.median([e - s for s, e in zip(st, en)]):.1f} us", flush=True)


dev = torch.device("cuda", 0)
torch.backends.cudnn.benchmark = True
torch.manual_seed(6216)
model = AlexNet().to(dev).to(memory_format=torch.channels_last)
ctx = pz.Context(rank=0, world=1, device=0)
sync = PoseidonSync(model, ctx, K=256, lr=0.01)
x = torch.rand((256, 3, 227, 227), device=dev).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, 1000, (256,), device=dev)
for it in range(8):
    F.cross_entropy(model(x), y).backward()
    sync.iteration_end()
sync.wait_all()
torch.cuda.synchronize()
report("in-step (DWBP, beside the conv backward)", *stamps())
ks = [ctx.layer_stats(0, a)["kernel_ms"] for a in range(5)]
print(f"in-step fc6 K1 event time (layer stats, 5 iterations): {[round(k * 1e3, 1) for k in ks]} us")
# alone
P, K, M, N = 1, 256, 4096, 9216
Ug = torch.randn(P, M, K, device=dev) * 0.01
Vg = torch.randn(P, N, K, device=dev).relu()
W = torch.zeros(M, N, device=dev)
for _ in range(3):
    torch.cuda._sleep(1_000_000)
    pz.reconstruct_sgd(Ug, Vg, P, K, K, M, N, W, -1e-3)
torch.cuda.synchronize()
report("alone", *stamps())
ctx.close()
