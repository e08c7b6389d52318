"""K1 A/B (round 2): time the reconstruct+SGD kernel on the bench's shapes and print a digest of the updated W,
so configurations selected by the POSEIDON_K1_* knobs (read once per process) can be compared for speed and
for bit-identical results.  One process per configuration:

    POSEIDON_K1_RW=0 python tools/k1_ab.py      # round-1 TMA W ring
    POSEIDON_K1_RWD=3 python tools/k1_ab.py     # RW epilogue, 3 chunks in flight
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402
from paper_1512_06216_b200 import binding as B  # noqa: E402

HBM = 6458.7e9


def timeit(fn, iters=30, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(200_000)  # queue the launch before the GPU reaches s
        s.record(); fn(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


MN = os.environ.get("K1_AB_MN") == "1"   # MN-major operands (poseidon_reconstruct_sgd_mn)
tag = ("MN " if MN else "") + " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("POSEIDON_K1")) or "default"
SHAPES = [(4096, 9216, 256, 1), (4096, 9216, 256, 2), (4096, 9216, 256, 4), (4096, 4096, 256, 1),
          (1000, 4096, 256, 1), (1000, 4100, 37, 3), (21841, 4096, 256, 4), (4096, 9216, 256, 8)]
for (M, N, K, P) in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(1234 + M + N + K + P)
    ldk = (K + 3) // 4 * 4
    Ug = torch.randn(P, M, ldk, device="cuda", generator=g) * 0.01
    Vg = torch.randn(P, N, ldk, device="cuda", generator=g).relu()
    W0 = torch.randn(M, N, device="cuda", generator=g)
    W = W0.clone()
    if MN:   # the same factors in the layer's own layout: U [P][K][Mp], V [P][K][N]
        Mp = (M + 3) // 4 * 4
        Um = torch.zeros(P, K, Mp, device="cuda")
        Um[:, :, :M] = Ug[:, :, :K].transpose(1, 2)
        Vm = Vg[:, :, :K].transpose(1, 2).contiguous()
        run = lambda: B.reconstruct_sgd_mn(Um, Vm, P, K, M, N, W, -1e-3)  # noqa: E731
    else:
        run = lambda: pz.reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, W, -1e-3)  # noqa: E731
    run()   # one update for the digest
    torch.cuda.synchronize()
    dig = hashlib.sha1(W.cpu().numpy().tobytes()).hexdigest()[:12]
    ms = timeit(run)
    flops = 2.0 * M * N * K * P
    byts = 8.0 * M * N + 4.0 * P * K * (M + N)
    print(f"[{tag}] M={M} N={N} K={K} P={P}: {ms * 1e3:7.1f} us  {flops / ms / 1e9:6.1f} TFLOP/s  "
          f"{byts / ms / 1e6:6.0f} GB/s ({byts / ms / 1e3 / HBM * 1e3 * 100:.0f}% HBM)  W digest {dig}", flush=True)
    del Ug, Vg, W0, W
