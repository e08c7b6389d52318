"""f2 probe (round 2): what would splitting K1 around the factor exchange buy?  ("f2 AG+K1").

The SFB sync of a layer at P ranks is exchange -> K1 over all P factor blocks.  The split alternative starts K1
on the rank's own block while the other P-1 blocks travel, then runs K1 on those:
    serial  = t_exchange + K1(P blocks)
    split   = max(t_exchange, K1(1 block)) + K1(P-1 blocks)
One GPU can time the three K1 launches (the exchange times are the measured ones of profiles/r2/collectives_r2.md,
library broadcast kernel, K = 256); the split's second W read-modify-write is inside K1(1) + K1(P-1) - K1(P).
Run:  python tools/k1_split_probe.py   (one GPU; prints one line per layer and P)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402

# measured factor exchange (broadcast kernel, ms), profiles/r2/collectives_r2.md
EXCHANGE_MS = {("fc6", 2): 0.043, ("fc6", 4): 0.084, ("fc7", 2): 0.033, ("fc7", 4): 0.059,
               ("i22k_fc8", 2): 0.061, ("i22k_fc8", 4): 0.145}
LAYERS = [("fc6", 4096, 9216), ("fc7", 4096, 4096), ("i22k_fc8", 21841, 4096)]
K = 256


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(200_000)   # queue the launches before the GPU reaches s
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for name, M, N in LAYERS:
    for P in (2, 4, 8):
        g = torch.Generator(device="cuda").manual_seed(M + N + P)
        Ug = torch.randn(P, M, K, device="cuda", generator=g) * 0.01
        Vg = torch.randn(P, N, K, device="cuda", generator=g).relu()
        W = torch.randn(M, N, device="cuda", generator=g)
        full = timeit(lambda: pz.reconstruct_sgd(Ug, Vg, P, K, K, M, N, W, -1e-4))
        local = timeit(lambda: pz.reconstruct_sgd(Ug[:1], Vg[:1], 1, K, K, M, N, W, -1e-4))
        rest = timeit(lambda: pz.reconstruct_sgd(Ug[1:], Vg[1:], P - 1, K, K, M, N, W, -1e-4))
        both = timeit(lambda: (pz.reconstruct_sgd(Ug[:1], Vg[:1], 1, K, K, M, N, W, -1e-4),
                               pz.reconstruct_sgd(Ug[1:], Vg[1:], P - 1, K, K, M, N, W, -1e-4)))
        ex = EXCHANGE_MS.get((name, P))
        line = (f"{name} M={M} N={N} K={K} P={P}: K1(P) {full * 1e3:6.1f} us  K1(1) {local * 1e3:6.1f}  "
                f"K1(P-1) {rest * 1e3:6.1f}  K1(1)+K1(P-1) back to back {both * 1e3:6.1f} "
                f"(split overhead {(both - full) * 1e3:+6.1f} us)")
        if ex is not None:
            serial = ex + full
            split = max(ex, local) + rest
            line += f"  | exchange {ex * 1e3:5.1f}: serial {serial * 1e3:6.1f} us, split {split * 1e3:6.1f} us"
        print(line, flush=True)
        del Ug, Vg, W
