"""K3 (factor pack) alone: C3's three SFB layers at K = 256 (+ C5's fc8), CUDA events with the launch queued
behind a device spin, median of 20; algorithmic bytes = 8 B per packed element + 4 B per column sum."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1512_06216_b200 as pz  # noqa: E402

HBM = 6543.7e9


def timeit(fn, iters=21):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(2_000_000)
        s.record(); fn(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts[1:])


total_us, total_b = 0.0, 0.0
for name, M, N, K in [("fc6", 4096, 9216, 256), ("fc7", 4096, 4096, 256), ("fc8", 1000, 4096, 256),
                      ("i22k fc8", 21841, 4096, 256), ("fc6 K=2048", 4096, 9216, 2048)]:
    U = torch.randn(K, M, device="cuda")
    V = torch.randn(K, N, device="cuda").relu()
    ud = torch.zeros(M, K, device="cuda")
    vd = torch.zeros(N, K, device="cuda")
    cs = torch.zeros(M, device="cuda")
    ms = timeit(lambda: pz.pack_factors(U, V, K, K, ud, vd, cs))
    b = 8.0 * K * (M + N) + 4.0 * M
    if name in ("fc6", "fc7", "fc8"):
        total_us += ms * 1e3
        total_b += b
    print(f"K3 {name:10s} M={M:5d} N={N:5d} K={K:4d}: {ms*1e3:7.2f} us  {b/ms/1e6:8.1f} GB/s  {b/ms/1e6/HBM*1e3:.2f} of HBM")
    # copy of the same bytes for reference (torch, contiguous)
    ms_c = timeit(lambda: (ud.view(-1)[:K * M].copy_(U.view(-1)), vd.view(-1)[:K * N].copy_(V.view(-1))))
    print(f"   torch copy of the same bytes: {ms_c*1e3:7.2f} us")
print(f"K3 C3 step (fc6+fc7+fc8): {total_us:.2f} us, {total_b/total_us/1e3:.1f} GB/s = {total_b/total_us/1e3/HBM*1e9*1e-6:.2f} of HBM")
