"""Run K1 on one shape a few times (for ncu).  python tools/k1_run.py M N K P [iters] [recon]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1512_06216_b200 as pz  # noqa: E402

M, N, K, P = (int(a) for a in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
ldk = (K + 3) // 4 * 4
Ug = torch.randn(P, M, ldk, device="cuda") * 0.01
Vg = torch.randn(P, N, ldk, device="cuda").relu()
W = torch.randn(M, N, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(iters):
    torch.cuda._sleep(200_000)  # queue the launch before the GPU reaches s (device time, not host latency)
    s.record()
    pz.reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, W, -1e-3)
    e.record()
    e.synchronize()
    ts.append(s.elapsed_time(e))
ms = sorted(ts[1:] or ts)[len(ts[1:] or ts) // 2]  # median after the first launch
print(f"K1 M={M} N={N} K={K} P={P}: {ms*1e3:.1f} us  {2*M*N*K*P/ms/1e9:.1f} TFLOP/s  "
      f"{(8*M*N + 4*P*ldk*(M+N))/ms/1e6:.1f} GB/s")
