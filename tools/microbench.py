"""Quick K1/K2 microbenchmarks with CUDA events (not the bench contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1512_06216_b200 as pz  # noqa: E402
from paper_1512_06216_b200 import binding as B  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(200_000)  # queue the launch before the GPU reaches s (device time, not host latency)
        s.record(); fn(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


HBM = 6543.7e9
for (M, N, K, P) in [(4096, 9216, 256, 1), (4096, 9216, 256, 2), (4096, 9216, 256, 4), (4096, 9216, 256, 8),
                     (4096, 4096, 256, 8), (1000, 4096, 256, 1), (21841, 4096, 256, 8), (8192, 8192, 1024, 8)]:
    ldk = (K + 3) // 4 * 4
    Ug = torch.randn(P, M, ldk, device="cuda") * 0.01
    Vg = torch.randn(P, N, ldk, device="cuda").relu()
    W = torch.randn(M, N, device="cuda")
    for recon, name in ((pz.RECON_TF32, "K1 tcgen05"), (pz.RECON_FP32, "K1r simt")):
        if recon == pz.RECON_FP32 and P > 2:
            continue
        ms = timeit(lambda: pz.reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, W, -1e-3, recon=recon))
        flops = 2.0 * M * N * K * P
        byts = 8.0 * M * N + 4.0 * P * K * (M + N)
        print(f"{name:11s} M={M} N={N} K={K} P={P}: {ms*1e3:8.1f} us  {flops/ms/1e9:8.1f} TFLOP/s  "
              f"{byts/ms/1e6:8.1f} GB/s ({byts/ms/1e6/HBM*1e9*1e-3*1e-3*1e3:.0f}%HBM)  AI={flops/byts:.0f}")
    # torch TF32 reference for the same GEMM (library, context only)
    torch.backends.cuda.matmul.allow_tf32 = True
    A = Ug.permute(1, 0, 2).reshape(M, P * ldk)
    Bm = Vg.permute(1, 0, 2).reshape(N, P * ldk)
    ms = timeit(lambda: W.addmm_(A, Bm.t(), alpha=-1e-3))
    print(f"{'torch addmm':11s} tf32: {ms*1e3:8.1f} us  {2.0*M*N*K*P/ms/1e9:8.1f} TFLOP/s")
    del Ug, Vg, W, A, Bm

n = 37_748_736
g = torch.randn(n, device="cuda"); W = torch.randn(n, device="cuda")
ms = timeit(lambda: pz.ps_shard_update(g, W, n, -1e-3))
print(f"K2 n={n}: {ms*1e3:.1f} us  {12*n/ms/1e6:.1f} GB/s")
ms = timeit(lambda: W.add_(g, alpha=-1e-3))
print(f"torch add_ n={n}: {ms*1e3:.1f} us  {12*n/ms/1e6:.1f} GB/s")
