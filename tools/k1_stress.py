"""Stress K1 (2-SM tcgen05) concurrently with cuBLAS GEMMs on another stream; checks every result."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1512_06216_b200 as pz  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = True
side = torch.cuda.Stream()
a = torch.randn(4096, 4096, device="cuda")
shapes = [(4096, 9216, 256, 1), (1000, 4096, 256, 1), (4096, 4096, 256, 2), (640, 512, 64, 4), (21841, 4096, 32, 1)]
bufs = []
for (M, N, K, P) in shapes:
    ldk = (K + 3) // 4 * 4
    U = torch.randint(-3, 4, (P, M, ldk), device="cuda").float()
    V = torch.randint(0, 4, (P, N, ldk), device="cuda").float()
    U[:, :, K:] = 0
    V[:, :, K:] = 0
    ref = torch.einsum("pmk,pnk->mn", U.double(), V.double()).float()
    bufs.append((M, N, K, P, ldk, U, V, ref))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for it in range(iters):
    with torch.cuda.stream(side):
        for _ in range(3):
            a = a @ a * 1e-3
    for (M, N, K, P, ldk, U, V, ref) in bufs:
        W = torch.zeros(M, N, device="cuda")
        pz.reconstruct_sgd(U, V, P, K, ldk, M, N, W, 1.0)
        if it % 20 == 0:
            torch.cuda.synchronize()
            assert torch.equal(W, ref), (it, M, N, K, P)
torch.cuda.synchronize()
print("K1 stress ok", iters)
