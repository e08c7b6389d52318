"""Debug harness for K1 (tcgen05): dumps smem stage 0 and the raw accumulator of tile 0."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1512_06216_b200 import binding as B  # noqa: E402

f = B.lib.poseidon_debug_recon_tcgen05
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
              ctypes.c_int64, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]

M, N, rows = 128, 256, 32
g = np.random.default_rng(0)
for name, U, V in [("ones", np.ones((rows, M), np.float32), np.ones((rows, N), np.float32)),
                   ("ints", g.integers(-3, 4, (rows, M)).astype(np.float32),
                    g.integers(0, 4, (rows, N)).astype(np.float32))]:
    Ud, Vd = torch.from_numpy(U).cuda(), torch.from_numpy(V).cuda()
    W = torch.zeros(M, N, device="cuda")
    dbg = torch.full((48 * 1024 // 4 + M * N,), -7.0, device="cuda")
    rc = f(Ud.data_ptr(), M, Vd.data_ptr(), N, rows, M, N, W.data_ptr(), 1.0, dbg.data_ptr())
    d = dbg.cpu().numpy()
    stage = d[:12288]
    acc = d[12288:].reshape(M, N)
    ref = U.T.astype(np.float64) @ V.astype(np.float64)
    print(name, "rc", rc, "W err", np.abs(W.cpu().numpy() - ref).max(), "W[0,:4]", W.cpu().numpy()[0, :4],
          "ref[0,:4]", ref[0, :4])
    print("  stage A first 8", stage[:8], "A nonzero", np.count_nonzero(stage[:4096]), "B nonzero",
          np.count_nonzero(stage[4096:]))
    print("  acc[0,:8]", acc[0, :8], "acc[5,:8]", acc[5, :8], "acc max", np.abs(acc).max())
    print("  acc==ref", np.abs(acc - ref).max())
    # try to find a transposition / permutation hint
    if np.abs(acc - ref).max() > 0:
        print("  acc vs ref.T-ish? shapes", acc.shape, "acc sum", acc.sum(), "ref sum", ref.sum())
