"""Multi-GPU parity (NCCL over NVLink) — runs tests/mp_sync_check.py under
torchrun on every visible GPU (needs >= 2; skipped otherwise)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_multi_gpu_sync(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29611 + nproc),
           os.path.join(ROOT, "tests", "mp_sync_check.py")]
    # every check creates its own communicators; NCCL bring-up grows with the rank count
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300 + 150 * nproc, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for rank in range(nproc):
        assert f"MP_OK {rank}" in out, out[-4000:]


@pytest.mark.parametrize("nproc", [2, 4])
def test_multi_gpu_bcast_grid_cap_of_more_than_4_ranks(nproc):
    """The factor broadcast kernel's grid cap for > 4 ranks (64 CTAs) exercised at the GPU count at hand:
    checks 1b + 9 of mp_sync_check with POSEIDON_SFB_BCAST_GRID=64."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29631 + nproc),
           os.path.join(ROOT, "tests", "mp_sync_check.py"), "--wire-only"]
    env = dict(os.environ, POSEIDON_SFB_BCAST_GRID="64")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for rank in range(nproc):
        assert f"MP_OK {rank}" in out, out[-4000:]
