"""CPU tests of bench.py's reference arm (the fp64 oracle, `--impl reference`): the JSON line the driver
parses, its config identical to the one the GPU arm prints, and the torchrun contract (only rank 0 works and
prints).  C2 keeps the oracle step to milliseconds; the GPU arm's line is checked on the GPU
(`tests/test_gpu_bench_path.py`)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=240):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "C2", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "images/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 1 and d["dtype"] == "f64"
    assert d["ms_per_step"] > 0 and abs(d["value"] - 100 / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2 ") and d["config"]["global_batch"] == 100


def test_reference_arm_config_matches_gpu_arm():
    """Both arms print workload_config(args, cfg, P): the driver divides the two values only if they name the
    same workload."""
    sys.path.insert(0, ROOT)
    try:
        import bench
        from drivers.cnn import CONFIGS
    finally:
        sys.path.remove(ROOT)
    old = sys.argv
    try:
        sys.argv = ["bench.py", "--config", "C3", "--gpus", "4", "--ssp", "2"]
        a = bench.parse()
    finally:
        sys.argv = old
    c = bench.workload_config(a, CONFIGS["C3"], 4)
    assert c["global_batch"] == 4 * CONFIGS["C3"]["batch"] and c["parallelism"] == "dp4"
    assert "SSP staleness 2" in c["workload"]


def test_reference_arm_nonzero_ranks_exit_quietly():
    """Under torchrun only rank 0 runs the oracle and prints; the other ranks exit 0 without work."""
    r = _run(["--impl", "reference", "--config", "C2", "--gpus", "2", "--steps", "1", "--warmup", "0"],
             env_extra={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
