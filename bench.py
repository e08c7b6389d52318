#!/usr/bin/env python
"""Poseidon-on-B200 benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --impl reference ...                     (fp64 CPU oracle arm)

A step is one synchronous data-parallel training iteration of the config's CNN
on synthetic data: forward, backward with DWBP (each layer's sync — SACP's SFB
all-gather + tcgen05 reconstruct+SGD, or PS reduce-scatter + K2 + all-gather —
launched by the library as soon as the layer's backward is done), and the
next-forward barrier.  The optimiser step IS the sync (Alg. 1/3).  Metric
(BASELINE.json): images/sec (whole job), plus exposed sync ms/iter and the
roofline fraction of the dominant sync kernel.  Default config C3 (AlexNet,
batch 256/GPU): the config the north-star target is stated on and the only
one that exercises every hot-path step (SFB on FC + PS on conv + DWBP).
Defaults at N > 1: PS layers sync with the fused NVLink-SHARP kernel, SFB
factors move through the library's broadcast kernel, and SFB layer inputs are
broadcast at forward time (early V); every option has a flag to A/B it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="poseidon", choices=["poseidon", "reference"])
    ap.add_argument("--scheme", default=None, choices=[None, "auto", "ps", "sfb", "sfps"])
    ap.add_argument("--early-v", default="auto", choices=["auto", "on", "off"],
                    help="broadcast SFB layer inputs at forward time (POSEIDON_FLAG_EARLY_V); auto = on when N > 1 "
                         "(profiles/early_v_r1.md: summed sync -25%%, exposed sync -40%%, images/s unchanged)")
    ap.add_argument("--else-branch", default="ps", choices=["ps", "sfps"],
                    help="how FC layers the SACP rule sends to the server execute: full-gradient PS (reading Z7) "
                         "or the literal sharded SF-PS of Alg. 3 (reading Z20, POSEIDON_FLAG_SFPS)")
    ap.add_argument("--factors", default="auto", choices=["auto", "async", "mn", "pack"],
                    help="where the SFB factors are read: async = POSEIDON_FLAG_INPLACE_FACTORS (K3 on the library's "
                         "stream, off the backward's); mn = + POSEIDON_FLAG_INPLACE_MN (N = 1: K1 reads them MN-major, "
                         "no K3); pack = K3 on the backward's stream (round 1); auto = mn at N = 1 "
                         "(profiles/r2/factors_r2.md: +1%% images/s), pack at N > 1")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="capture one training step (forward, backward with every layer's DWBP sync, iteration_end) "
                         "in a CUDA graph after the warm-up and replay it per step; auto = on for C2 (host-bound: "
                         "2.4x) and at N > 1 (+1.3-1.9%%); off for C3-C5 at N = 1, where the replay packs K1 deeper "
                         "into the conv backward (in-step fraction 0.66 -> 0.48-0.60 for +1.3%%; DESIGN §6d)")
    ap.add_argument("--dwbp", default="on", choices=["on", "off"])
    ap.add_argument("--recon", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--nvls", default="auto", choices=["auto", "on", "off"],
                    help="fused one-kernel NVLink-SHARP PS sync (f1); auto = on when N > 1")
    ap.add_argument("--sfb-wire", default="auto", choices=["auto", "nccl", "symm", "nvls"],
                    help="SFB factor broadcast: NCCL all-gather on plain buffers, on NCCL symmetric windows, "
                         "or the library's broadcast kernel on symmetric windows (peer stores over NVLink; "
                         "POSEIDON_SFB_BCAST=mc for the multicast variant); auto = nvls when N > 1")
    ap.add_argument("--ssp", type=int, default=0, choices=[0, 1, 2, 3, 4, 5],
                    help="staleness s of the SSP consistency model (P:L399-402, E11); 0 = BSP (the paper's "
                         "headline setting)")
    ap.add_argument("--straggle-us", type=float, default=0.0,
                    help="ablation only: every step one rank (a fixed pseudo-random sequence) is delayed by this "
                         "many microseconds on its GPU before the forward (a straggler, P:L568)")
    ap.add_argument("--bucket-kb", type=int, default=0,
                    help="sync runs of small PS layers as one bucket of at most this many KB (f1; needs the arena)")
    ap.add_argument("--override", action="append", default=[], metavar="LAYER=SCHEME",
                    help="per-layer scheme (auto/ps/sfb/sfps), e.g. fc8=ps: C3's P >= 6 schedule at fewer GPUs")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--momentum", type=float, default=0.0, help="f4: Lambda momentum (0 = plain SGD hot path)")
    ap.add_argument("--weight-decay", type=float, default=0.0, help="f4: Lambda weight decay")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-input", default="u8", choices=["u8", "f32"],
                    help="e2e: images cross PCIe as uint8 pixels (scaled to fp32 on the GPU) or as fp32")
    ap.add_argument("--memory-format", default="channels_last", choices=["channels_last", "nchw"],
                    help="driver CNN activation layout (cuDNN NHWC kernels avoid layout transposes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layer-stats", action="store_true", help="print per-layer stats to stderr")
    ap.add_argument("--cudnn-benchmark", default="on", choices=["on", "off"])
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        out = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
               "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
               "source": "measured (MEASURED_PEAKS.json)"}
    else:
        # fallback stated in /opt/skills/guides/B200_PROFILING.md
        out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    # TF32 dense peak: the larger of (a) cuBLAS TF32 8192^3 measured on a pool B200 with the MEASURED_PEAKS
    # protocol (tools/peaks.py -> profiles/peaks_r2.json: best of 10 / 4 s back to back) and (b) the measured
    # bf16 peak x the guide's nominal dense ratio 1.1 / 2.25.  (a) came out BELOW (b) and below what cuBLAS and
    # K1 reach on the FC shapes (profiles/microbench_r1.txt), so the larger denominator keeps fractions <= 1.
    d_burst = out["bf16_tflops"] * TF32_OVER_BF16
    d_sust = out["bf16_tflops_sustained"] * TF32_OVER_BF16
    out["tf32_tflops"], out["tf32_tflops_sustained"] = d_burst, d_sust
    out["tf32_source"] = f"bf16 x 1.1/2.25 (nominal ratio): {d_burst:.1f} burst / {d_sust:.1f} sustained"
    tp = os.path.join(ROOT, "profiles", "peaks_r2.json")
    if os.path.exists(tp):
        with open(tp) as f:
            t = json.load(f)
        out["tf32_tflops_measured"] = t["tf32_tflops"]
        out["tf32_tflops_sustained_measured"] = t["tf32_tflops_sustained"]
        out["tf32_tflops"] = max(d_burst, t["tf32_tflops"])
        out["tf32_tflops_sustained"] = max(d_sust, t["tf32_tflops_sustained"])
        out["tf32_source"] = (f"max(bf16 x 1.1/2.25 = {d_burst:.1f} / {d_sust:.1f}; measured cuBLAS TF32 8192^3 "
                              f"(profiles/peaks_r2.json) = {t['tf32_tflops']:.1f} / {t['tf32_tflops_sustained']:.1f}) "
                              "burst / sustained")
    return out


TF32_OVER_BF16 = 1.1 / 2.25   # nominal dense ratio (B200_PROFILING.md table)
METRIC = "images/sec (exposed sync ms/iter and % of roofline alongside)"


def workload_config(args, cfg, world):
    """The `config` object both arms print (identical for the driver's ratio)."""
    consistency = "" if not getattr(args, "ssp", 0) else f", SSP staleness {args.ssp}"
    return {"workload": f"{args.config} {cfg['name']} data-parallel training step with Poseidon sync "
                        f"(SACP + DWBP{consistency}), synthetic data",
            "global_batch": world * cfg["batch"], "per_gpu_batch": cfg["batch"],
            "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (C3: images 158 MB + weights 244 MB per step)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------- oracle arm ----
def oracle_step_seconds(config: str, P: int, budget_s: float):
    """Time the fp64 oracle's synchronous step (O4 for SFB layers, O6 for PS
    layers) for one iteration of `config` at P workers on a bounded sample:
    each SFB layer is timed on its first R output rows (R sized to the budget)
    and scaled by M/R (each output row is independent work of equal size).
    Returns (seconds per full iteration, sample description, threads)."""
    import numpy as np

    import oracle as O
    import synthetic as S
    from drivers.cnn import CONFIGS
    import torch.nn as nn

    cfg = CONFIGS[config]
    K = cfg["batch"]
    with_meta = __import__("torch").device("meta")
    with with_meta:
        model = cfg["model"]()
    layers = []
    for name, m in model.named_modules():
        if isinstance(m, nn.Linear):
            layers.append((name, O.LAYER_FC, m.out_features, m.in_features, True))
        elif isinstance(m, nn.Conv2d):
            layers.append((name, O.LAYER_CONV, m.out_channels, m.weight[0].numel(), m.bias is not None))
    scheme_mode = cfg["scheme"]
    total = 0.0
    desc = []
    flops_budget = 2.0e9 * budget_s  # ~2 GFLOP/s/thread-ish fp64 BLAS is conservative; refined below
    for (name, kind, M, N, has_b) in layers:
        sch = O.choose_scheme(kind, M, N, K, P)
        if scheme_mode == "ps":
            sch = O.SCHEME_PS
        if sch == O.SCHEME_SFB:
            rows = max(1, min(M, int(flops_budget / max(1.0, 2.0 * N * K * P))))
            W = np.zeros((rows, N), np.float32)
            b = np.zeros(rows, np.float32)
            Us = [np.asarray(S.rng(p).standard_normal((K, rows)), np.float32) for p in range(P)]
            Vs = [np.asarray(S.rng(100 + p).standard_normal((K, N)), np.float32) for p in range(P)]
            t0 = time.perf_counter()
            O.sync_step(W, b, Us, Vs, 0.01)
            dt = time.perf_counter() - t0
            total += dt * (M / rows)
            desc.append(f"{name}:SFB O4 rows {rows}/{M}")
        else:
            n = M * N + (M if has_b else 0)
            grads = [np.zeros(n, np.float32) for _ in range(P)]
            w = np.zeros(n, np.float32)
            t0 = time.perf_counter()
            O.ps_step_flat(w, grads, 0.01)
            total += time.perf_counter() - t0
            desc.append(f"{name}:PS O6 n={n}")
    try:
        from threadpoolctl import threadpool_info
        threads = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count() or 1
    return total, "; ".join(desc), threads


def c1_step(pz, dev):
    """BASELINE.json config C1: one FC layer M=128 (out), N=256 (in), K=8, P=2 simulated workers, one
    synchronous SGD step, SFB (TF32 K1 and fp32 K1r) and PS on the GPU (CUDA events, median of 50, each
    launch after a device spin) beside the fp64 oracle's O4 on 1 host thread and on all threads."""
    import numpy as np
    import torch

    import oracle as O
    import synthetic as S
    from threadpoolctl import threadpool_limits

    M, N, K, P = 128, 256, 8, 2
    W, b, Us, Vs, lr = S.integer_factors(M, N, K, P, seed=1)
    Ud = torch.from_numpy(np.concatenate(Us)).to(dev)
    Vd = torch.from_numpy(np.concatenate(Vs)).to(dev)
    Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    n = M * N + M
    _, _, padded = pz.shard_range(n, P, 0)
    grads = np.zeros((P, padded), np.float32)
    for p in range(P):
        grads[p, :n] = O.flatten_params(O.reconstruct(Us[p], Vs[p]), Us[p].astype(np.float64).sum(0))
    gd = torch.from_numpy(grads).to(dev)
    wflat = torch.zeros(padded, device=dev)
    stream = torch.cuda.current_stream()

    spin = int(os.environ.get("C1_SPIN_CYCLES", "10000000"))

    def gpu_ms(fn):
        """Device time of one call: a device spin (~5 ms) lets the host enqueue the whole call (the simulated
        entry points allocate their scratch stream-ordered) before e0 fires, so the events see the GPU work."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(31):
            torch.cuda._sleep(spin)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts[1:])

    def call_ms(fn):
        """Host wall time of one call through the binding until its result is ready (what a caller waits)."""
        ts = []
        for _ in range(31):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts[1:])

    out = {"workload": "C1: FC 256->128 (M=128, N=256), K=8, P=2 simulated workers, one sync step",
           "note": "gpu_*: device time of the call; call_*: host wall time until the result is ready (the "
                   "simulated entry points are test helpers that allocate scratch per call)"}
    sfb_tf32 = lambda: pz.sfb_simulated(Ud, Vd, P, K, M, N, Wd, bd, lr, recon=pz.RECON_TF32)  # noqa: E731
    sfb_fp32 = lambda: pz.sfb_simulated(Ud, Vd, P, K, M, N, Wd, bd, lr, recon=pz.RECON_FP32)  # noqa: E731
    ps = lambda: pz.ps_simulated(gd, P, wflat, n, lr)  # noqa: E731
    for name, fn in (("sfb_tf32", sfb_tf32), ("sfb_fp32", sfb_fp32), ("ps", ps)):
        out[f"gpu_{name}_ms"] = gpu_ms(fn)
        out[f"call_{name}_ms"] = call_ms(fn)

    def cpu_ms(threads):
        with threadpool_limits(threads):
            ts = []
            for _ in range(21):
                t0 = time.perf_counter()
                O.sync_step(W, b, Us, Vs, lr)
                ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    out["oracle_1core_ms"] = cpu_ms(1)
    out["oracle_all_cores_ms"] = cpu_ms(os.cpu_count() or 1)
    out["host_cores"] = os.cpu_count()
    return out


def oracle_per_config(P: int, budget_s: float = 1.5):
    """The fp64 oracle's sync step of one iteration of every BASELINE.json network config (C2-C5) at P
    workers, each on a bounded sample (SFB layers on R rows scaled by M/R): seconds and images/s."""
    from drivers.cnn import CONFIGS
    res = {}
    for name in ("C2", "C3", "C4", "C5"):
        sec, desc, threads = oracle_step_seconds(name, P, budget_s)
        res[name] = {"seconds_per_iteration": sec, "images_per_s": P * CONFIGS[name]["batch"] / sec,
                     "cores": threads, "sample": desc}
    return res


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from drivers.cnn import CONFIGS
    cfg = CONFIGS[args.config]
    P = args.gpus
    per_step_budget = max(0.5, 150.0 / max(1, args.steps + args.warmup))
    times = []
    desc, threads = "", 1
    for i in range(args.warmup + args.steps):
        sec, desc, threads = oracle_step_seconds(args.config, P, per_step_budget)
        if i >= args.warmup:
            times.append(sec)
    sec = statistics.median(times)
    value = P * cfg["batch"] / sec
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "images/s", "n_gpus": P, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg, P),
        "reference_note": "the fp64 CPU oracle's synchronous step (O4/O6) for one iteration, images/s = "
                          "P * batch / oracle seconds; the CNN forward/backward is not part of the oracle",
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "oracle",
                         "sample": "per step: " + desc + " (SFB rows scaled by M/R)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- poseidon arm ----
def run_poseidon(args):
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    import paper_1512_06216_b200 as pz
    from paper_1512_06216_b200.dwbp import PoseidonSync
    from drivers.cnn import CONFIGS

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.benchmark = args.cudnn_benchmark == "on"
    torch.backends.cudnn.allow_tf32 = True
    torch.backends.cuda.matmul.allow_tf32 = True

    cfg = CONFIGS[args.config]
    K, hw, classes = cfg["batch"], cfg["hw"], cfg["classes"]
    scheme = args.scheme or cfg["scheme"]

    # NCCL unique id from rank 0 through torch.distributed (plumbing only)
    nccl_id = None
    if world > 1:
        obj = [pz.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    flags = pz.FLAG_DWBP_OFF if args.dwbp == "off" else 0
    use_nvls = world > 1 and args.nvls != "off"
    if use_nvls:
        flags |= pz.FLAG_NVLS_PS
    # auto at N > 1: the library's own factor broadcast (peer stores over NVLink, 32 CTAs; profiles/
    # collectives_r1.md: faster than NCCL's symmetric all-gather alone and equal or better in the step)
    sfb_wire = ("nvls" if args.sfb_wire == "auto" else args.sfb_wire) if world > 1 else "none (P=1)"
    flags |= {"symm": pz.FLAG_SYMM_SFB, "nvls": pz.FLAG_NVLS_SFB}.get(sfb_wire, 0)
    if args.ssp:
        flags |= pz.FLAG_SSP1
    if args.else_branch == "sfps":
        flags |= pz.FLAG_SFPS
    # early V: BSP with DWBP only (the library refuses it with DWBP off or SSP)
    early_v = args.early_v == "on" or (args.early_v == "auto" and world > 1 and args.dwbp == "on" and not args.ssp)
    if early_v:
        flags |= pz.FLAG_EARLY_V
    if args.factors == "auto":
        args.factors = "mn" if world == 1 else "pack"
    if args.dwbp == "off" or args.ssp:
        args.factors = "pack"   # in-place factor reads are a BSP + DWBP feature (the library ignores the flags)
    if args.factors != "pack":
        flags |= pz.FLAG_INPLACE_FACTORS
    if args.factors == "mn":
        flags |= pz.FLAG_INPLACE_MN
    # MN-major K1 on the SFB layers whose M, N are multiples of 4: in place at N = 1, on the MN-major gather
    # buffers (slot filled by a copy-engine memcpy, no K3) at N > 1
    inplace = (args.factors == "mn" and not args.ssp and args.dwbp == "on" and args.recon == "tf32")
    ctx = pz.Context(rank=rank, world=world, device=local, nccl_id=nccl_id, flags=flags)
    if args.ssp > 1:
        ctx.set_staleness(args.ssp)

    torch.manual_seed(6216)          # identical weights on every rank
    model = cfg["model"]().to(dev)
    recon = pz.RECON_TF32 if args.recon == "tf32" else pz.RECON_FP32
    if args.memory_format == "channels_last":
        model.to(memory_format=torch.channels_last)   # before PoseidonSync makes params buffer views
    sync = PoseidonSync(model, ctx, K=K, lr=args.lr, scheme=scheme, recon=recon, arena=use_nvls or bool(args.ssp) or bool(args.bucket_kb),
                        bucket_bytes=args.bucket_kb * 1024,
                        overrides=dict(o.split("=", 1) for o in args.override))
    if args.momentum or args.weight_decay:
        ctx.set_momentum(args.momentum, args.weight_decay)

    g = torch.Generator(device=dev)
    g.manual_seed(1512 + rank)
    x = torch.rand((K, 3, hw, hw), device=dev, generator=g)
    if args.memory_format == "channels_last":
        x = x.contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, classes, (K,), device=dev, generator=g)

    step_no = [0]
    straggle_cycles = int(args.straggle_us * 1965)   # ~1965 MHz SM clock under load

    def step(xb, yb):
        if straggle_cycles and world > 1:
            if (step_no[0] * 2654435761 + 12345) % 1000003 % world == rank:
                torch.cuda._sleep(straggle_cycles)
        step_no[0] += 1
        out = model(xb)
        loss = F.cross_entropy(out, yb)
        loss.backward()
        sync.iteration_end()
        return loss

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region ----
    for _ in range(args.warmup):
        step(x, y)
    sync.wait_all()
    barrier()
    use_graph = args.graph == "on" or (args.graph == "auto" and (args.config == "C2" or world > 1)
                                         and not args.ssp and not args.straggle_us and args.dwbp == "on")
    if use_graph and (args.ssp or args.straggle_us or args.dwbp == "off"):
        raise SystemExit("--graph: BSP with DWBP only (no --ssp, --straggle-us, --dwbp off)")
    run_step, graph_launches, graph_fallback = step, None, None
    if use_graph:
        # One captured step: the library sees the capture on the caller's stream, forks its comm / recon streams
        # from it, records its statistics events as graph nodes and rejoins at iteration_end, so one replay is
        # the whole iteration (Alg. 2) with no host launches; x, y are the graph's static inputs.
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        lc0 = pz.launch_count()
        try:
            with torch.cuda.graph(graph, stream=gs):
                static_loss = step(x, y)
            graph_launches = pz.launch_count() - lc0
        except Exception as exc:   # e.g. an untested topology: fall back to the eager loop, say so in the line
            graph_fallback = f"{type(exc).__name__}: {exc}"[:200]
            sys.stderr.write(f"bench: CUDA-graph capture failed, eager steps instead ({graph_fallback})\n")
            use_graph = False
        torch.cuda.current_stream().wait_stream(gs)
        if world > 1:   # every rank replays, or none does
            ok = torch.tensor([1.0 if use_graph else 0.0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if use_graph and float(ok) < 1.0:
                graph_fallback = graph_fallback or "another rank's capture failed"
                use_graph = False
        if not use_graph:
            del graph
            sync.wait_all()
            barrier()

    if use_graph:
        def run_step(xb, yb):
            if xb is not x:
                x.copy_(xb, non_blocking=True)
            if yb is not y:
                y.copy_(yb, non_blocking=True)
            graph.replay()
            return static_loss

        for _ in range(2):
            run_step(x, y)
        sync.wait_all()
        barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.25)  # let the sampler start
    l0 = pz.launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # process-wide start/end range (the backward and the library hooks run on autograd's thread):
    # ncu --nvtx --nvtx-include "timed" selects exactly the timed launches
    nvtx_id = torch.cuda.nvtx.range_start("timed")
    ev0.record(stream)
    for _ in range(args.steps):
        run_step(x, y)
    sync.wait_all()
    ev1.record(stream)
    torch.cuda.nvtx.range_end(nvtx_id)
    ev1.synchronize()
    # graph mode: the host launches nothing per step; every replay runs the captured launches
    launches = pz.launch_count() - l0 if graph_launches is None else graph_launches * args.steps
    clk = clocks.stop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    images = world * K * args.steps
    value = images / (ms / 1e3)

    # per-iteration sync statistics (device events kept by the library)
    n_stats = 1 if use_graph else min(args.steps, 7)   # graph: the captured iteration's events (last replay)
    its = [ctx.iter_stats(a) for a in range(n_stats)]
    exposed = statistics.mean(i["exposed_ms"] for i in its)
    sync_total = statistics.mean(i["sync_total_ms"] for i in its)
    nccl_sent = its[0]["nccl_bytes_sent"]
    nccl_recv = its[0]["nccl_bytes_recv"]
    if world > 1:
        t = torch.tensor([exposed, sync_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        exposed, sync_total = float(t[0]), float(t[1])

    # dominant sync kernel: the largest SFB layer's K1 (else the largest PS layer's K2)
    sfb = [p for p in sync.plans if p.scheme == pz.SCHEME_SFB]
    peaks = measured_peaks()
    roof = None
    if sfb:
        top = max(sfb, key=lambda p: p.M * p.N)
        kms = statistics.mean(ctx.layer_stats(top.layer_id, a)["kernel_ms"] for a in range(n_stats))
        M, N, Kf, P = top.M, top.N, top.K, world
        top_inplace = inplace and M % 4 == 0 and N % 4 == 0   # else the library packed this layer (K-major)
        ldk = Kf if top_inplace else (Kf + 3) // 4 * 4
        flops = 2.0 * M * N * Kf * P
        byts = 8.0 * M * N + 4.0 * P * ldk * (M + N)
        tf32_peak = peaks["tf32_tflops_sustained"]
        ridge = tf32_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
        if flops / byts >= ridge:
            ach = flops / (kms / 1e3) / 1e12
            roof = {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": ach / tf32_peak}
        else:
            ach = byts / (kms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / peaks["hbm_gbs"]}
        roof.update({"kernel": f"K1 recon_tcgen05 ({top.name} {M}x{N}, P*K={P * Kf})" if args.recon == "tf32"
                     else f"K1r recon_simt ({top.name})", "kernel_ms": kms,
                     "algorithmic_flops": flops, "algorithmic_bytes": byts,
                     "peak_source": f"hbm: {peaks['source']}; tf32 (sustained): {peaks['tf32_source']}"})
        if args.recon == "tf32":
            # context for `frac` (which is the in-step number): the same K1 launch on the same shape ALONE,
            # after the timed region, each launch queued behind a device spin (device time only)
            if top_inplace:   # the factors as the layers leave them: U [P][K][M], V [P][K][N] (MN-major K1)
                Ug = torch.randn(P, Kf, M, device=dev).mul_(0.01)
                Vg = torch.randn(P, Kf, N, device=dev).relu_()
            else:
                Ug = torch.randn(P, M, ldk, device=dev).mul_(0.01)
                Vg = torch.randn(P, N, ldk, device=dev).relu_()
            Wt = torch.zeros(M, N, device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(6):
                torch.cuda._sleep(200_000)
                e0.record(stream)
                if top_inplace:
                    pz.reconstruct_sgd_mn(Ug, Vg, P, Kf, M, N, Wt, -1e-3, stream=stream)
                else:
                    pz.reconstruct_sgd(Ug, Vg, P, Kf, ldk, M, N, Wt, -1e-3, stream=stream)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            iso = statistics.median(ts[1:])
            iso_ach = (flops / (iso / 1e3) / 1e12) if roof["bound"] == "tensor" else (byts / (iso / 1e3) / 1e9)
            roof.update({"isolated_kernel_ms": iso, "isolated_frac": iso_ach / roof["peak"],
                         "isolated_note": "same K1 launch alone after the timed region (not part of value); "
                                          "frac is the in-step number, where DWBP runs K1 beside the backward"})
            del Ug, Vg, Wt
    else:
        top = max(sync.plans, key=lambda p: p.n)
        kms = statistics.mean(ctx.layer_stats(top.layer_id, a)["kernel_ms"] for a in range(n_stats))
        b0, e0, _ = pz.shard_range(top.n, world, rank)
        byts = 12.0 * (e0 - b0)
        ach = byts / (kms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "kernel": f"K2 ps_shard_sgd ({top.name})", "kernel_ms": kms,
                "algorithmic_bytes": byts, "peak_source": peaks["source"]}
    # K3 (factor pack) of every SFB layer, summed per step: 8 B per packed element (read + write) plus the
    # column sums; timed by the library's events on the producer stream (layer stats pack_ms)
    packed_layers = [p for p in sfb if not (inplace and p.M % 4 == 0 and p.N % 4 == 0)]
    if sfb and not packed_layers:
        roof["pack"] = {"kernel": ("none: factors read in place by K1 (POSEIDON_FLAG_INPLACE_MN, N = 1)" if world == 1
                                   else "none: copy-engine memcpy of the factors into the MN-major gather slot "
                                        "(POSEIDON_FLAG_INPLACE_MN, N > 1)"),
                        "ms_per_step": 0.0, "algorithmic_bytes": 0.0, "achieved": None, "unit": "GB/s", "frac": None,
                        "note": "K1 consumes dl/dy and a_i MN-major where the backward wrote them; its idle lanes form "
                                "the bias sums (4 K M B of extra reads per SFB layer, not counted as algorithmic)"}
    elif sfb:
        pk_ms, pk_bytes = 0.0, 0.0
        for p in packed_layers:
            pk_ms += statistics.mean(ctx.layer_stats(p.layer_id, a)["pack_ms"] for a in range(n_stats))
            cols = p.M + (0 if early_v else p.N)
            pk_bytes += 8.0 * p.K * cols + 4.0 * p.M
        ach = pk_bytes / (pk_ms / 1e3) / 1e9 if pk_ms > 0 else None
        roof["pack"] = {"kernel": "K3 pack_uv (all SFB layers of one step)", "ms_per_step": pk_ms,
                        "algorithmic_bytes": pk_bytes, "achieved": ach, "unit": "GB/s",
                        "frac": (ach / peaks["hbm_gbs"]) if ach else None,
                        "note": ("in-step, on the library's sync stream (POSEIDON_FLAG_INPLACE_FACTORS)"
                                 if args.factors == "async" else "in-step, on the compute stream")
                                + "; V packed at forward time when early_v"
                                + ("; layers packed: " + ", ".join(p.name for p in packed_layers)
                                   + " (M or N not a multiple of 4: no in-place K1)" if inplace else "")}
    roof["traffic"] = None
    tr_path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tr_path):
        try:
            with open(tr_path) as f:
                tr = json.load(f)
            key = f"{args.config}_P{world}"
            if key in tr:
                roof["traffic"] = tr[key]
        except Exception:
            pass

    if args.layer_stats and rank == 0:
        for p in sync.plans:
            sys.stderr.write(json.dumps({"layer": p.name, **ctx.layer_stats(p.layer_id, 0)}) + "\n")

    # ---- end to end: pinned host batch -> device each step, loss back to host ----
    e2e = None
    if not args.no_e2e:
        # End to end through the public API: every step copies its batch from pinned host memory
        # (on a copy stream, double-buffered, so step t+1's copy overlaps step t's compute) and
        # reads its loss back to pinned host memory (the read of step t completes during step t+1).
        # The images travel as 8-bit pixels (--e2e-input u8, what an image pipeline delivers; 4x fewer PCIe
        # bytes than fp32) and are scaled to [0, 1) fp32 on the GPU in the step's stream; f32 ships them as fp32.
        u8 = args.e2e_input == "u8"
        if u8:
            xq = (x * 255.0).to(torch.uint8)
            xh = [xq.cpu().pin_memory(), xq.cpu().pin_memory()]
        else:
            xh = [x.cpu().pin_memory(), (x.cpu() + 0.0).pin_memory()]
        yh = [y.cpu().pin_memory(), y.cpu().pin_memory()]
        xd = [torch.empty_like(xh[0], device=dev), torch.empty_like(xh[0], device=dev)]
        yd = [torch.empty_like(y), torch.empty_like(y)]
        xf = x if use_graph else torch.empty_like(x)   # the step's fp32 input (u8 path; the graph's own input)
        loss_h = torch.empty(args.steps + 4, dtype=torch.float32).pin_memory()
        copy_stream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(i):
            b = i % 2
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[b])        # step i-2 finished with this buffer
                xd[b].copy_(xh[b], non_blocking=True)
                yd[b].copy_(yh[b], non_blocking=True)
                copied[b].record(copy_stream)

        def e2e_steps(n, base):
            h2d(0)
            for i in range(n):
                b = i % 2
                stream.wait_event(copied[b])
                if u8:
                    torch.mul(xd[b], 1.0 / 255.0, out=xf)
                    loss = run_step(xf, yd[b])
                else:
                    loss = run_step(xd[b], yd[b])
                consumed[b].record(stream)
                if i + 1 < n:
                    h2d(i + 1)
                loss_h[base + i].copy_(loss.detach(), non_blocking=True)

        e2e_steps(2, 0)
        sync.wait_all()
        barrier()
        ev0.record(stream)
        e2e_steps(args.steps, 2)
        sync.wait_all()
        ev1.record(stream)
        ev1.synchronize()
        ms_e = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms_e], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e = float(t.item())
        loss_val = float(loss_h[args.steps + 1])
        e2e = {"value": images / (ms_e / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": int(xh[0].numel() * xh[0].element_size() + yh[0].numel() * 8),
               "d2h_bytes_per_step": 4, "ms_per_step": ms_e / args.steps, "last_loss": loss_val,
               "input": "uint8 pixels, scaled on the GPU" if u8 else "fp32",
               "note": "pinned H2D of each step's batch on a copy stream (double-buffered, overlaps the "
                       "previous step), loss D2H every step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # repeat the bounded sample until ~10 s of CPU work, report the median iteration
        secs, t_start = [], time.perf_counter()
        while time.perf_counter() - t_start < 10.0 or len(secs) < 3:
            sec_i, desc, threads = oracle_step_seconds(args.config, world, 12.0)
            secs.append(sec_i)
            if len(secs) >= 50:
                break
        sec = statistics.median(secs)
        cpu = {"value": world * K / sec, "unit": "images/s", "cores": threads, "kind": "oracle",
               "sample": f"fp64 oracle sync step of one {args.config} iteration at P={world}, median of "
                         f"{len(secs)} repetitions ({time.perf_counter() - t_start:.1f} s CPU wall): {desc} "
                         "(SFB layers timed on R rows, scaled by M/R)",
               "seconds_per_iteration": sec}
        try:
            cpu["per_config"] = oracle_per_config(world)
            cpu["c1"] = c1_step(pz, dev)
        except Exception as e:   # the extra oracle legs are context, never fatal to the bench line
            cpu["per_config_error"] = repr(e)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "tf32" if args.recon == "tf32" else "f32", "data": "synthetic",
            "config": workload_config(args, cfg, world),
            "details": {"scheme": scheme, "else_branch": args.else_branch, "early_v": early_v, "factors": args.factors, "cuda_graph": use_graph, "graph_fallback": graph_fallback, "inplace_mn_k1": inplace, "dwbp": args.dwbp, "recon": args.recon, "lr": args.lr,
                        "momentum": args.momentum, "weight_decay": args.weight_decay,
                        "memory_format": args.memory_format,
                        "ps_path": ("nvls-fused" if sync.nvls_active else
                                    ("nccl rs/k2/ag" if world > 1 else "k2 (P=1)")),
                        "nvls_status": ctx.nvls_status(),
                        "sfb_wire": sfb_wire, "ssp": args.ssp, "straggle_us": args.straggle_us,
                        "bucket_kb": args.bucket_kb, "overrides": args.override,
                        "sfb_paths": sorted({ctx.sfb_path(d["id"]) for d in sync.describe()
                                             if d["scheme"] == "SFB"}) if world > 1 else []},
            "exposed_sync_ms": exposed, "sync_total_ms": sync_total,
            "exposed_frac": (exposed / sync_total) if sync_total > 0 else None,
            "nccl_bytes_sent_per_iter": nccl_sent, "nccl_bytes_recv_per_iter": nccl_recv,
            "layers": [{k: d[k] for k in ("name", "scheme", "rule", "model", "model3", "M", "N")} for d in sync.describe()],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if use_graph:
        del graph   # captured NCCL work holds the communicator: release the graph before ncclCommDestroy
        torch.cuda.synchronize()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_poseidon(args)


if __name__ == "__main__":
    sys.exit(main())
