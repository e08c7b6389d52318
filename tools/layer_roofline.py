"""Per-layer sync against its roofline, each layer in isolation.

    torchrun --nproc-per-node P tools/layer_roofline.py [--reps 50] [--configs C2,C3,C4,C5]

Every parameterised layer of the configs is synced alone through the context API (the same calls the
DWBP glue makes), `reps` times with a barrier before each, and the library's device-event
`start_to_done` (collectives + update kernels) is taken: median over reps, max over ranks.
A ~100 us device spin precedes every timed sync so that all of its launches are queued before it runs.
Also measured: alpha (8-byte NCCL all-gather) and the NCCL all-gather busbw at 256 MB per rank.
PS layers run both on the NCCL path and (P > 1) on the fused NVLS kernel; at P > 1 every FC layer is
also synced as SF-PS (the literal else-branch of Alg. 3, reading Z20; scheme_override = SFPS).
Prints JSON lines (rank 0); tools/layer_roofline_md.py applies the §8(d) roofline formulas.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.nn as nn

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402
from drivers.cnn import CONFIGS  # noqa: E402

BW_NVL_SPEC = 900e9
SFPS_ID = 2000   # layer ids of the SF-PS registrations of the FC layers
SLEEP_CYCLES = 200_000


def layers_of(cfg):
    c = CONFIGS[cfg]
    model = c["model"]()
    out = []
    for name, mod in model.named_modules():
        if isinstance(mod, nn.Linear):
            out.append((f"{cfg}.{name}", pz.LAYER_FC, mod.out_features, mod.in_features, mod.bias is not None))
        elif isinstance(mod, nn.Conv2d):
            out.append((f"{cfg}.{name}", pz.LAYER_CONV, mod.out_channels, mod.weight[0].numel(), mod.bias is not None))
    if cfg == "C5":  # only the 21841-way classifier differs from C3
        out = [l for l in out if l[2] == 21841]
    return out, c["batch"], c["scheme"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--configs", default="C2,C3,C4,C5")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P = world
    s = torch.cuda.current_stream()

    def out(d):
        if rank == 0:
            print(json.dumps(d), flush=True)

    def maxr(x):
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # alpha (8-byte all-gather) and the large-message all-gather busbw
    alpha, bw_nvl_meas = 0.0, BW_NVL_SPEC
    if P > 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x, y = torch.zeros(2, device=dev), torch.zeros(2 * P, device=dev)
        ts = []
        for i in range(60):
            dist.barrier()
            torch.cuda._sleep(SLEEP_CYCLES)   # absorb the ranks' host skew (see measure())
            e0.record(s)
            dist.all_gather_into_tensor(y, x)
            e1.record(s)
            e1.synchronize()
            if i >= 10:
                ts.append(e0.elapsed_time(e1) * 1e-3)
        alpha = maxr(sorted(ts)[len(ts) // 2])
        n = 64 << 20
        x, y = torch.zeros(n, device=dev), torch.zeros(n * P, device=dev)
        dist.all_gather_into_tensor(y, x)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(s)
        for _ in range(5):
            dist.all_gather_into_tensor(y, x)
        e1.record(s)
        e1.synchronize()
        t = maxr(e0.elapsed_time(e1) * 1e-3 / 5)
        bw_nvl_meas = n * 4 * P / t * (P - 1) / P
        del x, y
    out({"P": P, "alpha_us": round(alpha * 1e6, 2), "bw_nvl_measured_GBps": round(bw_nvl_meas / 1e9, 1)})

    def new_ctx(flags):
        obj = [pz.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return pz.Context(rank=rank, world=world, device=local, nccl_id=obj[0], flags=flags)

    # bench.py's N > 1 configuration: SFB factors through the library broadcast kernel; PS on both paths
    ctx = new_ctx(pz.FLAG_NVLS_SFB if P > 1 else 0)
    nv = new_ctx(pz.FLAG_NVLS_PS) if P > 1 else None
    plan = []   # (name, lid, kind, M, N, K, scheme, n)
    lid = 0
    for cfg in a.configs.split(","):
        ls, K, cscheme = layers_of(cfg)
        for (name, kind, M, N, hb) in ls:
            override = pz.SCHEME_PS if cscheme == "ps" else -1
            sch = ctx.register_layer(lid, kind, M, N, K, hb, override)
            n = M * N + (M if hb else 0)
            if nv is not None and sch == pz.SCHEME_PS:
                nv.register_layer(lid, kind, M, N, K, hb, pz.SCHEME_PS)
            plan.append((name, lid, kind, M, N, K, sch, n, hb))
            if P > 1 and kind == pz.LAYER_FC:
                ctx.register_layer(SFPS_ID + lid, kind, M, N, K, hb, pz.SCHEME_SFPS)
            lid += 1
    nvls_active = nv.ps_arena() if nv is not None else False
    out({"P": P, "nvls": nv.nvls_status() if nv is not None else "P=1", "layers": len(plan)})

    def measure(c, l, fn):
        # The producer stream first runs a ~100 us spin, so every launch of the sync is queued before
        # the GPU reaches it: start_to_done is then device time, not the host's enqueue latency on an
        # idle GPU, and the ranks' host skew after the barrier is absorbed.
        ts = []
        for i in range(a.reps + 3):
            dist.barrier()
            torch.cuda._sleep(SLEEP_CYCLES)
            fn()
            c.wait_layer(l, s)
            c.iteration_end(s)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(c.layer_stats(l)["start_to_done_ms"] * 1e-3)
        return maxr(sorted(ts)[len(ts) // 2])

    for (name, l, kind, M, N, K, sch, n, hb) in plan:
        rows = {}
        if sch == pz.SCHEME_SFB:
            U = torch.randn(K, M, device=dev) / K
            V = torch.randn(K, N, device=dev).relu()
            W = torch.zeros(M, N, device=dev)
            b = torch.zeros(M, device=dev) if hb else None
            rows["sfb"] = measure(ctx, l, lambda: ctx.sync_fc_sfb(l, U, V, W, b, 1e-3, s))
            del U, V, W, b
        else:
            _, _, padded = pz.shard_range(n, P, rank)
            g, w = torch.zeros(padded, device=dev), torch.zeros(padded, device=dev)
            ctx.bind_ps_buffers(l, g, w, n, pz.PS_ZERO_GRAD)
            rows["ps_nccl"] = measure(ctx, l, lambda: ctx.backprop_hook(l, s))
            if nvls_active:
                rows["ps_nvls"] = measure(nv, l, lambda: nv.backprop_hook(l, s))
            del g, w
        if P > 1 and kind == pz.LAYER_FC:
            U = torch.randn(K, M, device=dev) / K
            V = torch.randn(K, N, device=dev).relu()
            W = torch.zeros(M, N, device=dev)
            b = torch.zeros(M, device=dev) if hb else None
            rows["sfps"] = measure(ctx, SFPS_ID + l, lambda: ctx.sync_fc_sfb(SFPS_ID + l, U, V, W, b, 1e-3, s))
            del U, V, W, b
        for path, t in rows.items():
            out({"P": P, "layer": name, "M": M, "N": N, "K": K, "n": n, "scheme": path,
                 "measured_us": round(t * 1e6, 2)})
    ctx.close()
    if nv is not None:
        nv.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
