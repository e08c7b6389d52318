"""Collective bus bandwidth on NVLink 5 (nccl-tests conventions: busbw = algbw * (P-1)/P).

    torchrun --nproc-per-node P tools/collective_bench.py [--ps-only | --sfb-only]

(a) raw NCCL all-gather / reduce-scatter through torch.distributed (the same libnccl.so.2 the
    library links), message sizes per rank 1 MB .. 512 MB;
(b) the library's own sync paths, measured by its device events:
    - SFB factor all-gather of fc6 / fc7 / the C5 softmax layer at K=256 (comm_ms of the layer);
    - PS of a 37.7M-parameter layer: NCCL reduce-scatter + K2 + all-gather vs the fused NVLS kernel.
Prints JSON lines; rank 0 only.  Peaks: 900 GB/s per direction nominal, 770 measured peer copy.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402
from paper_1512_06216_b200.binding import device_view  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P = world
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def out(d):
        if rank == 0:
            print(json.dumps(d), flush=True)

    only_ps = "--ps-only" in sys.argv
    only_sfb = "--sfb-only" in sys.argv
    for mb in (() if (only_ps or only_sfb) else (1, 4, 16, 64, 256, 512)):
        n = mb * (1 << 20) // 4
        x = torch.randn(n, device=dev)
        y = torch.empty(n * P, device=dev)
        t = timed(lambda: dist.all_gather_into_tensor(y, x))
        alg = n * 4 * P / (t / 1e3) / 1e9
        out({"what": "nccl all_gather", "P": P, "MB_per_rank": mb, "ms": round(t, 4),
             "busbw_GBps": round(alg * (P - 1) / P, 1)})
        t = timed(lambda: dist.reduce_scatter_tensor(x, y))
        alg = n * 4 * P / (t / 1e3) / 1e9
        out({"what": "nccl reduce_scatter", "P": P, "MB_per_rank": mb, "ms": round(t, 4),
             "busbw_GBps": round(alg * (P - 1) / P, 1)})
        del x, y

    def new_ctx(flags):
        obj = [pz.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return pz.Context(rank=rank, world=world, device=local, nccl_id=obj[0], flags=flags)

    # (b1) SFB factor all-gather inside poseidon_sync_fc_sfb: plain cudaMalloc gather buffers vs NCCL
    #      symmetric windows (FLAG_SYMM_SFB)
    sfb_layers = () if only_ps else (("fc6", 4096, 9216), ("fc7", 4096, 4096), ("i22k_fc8", 21841, 4096))
    for flags, tag in ((0, "cudaMalloc"), (pz.FLAG_SYMM_SFB, "symmetric window"),
                       (pz.FLAG_NVLS_SFB, "NVLS multicast broadcast")):
        ctx = new_ctx(flags)
        for lid, (name, M, N) in enumerate(sfb_layers):
            K = 256
            ctx.register_layer(lid, pz.LAYER_FC, M, N, K)
            U = torch.randn(K, M, device=dev) / K
            V = torch.randn(K, N, device=dev).relu()
            W = torch.zeros(M, N, device=dev)
            comm = []
            for _ in range(8):
                dist.barrier()
                torch.cuda._sleep(200_000)   # queue the whole sync before it runs (device time only)
                ctx.sync_fc_sfb(lid, U, V, W, None, 0.0, s)
                ctx.wait_layer(lid, s)
                ctx.iteration_end(s)
                torch.cuda.synchronize()
                comm.append(ctx.layer_stats(lid)["comm_ms"])
            t = sorted(comm[2:])[len(comm[2:]) // 2]
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
            per_rank = K * (M + N + M // K + 1) * 4  # U + V slot (+ bias column sums) per rank
            alg = per_rank * P / (t / 1e3) / 1e9
            out({"what": f"poseidon SFB all-gather ({name}, K=256, {tag})", "P": P, "path": ctx.sfb_path(lid),
                 "cta_policy": os.environ.get("POSEIDON_NCCL_CTA_POLICY", "default"),
                 "MB_per_rank": round(per_rank / 2**20, 2), "ms": round(t, 4),
                 "busbw_GBps": round(alg * (P - 1) / P, 1)})
        ctx.close()

    # (b2) PS of a 37.7M-parameter layer: NCCL path vs fused NVLS kernel
    M, N = 4096, 9216
    n = M * N
    for nv in (() if only_sfb else (True,) if only_ps else (False, True)):
        c = new_ctx(pz.FLAG_NVLS_PS if nv else 0)
        c.register_layer(0, pz.LAYER_FC, M, N, 256, False, pz.SCHEME_PS)
        if nv:
            active = c.ps_arena()
            gp, wp, padded = c.ps_layer_buffers(0)
            g, w = device_view(gp, (padded,)), device_view(wp, (padded,))
        else:
            active = False
            _, _, padded = pz.shard_range(n, P, rank)
            g, w = torch.zeros(padded, device=dev), torch.zeros(padded, device=dev)
            c.bind_ps_buffers(0, g, w, n, pz.PS_ZERO_GRAD)
        c.set_lr(0.0)
        ts = []
        for _ in range(6):
            g.fill_(1.0)
            torch.cuda.synchronize()
            dist.barrier()
            c.backprop_hook(0, s)
            c.wait_layer(0, s)
            c.iteration_end(s)
            torch.cuda.synchronize()
            ts.append(c.layer_stats(0)["start_to_done_ms"])
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        tt = torch.tensor([t], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        bus = 2.0 * (P - 1) / P * 4.0 * padded / (t / 1e3) / 1e9
        out({"what": "poseidon PS sync 37.7M params (" + ("fused NVLS kernel" if active else "NCCL RS + K2 + AG") + ")",
             "P": P, "MB": round(4 * n / 2**20, 1), "ms": round(t, 4), "busbw_GBps(RS+AG equiv)": round(bus, 1),
             "nvls": c.nvls_status(), "grid": os.environ.get("POSEIDON_NVLS_GRID", "auto"),
             "U": os.environ.get("POSEIDON_NVLS_U", "4")})
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
