"""Per-phase breakdown of one SFB layer sync (library device events): queue (ready -> start), comm (start ->
all-gather done), K1 (kernel start -> end), tail (K1 end -> done: bias update + event records), total.

    torchrun --nproc-per-node P tools/sfb_breakdown.py [--M 1000 --N 4096 --K 256] [--reps 30]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_06216_b200 as pz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="1000x4096,4096x4096,4096x9216")
    ap.add_argument("--K", type=int, default=256)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--flags", type=int, default=-1)
    a = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    obj = [pz.get_unique_id() if (rank == 0 and world > 1) else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    flags = a.flags if a.flags >= 0 else (pz.FLAG_SYMM_SFB if world > 1 else 0)
    ctx = pz.Context(rank=rank, world=world, device=local, nccl_id=obj[0], flags=flags)
    s = torch.cuda.current_stream()
    K = a.K
    for lid, shp in enumerate(a.shapes.split(",")):
        M, N = (int(x) for x in shp.split("x"))
        ctx.register_layer(lid, pz.LAYER_FC, M, N, K)
        U = torch.randn(K, M, device=dev) / K
        V = torch.randn(K, N, device=dev).relu()
        W = torch.zeros(M, N, device=dev)
        b = torch.zeros(M, device=dev)
        rows = []
        for i in range(a.reps + 3):
            if world > 1:
                dist.barrier()
            torch.cuda._sleep(200_000)
            ctx.sync_fc_sfb(lid, U, V, W, b, 1e-3, s)
            ctx.wait_layer(lid, s)
            ctx.iteration_end(s)
            torch.cuda.synchronize()
            if i >= 3:
                rows.append(ctx.layer_stats(lid))
        med = {k: sorted(r[k] for r in rows)[len(rows) // 2] * 1e3
               for k in ("ready_to_start_ms", "comm_ms", "kernel_ms", "start_to_done_ms")}
        med["tail_us"] = med["start_to_done_ms"] - med["comm_ms"] - med["kernel_ms"]
        if rank == 0:
            print(json.dumps({"P": world, "M": M, "N": N, "K": K,
                              **{k.replace("_ms", "_us"): round(v, 1) for k, v in med.items()}}), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
