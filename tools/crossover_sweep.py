"""C5: SFB vs PS crossover sweep over K on P GPUs for one FC layer (default the ImageNet-22K softmax
layer, M=21841, N=4096), against the paper's rule (Alg. 3).

    torchrun --nproc-per-node P tools/crossover_sweep.py [--M 21841 --N 4096] [--K 32,64,...]

For every K it measures, with CUDA events on the calling stream and the max over ranks:
  * SFB sync   : pack + all-gather of the factors + K1 reconstruct+SGD (poseidon_sync_fc_sfb);
  * PS sync    : reduce-scatter + K2 + all-gather (or the fused NVLS kernel) of the full gradient;
  * SF-PS sync : the literal Alg. 3 else-branch (reading Z20): U rows to their masters + all-gather
                 of V + K1 on the master's rows + broadcast of the rows (scheme_override = SFPS);
  * wgrad      : the local dW = G^T X GEMM (cuBLAS TF32) that PS needs and SFB / SF-PS skip.
and prints one JSON line per K with the rule's choice, the measured winner for sync-only and
sync+wgrad, and the regret of the rule.
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
    ap.add_argument("--M", type=int, default=21841)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", default="32,64,128,256,512,1024,2048")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nvls", action="store_true")
    a = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cuda.matmul.allow_tf32 = True
    obj = [pz.get_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    ctx = pz.Context(rank=rank, world=world, device=local, nccl_id=obj[0] if world > 1 else None,
                     flags=pz.FLAG_NVLS_PS if (a.nvls and world > 1) else 0)
    M, N = a.M, a.N
    W = torch.randn(M, N, device=dev) * 0.01
    b = torch.zeros(M, device=dev)
    n = M * N + M
    _, _, padded = pz.shard_range(n, world, rank)
    flat_w = torch.zeros(padded, device=dev)
    flat_g = torch.zeros(padded, device=dev)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        ts = []
        for r in range(a.reps + 1):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            if r > 0:
                ts.append(e0.elapsed_time(e1))
        t = torch.tensor([sorted(ts)[len(ts) // 2]], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    lid = 0
    for K in [int(k) for k in a.K.split(",")]:
        rule, costs = pz.choose_scheme(pz.LAYER_FC, M, N, K, world)
        ctx.register_layer(lid, pz.LAYER_FC, M, N, K, True, pz.SCHEME_SFB)
        ctx.register_layer(lid + 1, pz.LAYER_FC, M, N, K, True, pz.SCHEME_PS)
        ctx.register_layer(lid + 2, pz.LAYER_FC, M, N, K, True, pz.SCHEME_SFPS)
        ctx.bind_ps_buffers(lid + 1, flat_g, flat_w, n, pz.PS_ZERO_GRAD)
        U = torch.randn(K, M, device=dev) / K
        V = torch.randn(K, N, device=dev).relu()

        def sfb():
            ctx.sync_fc_sfb(lid, U, V, W, b, 0.01, s)
            ctx.wait_layer(lid, s)

        def ps():
            ctx.sync_ps(lid + 1, flat_g, flat_w, n, 0.01, s)
            ctx.wait_layer(lid + 1, s)

        def sfps():
            ctx.sync_fc_sfb(lid + 2, U, V, W, b, 0.01, s)
            ctx.wait_layer(lid + 2, s)

        gview = flat_g[: M * N].view(M, N)

        def wgrad():
            torch.mm(U.t(), V, out=gview)

        t_sfb, t_ps, t_wg, t_sfps = timed(sfb), timed(ps), timed(wgrad), timed(sfps)
        ctx.iteration_end(s)
        meas_sync = pz.SCHEME_SFB if t_sfb <= t_ps else pz.SCHEME_PS
        meas_total = pz.SCHEME_SFB if t_sfb <= t_ps + t_wg else pz.SCHEME_PS
        pick_t = t_sfb if rule == pz.SCHEME_SFB else t_ps + t_wg
        best_t = min(t_sfb, t_ps + t_wg)
        if rank == 0:
            name = {pz.SCHEME_SFB: "SFB", pz.SCHEME_PS: "PS"}
            print(json.dumps({"P": world, "M": M, "N": N, "K": K, "rule": name[rule],
                              "cost_sfb": costs[0], "cost_sf_ps": costs[1],
                              "sfb_ms": round(t_sfb, 4), "ps_ms": round(t_ps, 4), "wgrad_ms": round(t_wg, 4),
                              "sfps_ms": round(t_sfps, 4),
                              "winner_of_three": min((t_sfb, "SFB"), (t_ps + t_wg, "PS"), (t_sfps, "SFPS"))[1],
                              "winner_sync_only": name[meas_sync], "winner_with_wgrad": name[meas_total],
                              "rule_regret_ms": round(pick_t - best_t, 4)}), flush=True)
        lid += 3
        del U, V
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
