"""World-size-2 and -3 CPU (gloo) tests of the N>1 host logic: NCCL-id broadcast as
bench.py does it, cross-rank agreement of the library's host decisions (SACP
rule, shard map), and the exchange protocols' data layouts (rank-major
all-gather of SFB factors; reduce-scatter / shard update / all-gather of PS;
SF-PS's row masters from the library's row map)
emulated with gloo collectives and checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        import synthetic as S
        from paper_1512_06216_b200 import binding as B

        # 1. 128-byte id broadcast (bench.py / mp_sync_check.py pattern)
        fake_id = bytes(range(128)) if rank == 0 else None
        obj = [fake_id]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        # 2. host decisions agree across ranks and with the oracle
        for (M, N, K) in [(4096, 9216, 256), (1000, 4096, 256), (64, 1024, 100)]:
            s, c = B.choose_scheme(B.LAYER_FC, M, N, K, world)
            t = torch.tensor([s, c[0], c[1], c[2]], dtype=torch.int64)
            parts = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            assert all(torch.equal(parts[0], p) for p in parts)
            assert s == O.choose_scheme(O.LAYER_FC, M, N, K, world)
        for n in (650, 34944, 145578, 4097000):
            b, e, padded = B.shard_range(n, world, rank)
            t = torch.tensor([b, e, padded], dtype=torch.int64)
            parts = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            cover = 0
            for r, p in enumerate(parts):
                assert int(p[2]) == padded and int(p[0]) == cover and (int(p[0]), int(p[1]), int(p[2])) == \
                    O.shard_range(n, world, r)
                cover = int(p[1])
            assert cover == n

        # 3. SFB exchange: rank-major all-gather of (U_p, V_p), then local reconstruct+update
        M, N, K = 24, 40, 6
        W, b = S.fc_weights_randbias(M, N)
        Us, Vs = S.hidden_factors(M, N, K, world)
        u = torch.from_numpy(Us[rank])
        v = torch.from_numpy(Vs[rank])
        ug = [torch.zeros_like(u) for _ in range(world)]
        vg = [torch.zeros_like(v) for _ in range(world)]
        dist.all_gather(ug, u)
        dist.all_gather(vg, v)
        W1, b1 = O.sfb_simulated(W, b, [x.numpy() for x in ug], [x.numpy() for x in vg], 0.3)
        W4, b4 = O.sync_step(W, b, Us, Vs, 0.3)
        assert np.max(np.abs(W1 - W4)) < 1e-12 and np.max(np.abs(b1 - b4)) < 1e-12
        res = torch.from_numpy(W1)
        parts = [torch.zeros_like(res) for _ in range(world)]
        dist.all_gather(parts, res)
        assert all(torch.equal(parts[0], p) for p in parts)

        # 4. PS exchange: reduce-scatter (all_reduce + own shard), shard SGD, all-gather of W
        n = M * N + M
        _, _, padded = O.shard_range(n, world, 0)
        S_ = padded // world
        g = np.zeros(padded)
        g[:n] = O.flatten_params(O.reconstruct(Us[rank], Vs[rank]), Us[rank].astype(np.float64).sum(0))
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)
        w = np.zeros(padded)
        w[:n] = O.flatten_params(W, b)
        lo, hi, _ = O.shard_range(n, world, rank)
        shard = torch.from_numpy(w[rank * S_:(rank + 1) * S_].copy())
        shard[: hi - lo] += (-0.3 / world) * gt[lo:hi]
        out = [torch.zeros_like(shard) for _ in range(world)]
        dist.all_gather(out, shard)
        w1 = torch.cat(out).numpy()[:n]
        W6, b6 = O.ps_simulated(W, b, Us, Vs, 0.3)
        assert np.max(np.abs(w1 - O.flatten_params(W6, b6))) < 1e-12

        # 5. SF-PS exchange (Alg. 3 else-branch, reading Z20) with the library's row map: U columns of master
        #    m's rows to m (send/recv), V to everyone (all-gather), master reconstructs its rows, rows broadcast
        M2 = 70                                   # 32-row masters: rank 0 owns 64 rows, rank 1 owns 6 at P = 2
        W, b = S.fc_weights_randbias(M2, N)
        Us, Vs = S.hidden_factors(M2, N, K, world, seed=17)
        rows = [B.shard_range(M2, world, m)[:2] for m in range(world)]
        assert rows == [O.row_shard_range(M2, world, m) for m in range(world)]
        lo, hi = rows[rank]
        mine = {rank: torch.from_numpy(np.ascontiguousarray(Us[rank][:, lo:hi]))}
        reqs = []
        for m in range(world):
            if m == rank:
                continue
            qb, qe = rows[m]
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Us[rank][:, qb:qe])), m))
            mine[m] = torch.zeros(K, hi - lo, dtype=torch.float32)
            reqs.append(dist.irecv(mine[m], m))
        for r_ in reqs:
            r_.wait()
        vg = [torch.zeros(K, N, dtype=torch.float32) for _ in range(world)]
        dist.all_gather(vg, torch.from_numpy(Vs[rank]))
        G = sum(mine[p].double().numpy().T @ vg[p].double().numpy() for p in range(world))
        gb = sum(mine[p].double().numpy().sum(0) for p in range(world))
        Wout = torch.from_numpy(W.astype(np.float64).copy())
        Wout[lo:hi] += (-0.3 / world) * torch.from_numpy(G)
        bout = torch.from_numpy(b.astype(np.float64).copy())
        bout[lo:hi] += (-0.3 / world) * torch.from_numpy(gb)
        for m in range(world):
            qb, qe = rows[m]
            blk = Wout[qb:qe].contiguous()
            dist.broadcast(blk, src=m)
            Wout[qb:qe] = blk
            bb = bout[qb:qe].contiguous()
            dist.broadcast(bb, src=m)
            bout[qb:qe] = bb
        W11, b11, _ = O.sf_ps_simulated(W, b, Us, Vs, 0.3)
        assert np.max(np.abs(Wout.numpy() - W11)) < 1e-12 and np.max(np.abs(bout.numpy() - b11)) < 1e-12
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "".join(traceback.format_exception(ex))))


@pytest.mark.parametrize("world", [2, 3])   # 3: ragged shard maps (padded / P not a multiple of the 4-float unit)
def test_gloo_host_logic_and_protocols(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r, msg in results:
        assert msg == "ok", f"rank {r}: {msg}"
