"""Multi-GPU worker (torchrun, one process per GPU, NCCL through libposeidon).

Checks, at world = P:
  1. SFB sync of the C1 layer (M=128, N=256, K=8): integer variant bit-exact
     vs the oracle O4 (TF32 and fp32 reconstruction), random factors within
     the Z13 gate; every rank's W bit-identical.
  2. PS sync of the same layer's flat buffer (RS -> K2 -> AG): integer variant
     bit-exact vs O6, random within 1e-5; every rank bit-identical.
  1b. SFB on NCCL symmetric windows and over the NVLS multicast broadcast: integer variant
     bit-exact vs O4 for three shapes (odd M, K not a multiple of 4) over three iterations.
  3. A layer with an empty shard (n=650 at P=8 has one) and odd sizes.
  4. Two DWBP training steps of CIFAR-10 quick (C2 shapes, K=16/GPU, SACP
     auto and forced PS, DWBP on and off, NCCL and NVLS PS, SF-PS): every
     iteration every layer's update equals the oracle's O6 / O4 recomputed from
     all ranks' captured gradients / factors (Z13 metric, fp32 1e-5 for PS,
     TF32 2e-3 for factor layers; O7 makes this the concatenated-batch SGD
     step), all ranks' parameters bit-identical, DWBP on == off bitwise.
  8. SF-PS (the literal else-branch of Alg. 3, reading Z20): integer variant bit-exact vs O11 on three
     shapes (masters with no rows at P = 4), plain / symmetric buffers / DWBP off, both kernels, NCCL
     byte counts; random factors with momentum vs O4m; FLAG_SFPS auto-selection; CIFAR-quick with
     every FC layer as SF-PS in test 4.
  9. Early input broadcast (FLAG_EARLY_V): V posted at forward time, NCCL and broadcast-kernel wires,
     integer bit-exact vs O4 with garbage V at the sync; CIFAR-quick training bit-identical to the plain run.
  6. SSP, staleness 1: SFB + PS over 4 iterations and a flush, integer variant bit-exact vs O10 on
     the NCCL and the NVLS paths.
  7. PS buckets: six layers of mixed sizes, NCCL and fused NVLS paths, integer bit-exact per layer.
  10. Fused NVLS PS zero-grad ordering: the five C3 conv layers' sizes (shard starts not aligned to the
     kernel's grid stride, several CTAs per layer), four iterations of integer gradients through the
     DWBP hook, bit-exact vs O6 every iteration.  Run with POSEIDON_FUZZ_US set, every CTA sleeps a
     pseudo-random time after the entry barrier (`--race-only` runs just this check).
  11. C3 with the schedule the rule picks at P >= 6 (fc8 forced to PS) in bench.py's N > 1 launch
     configuration, one step, every layer vs the oracle (tests/stepcheck.py).
  `--wire-only` runs only 1b and 9 (the factor broadcast kernel), for POSEIDON_SFB_BCAST_GRID sweeps.
  5. Full size in bench.py's N > 1 configuration: C3 fc6 SFB through the library's broadcast kernel (sampled
     rows vs O4)
     and a 37.7M-parameter PS layer through the fused NVLS kernel (sampled elements vs O6).
Prints "MP_OK <rank>" on success; any failure raises.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synthetic as S  # noqa: E402
from parity import check_update, w0_like  # noqa: E402
import paper_1512_06216_b200 as pz  # noqa: E402
from paper_1512_06216_b200.dwbp import PoseidonSync  # noqa: E402
from drivers.cnn import CifarQuick  # noqa: E402


def allsame(t):
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return all(torch.equal(parts[0], p) for p in parts[1:])


def wire_bytes(shapes, flags):
    """Bytes one rank hands to the factor exchange of one iteration: K-major slots (M, N padded to ldk) plus the
    bias sums, or, with FLAG_INPLACE_MN on layers with M, N multiples of 4, the MN-major slots K x (M + N)."""
    mn = (flags & pz.FLAG_INPLACE_FACTORS) and (flags & pz.FLAG_INPLACE_MN)
    out = 0
    for _, M_, N_, K_ in shapes:
        if mn and M_ % 4 == 0 and N_ % 4 == 0:
            out += K_ * (M_ + N_) * 4
        else:
            ldk = (K_ + 3) // 4 * 4
            out += (M_ * ldk + N_ * ldk + M_) * 4
    return out


def sfb_wire_checks(new_ctx, rank, P, dev):
    # ---- 1b. SFB on symmetric buffers: NCCL all-gather (SYMM_SFB) and the NVLS multicast broadcast
    #          (NVLS_SFB); odd M (bias slot not a multiple of 4), ldk padding, 3 iterations in a row
    #          (the broadcast's entry barrier guards the gather buffers the previous K1 read) ----
    # (+ FLAG_INPLACE_FACTORS: the pack reads U / V in place on the comm stream; the caller keeps them alive)
    # (+ FLAG_INPLACE_MN: MN-major gather layout, copy-engine slot fill, K1 on MN-major operands, bias sums in
    #  K1 -- for the layers with M, N multiples of 4; the 10 x 64 layer keeps the pack)
    mnf = pz.FLAG_INPLACE_FACTORS | pz.FLAG_INPLACE_MN
    for flags in (pz.FLAG_SYMM_SFB, pz.FLAG_NVLS_SFB, pz.FLAG_NVLS_SFB | pz.FLAG_INPLACE_FACTORS,
                  pz.FLAG_INPLACE_FACTORS, pz.FLAG_NVLS_SFB | mnf, mnf):
        cs = new_ctx(flags)
        shapes = [(0, 128, 256, 8), (1, 10, 64, 4), (2, 1000, 4096, 33)]
        for lid, M_, N_, K_ in shapes:   # SFB forced: the rule sends the 10 x 64, K = 4 layer to PS at P >= 5
            assert cs.register_layer(lid, pz.LAYER_FC, M_, N_, K_, True, pz.SCHEME_SFB) == pz.SCHEME_SFB
        path = cs.sfb_path(0)
        assert path >= pz.SFB_PATH_NCCL_SYMM or not (flags & (pz.FLAG_SYMM_SFB | pz.FLAG_NVLS_SFB)), path
        if rank == 0:
            print(f"SFB path flags={flags}: {path}", flush=True)
        for it in range(3):
            for lid, M_, N_, K_ in shapes:
                W, b, Us, Vs, lr = S.integer_factors(M_, N_, K_, P, seed=100 * it + lid)
                Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
                Ud, Vd = torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev)
                cs.sync_fc_sfb(lid, Ud, Vd, Wd, bd, lr)
                cs.wait_layer(lid)
                W1, b1 = O.sync_step(W, b, Us, Vs, lr)
                torch.cuda.synchronize()
                assert np.array_equal(Wd.cpu().numpy().astype(np.float64), W1), f"SFB flags={flags} it={it} lid={lid}"
                assert np.array_equal(bd.cpu().numpy().astype(np.float64), b1)
                assert allsame(Wd) and allsame(bd)
            st = cs.iteration_end(stats=True)
            assert st["nccl_bytes_recv"] == wire_bytes(shapes, flags) * (P - 1), st
        cs.close()


def early_v_checks(new_ctx, rank, P, dev):
    # ---- 9. early input broadcast (FLAG_EARLY_V): V posted at "forward" time, only U at the sync (whose V
    #          argument is garbage here); NCCL and broadcast-kernel wires; integer bit-exact vs O4, two
    #          iterations, and the same NCCL byte total as the plain sync ----
    for flags in (pz.FLAG_EARLY_V, pz.FLAG_EARLY_V | pz.FLAG_NVLS_SFB,
                  pz.FLAG_EARLY_V | pz.FLAG_NVLS_SFB | pz.FLAG_INPLACE_FACTORS,
                  pz.FLAG_EARLY_V | pz.FLAG_NVLS_SFB | pz.FLAG_INPLACE_FACTORS | pz.FLAG_INPLACE_MN):
        ce = new_ctx(flags)
        keep = []   # FLAG_INPLACE_FACTORS: the factors stay alive until the syncs are done
        shapes = [(0, 128, 256, 8), (1, 10, 64, 4), (2, 1000, 4096, 33)]
        for lid, M_, N_, K_ in shapes:   # SFB forced (the 10 x 64 layer is PS by the rule at P >= 5)
            assert ce.register_layer(lid, pz.LAYER_FC, M_, N_, K_, True, pz.SCHEME_SFB) == pz.SCHEME_SFB
        for it in range(2):
            outs = []
            for lid, M_, N_, K_ in shapes:   # "forward": every layer posts its input
                W, b, Us, Vs, lr = S.integer_factors(M_, N_, K_, P, seed=700 + 10 * it + lid)
                ce.sfb_post_input(lid, torch.from_numpy(Vs[rank]).to(dev))
                outs.append((W, b, Us, Vs, lr))
            res = []
            for lid, (W, b, Us, Vs, lr) in reversed(list(enumerate(outs))):   # "backward": top layer first
                Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
                junk = torch.full((Vs[rank].shape[0], Vs[rank].shape[1]), 5.0, device=dev)
                Ud = torch.from_numpy(Us[rank]).to(dev)
                keep += [Ud, junk]
                ce.sync_fc_sfb(lid, Ud, junk, Wd, bd, lr)
                res.append((lid, Wd, bd))
            st = ce.iteration_end(stats=True)
            for lid, Wd, bd in res:
                ce.wait_layer(lid)
            torch.cuda.synchronize()
            for lid, Wd, bd in res:
                W, b, Us, Vs, lr = outs[lid]
                W1, b1 = O.sync_step(W, b, Us, Vs, lr)
                assert np.array_equal(Wd.cpu().numpy().astype(np.float64), W1), f"early V flags={flags} lid={lid}"
                assert np.array_equal(bd.cpu().numpy().astype(np.float64), b1)
                assert allsame(Wd) and allsame(bd)
            assert st["nccl_bytes_recv"] == wire_bytes(shapes, flags) * (P - 1), st
        ce.close()


def graph_checks(new_ctx, rank, P, dev, batch, lr, Kc):
    """Check 12 (round 2): one CIFAR-quick DWBP step captured in a CUDA graph (bench.py --graph) on the bench's
    N > 1 paths -- the fused NVLS PS kernel, the SFB broadcast wire with early V, NCCL RS/AG -- replayed twice
    after two eager steps, equals four eager steps bit for bit on every rank (cuDNN deterministic)."""
    from paper_1512_06216_b200.dwbp import PoseidonSync
    det, bench_ = torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    variants = [("ps", pz.FLAG_NVLS_PS, True), ("auto", pz.FLAG_NVLS_PS | pz.FLAG_NVLS_SFB | pz.FLAG_EARLY_V, True),
                ("auto", 0, False)]
    if os.environ.get("MP_GRAPH_VARIANT"):
        variants = [variants[int(os.environ["MP_GRAPH_VARIANT"])]]
    for scheme, flags, arena in variants:
        out = []
        for graph in (False, True):
            if rank == 0 and os.environ.get("MP_VERBOSE"):
                print(f"graph check: {scheme} flags {flags} graph {graph}", flush=True)
            cg = new_ctx(flags)
            torch.manual_seed(1234)
            model = CifarQuick().to(dev)
            sync = PoseidonSync(model, cg, K=Kc, lr=lr, scheme=scheme, recon=pz.RECON_TF32, arena=arena)
            x = torch.empty(Kc, 3, 32, 32, device=dev)
            y = torch.empty(Kc, dtype=torch.long, device=dev)

            def step():
                F.cross_entropy(model(x), y).backward()
                sync.iteration_end()

            for it in range(4):
                xb, yb = batch(it)
                x.copy_(xb)
                y.copy_(yb)
                if graph and it == 2:
                    sync.wait_all()
                    torch.cuda.synchronize()
                    gs = torch.cuda.Stream(device=dev)
                    gs.wait_stream(torch.cuda.current_stream())
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=gs):
                        step()
                    torch.cuda.current_stream().wait_stream(gs)
                    if os.environ.get("MP_VERBOSE"):
                        print(f"[rank {rank}] captured", flush=True)
                if graph and it >= 2:
                    g.replay()
                    if os.environ.get("MP_VERBOSE"):
                        torch.cuda.synchronize()
                        print(f"[rank {rank}] replay {it} done", flush=True)
                else:
                    step()
            sync.wait_all()
            torch.cuda.synchronize()
            flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
            assert allsame(flat), f"graph check: ranks differ ({scheme}, flags {flags}, graph {graph})"
            if graph:
                st = cg.iter_stats(0)
                assert st["n_layers"] == 5 and st["sync_total_ms"] > 0, st
            out.append(flat.cpu())
            if graph:
                # a graph with captured NCCL work keeps the communicator's persistent plans alive: release it
                # before ncclCommDestroy (poseidon_finalize would otherwise wait for it forever)
                del g
                torch.cuda.synchronize()
            cg.close()
        assert torch.equal(out[0], out[1]), f"graph replay != eager ({scheme}, flags {flags})"
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = det, bench_
    if rank == 0:
        print(f"graph check ok ({len(variants)} variants: 2 eager + 2 replays == 4 eager)", flush=True)


def alexnet_p6_schedule_check(new_ctx, rank, P, dev, world):
    """Check 11: the schedule the rule picks for C3 at P >= 6 (fc6 / fc7 SFB, fc8 PS, conv PS) on the P GPUs at
    hand (fc8 forced to PS), in bench.py's N > 1 launch configuration (NVLS PS arena, broadcast wire, early V,
    channels_last, batch 256 / GPU): one DWBP step, every layer's update vs the oracle from all ranks'
    captures (O4 on sampled rows for fc6 / fc7, O6 on every element of fc8 and the convs)."""
    import torch.nn.functional as F
    from drivers.cnn import AlexNet
    from stepcheck import StepCapture, oracle_check, safe_lr
    torch.backends.cudnn.deterministic = True
    torch.manual_seed(6216)
    model = AlexNet().to(dev).to(memory_format=torch.channels_last)
    g = torch.Generator(device=dev)
    g.manual_seed(1512 + rank)
    x = torch.rand((256, 3, 227, 227), device=dev, generator=g).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (256,), device=dev, generator=g)
    lr = safe_lr(model, lambda m: F.cross_entropy(m(x), y), world)
    flags = pz.FLAG_NVLS_PS | pz.FLAG_NVLS_SFB | pz.FLAG_EARLY_V if P > 1 else 0
    c = new_ctx(flags)
    sync = PoseidonSync(model, c, K=256, lr=lr, arena=P > 1, overrides={"fc8": "ps"})
    picks = {p.name: p.scheme for p in sync.plans}
    assert picks["fc6"] == pz.SCHEME_SFB and picks["fc7"] == pz.SCHEME_SFB and picks["fc8"] == pz.SCHEME_PS, picks
    cap = StepCapture(sync)
    cap.snapshot()
    F.cross_entropy(model(x), y).backward()
    sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()
    errs = oracle_check(cap, lr, world)
    assert len(errs) == 8, errs
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
    assert allsame(flat)
    c.close()
    if rank == 0:
        print(f"C3 P>=6 schedule (fc8 PS) ok at P={P}: " + ", ".join(f"{k} {v:.1e}" for k, v in errs.items()),
              flush=True)


def nvls_race_check(new_ctx, rank, P, dev):
    """Check 10: every CTA of the fused NVLS PS kernel may clear only what the same-index CTAs of all
    ranks reduced (LSA barrier j pairs block j only).  C3 conv layer sizes; 4 iterations."""
    from paper_1512_06216_b200.binding import device_view
    cr = new_ctx(pz.FLAG_NVLS_PS)
    shapes = [(96, 363), (256, 1200), (384, 2304), (384, 1728), (256, 1728)]   # conv1..conv5 (M, C*kh*kw)
    for lid, (M_, N_) in enumerate(shapes):
        cr.register_layer(lid, pz.LAYER_CONV, M_, N_, 1, True, pz.SCHEME_PS)
    lr = 2.0 ** -7
    cr.set_lr(lr)
    cr.ps_arena()
    status = cr.nvls_status()
    views, ws = [], []
    for lid, (M_, N_) in enumerate(shapes):
        n = M_ * N_ + M_
        gp, wp, padded = cr.ps_layer_buffers(lid)
        wv, gv = device_view(wp, (padded,)), device_view(gp, (padded,))
        w0 = (S.rng(1000 + lid).integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
        wv[:n] = torch.from_numpy(w0).to(dev)
        views.append((wv, gv, n))
        ws.append(w0.astype(np.float64))
    bad = 0
    for it in range(4):
        refs = []
        for lid, (wv, gv, n) in enumerate(views):
            grads = S.integer_grads(n, P, seed=2000 + 10 * it + lid)
            gv[:n] = torch.from_numpy(grads[rank]).to(dev)
            refs.append(O.ps_step_flat(ws[lid], grads, lr))
        torch.cuda.synchronize()
        dist.barrier()
        for lid in reversed(range(len(shapes))):
            cr.backprop_hook(lid, torch.cuda.current_stream())
        for lid in range(len(shapes)):
            cr.wait_layer(lid)
        cr.iteration_end()
        torch.cuda.synchronize()
        for lid, ((wv, gv, n), ref) in enumerate(zip(views, refs)):
            out = wv[:n].cpu().numpy().astype(np.float64)
            nbad = int(np.count_nonzero(out != ref))
            if nbad:
                print(f"[rank {rank}] NVLS race check: iteration {it} layer {lid}: {nbad} of {n} elements "
                      f"differ from O6", flush=True)
            bad += nbad
            assert float(gv.abs().sum()) == 0.0, "gradient not cleared"
            assert allsame(wv[:n].contiguous())
            ws[lid] = ref
    cr.close()
    assert bad == 0, f"fused NVLS PS lost gradient contributions ({bad} elements, {status})"
    if rank == 0:
        print(f"NVLS race check ok ({status}, POSEIDON_FUZZ_US={os.environ.get('POSEIDON_FUZZ_US', '0')})",
              flush=True)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    # DWBP on/off must be bit-identical: only scheduling differs, so the driver's own
    # convolutions must be deterministic too (cuDNN wgrad may otherwise use atomics)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    P = world

    def new_ctx(flags=0):
        # an ncclUniqueId bootstraps exactly one communicator: fresh id per context
        obj = [pz.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return pz.Context(rank=rank, world=world, device=local, nccl_id=obj[0], flags=flags)

    if "--wire-only" in sys.argv:   # the factor broadcast kernel alone (e.g. with POSEIDON_SFB_BCAST_GRID set)
        sfb_wire_checks(new_ctx, rank, P, dev)
        early_v_checks(new_ctx, rank, P, dev)
        dist.barrier()
        print(f"MP_OK {rank}", flush=True)
        dist.destroy_process_group()
        return
    if "--graph-only" in sys.argv:   # check 12 alone
        Kc = 16

        def batch(it):
            gen = torch.Generator().manual_seed(100 + it)
            xall = torch.rand(P * Kc, 3, 32, 32, generator=gen).to(dev)
            yall = torch.randint(0, 10, (P * Kc,), generator=gen).to(dev)
            return xall[rank * Kc:(rank + 1) * Kc], yall[rank * Kc:(rank + 1) * Kc]

        graph_checks(new_ctx, rank, P, dev, batch, 0.05, Kc)
        dist.barrier()
        print(f"MP_OK {rank}", flush=True)
        dist.destroy_process_group()
        return
    if "--race-only" in sys.argv:
        nvls_race_check(new_ctx, rank, P, dev)
        dist.barrier()
        print(f"MP_OK {rank}", flush=True)
        dist.destroy_process_group()
        return
    nvls_race_check(new_ctx, rank, P, dev)

    ctx = new_ctx()
    M, N, K = 128, 256, 8
    assert ctx.register_layer(0, pz.LAYER_FC, M, N, K) == pz.SCHEME_SFB
    assert ctx.register_layer(1, pz.LAYER_FC, M, N, K, scheme_override=pz.SCHEME_PS) == pz.SCHEME_PS

    # ---- 1. SFB, integer variant, both reconstruction kernels ----
    for recon in (pz.RECON_TF32, pz.RECON_FP32):
        ctx.set_recon(recon, 0)
        W, b, Us, Vs, lr = S.integer_factors(M, N, K, P, seed=3)
        Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
        ctx.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, lr)
        ctx.wait_layer(0)
        st = ctx.iteration_end(stats=True)
        torch.cuda.synchronize()
        W1, b1 = O.sync_step(W, b, Us, Vs, lr)
        assert np.array_equal(Wd.cpu().numpy().astype(np.float64), W1), f"SFB int mismatch recon={recon}"
        assert np.array_equal(bd.cpu().numpy().astype(np.float64), b1)
        assert allsame(Wd) and allsame(bd)
        per = (M * 8 + N * 8 + M) * 4  # ldk = 8
        assert st["nccl_bytes_sent"] == per and st["nccl_bytes_recv"] == per * (P - 1), st

    # random factors (hidden-layer recipe), TF32 gate
    ctx.set_recon(pz.RECON_TF32, 0)
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P)
    Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    ctx.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, 0.5)
    ctx.wait_layer(0)
    ctx.iteration_end()
    torch.cuda.synchronize()
    W1, b1 = O.sync_step(W, b, Us, Vs, 0.5)
    check_update(W, Wd.cpu().numpy(), W1, 2e-3)
    check_update(b, bd.cpu().numpy(), b1, 1e-5)
    assert allsame(Wd)

    sfb_wire_checks(new_ctx, rank, P, dev)
    alexnet_p6_schedule_check(new_ctx, rank, P, dev, world)

    # ---- 2. PS of the same layer ----
    for variant in ("int", "rand"):
        if variant == "int":
            W, b, Us, Vs, lr = S.integer_factors(M, N, K, P, seed=5)
        else:
            W, b = S.fc_weights_randbias(M, N)
            Us, Vs = S.hidden_factors(M, N, K, P, seed=21)
            lr = 0.5
        n = M * N + M
        _, _, padded = pz.shard_range(n, P, rank)
        gflat = torch.zeros(padded, device=dev)
        wflat = torch.zeros(padded, device=dev)
        wflat[:n] = torch.from_numpy(O.flatten_params(W, b).astype(np.float32)).to(dev)
        grads = [O.flatten_params(O.reconstruct(Us[p], Vs[p]), Us[p].astype(np.float64).sum(0)).astype(np.float32)
                 for p in range(P)]
        gflat[:n] = torch.from_numpy(grads[rank]).to(dev)
        ctx.bind_ps_buffers(1, gflat, wflat, n, pz.PS_ZERO_GRAD)
        ctx.sync_ps(1, gflat, wflat, n, lr)
        ctx.wait_layer(1)
        st = ctx.iteration_end(stats=True)
        torch.cuda.synchronize()
        ref = O.ps_step_flat(O.flatten_params(W, b), grads, lr)
        out = wflat.cpu().numpy()[:n]
        if variant == "int" and P in (1, 2, 4, 8):
            assert np.array_equal(out.astype(np.float64), ref), "PS int mismatch"
        else:
            check_update(O.flatten_params(W, b), out, ref, 1e-5)
        assert allsame(wflat)
        assert float(gflat.abs().sum()) == 0.0
        S_ = padded // P
        assert st["nccl_bytes_sent"] == 2 * S_ * 4 * (P - 1)

    # ---- 3. odd sizes / empty shard ----
    ctx.register_layer(2, pz.LAYER_FC, 10, 64, 4, 1, pz.SCHEME_PS)  # n = 650
    n = 650
    g0 = S.rng(9)
    W = (g0.integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
    grads = S.integer_grads(n, P, seed=10)
    _, _, padded = pz.shard_range(n, P, rank)
    gflat = torch.full((padded,), 7.0, device=dev)   # padding holds garbage: it must be cleared too
    gflat[:n] = torch.from_numpy(grads[rank]).to(dev)
    wflat = torch.zeros(padded, device=dev)
    wflat[:n] = torch.from_numpy(W).to(dev)
    lr = 2.0 ** -7
    ctx.bind_ps_buffers(2, gflat, wflat, n, pz.PS_ZERO_GRAD)   # K2 clears the gradient in-kernel
    ctx.sync_ps(2, gflat, wflat, n, lr)
    ctx.wait_layer(2)
    ctx.iteration_end()
    torch.cuda.synchronize()
    ref = O.ps_step_flat(W, grads, lr)
    out = wflat.cpu().numpy()[:n].astype(np.float64)
    if P in (1, 2, 4, 8):
        assert np.array_equal(out, ref)
    else:
        check_update(W, out, ref, 1e-5)
    assert float(gflat.abs().sum()) == 0.0, "odd-size PS gradient not cleared"
    ctx.close()

    # ---- 3b. fused NVLS PS (f1): arena in NCCL symmetric windows, one multimem kernel per layer ----
    cn = new_ctx(pz.FLAG_NVLS_PS)
    # n = 32896, 650, 34944, 2080 (at P=2 the last shard is 1024 floats vs S=1056: unequal local
    # ranges must still launch identical grids on every rank)
    layers = [(0, 128, 256, 8), (1, 10, 64, 4), (2, 96, 363, 2), (3, 16, 129, 2)]
    for lid, M_, N_, K_ in layers:
        cn.register_layer(lid, pz.LAYER_CONV, M_, N_, K_)
    cn_lr = 2.0 ** -7
    cn.set_lr(cn_lr)
    active = cn.ps_arena()
    status = cn.nvls_status()
    if rank == 0:
        print(f"NVLS {status}", flush=True)
    for lid, M_, N_, K_ in layers:
        n = M_ * N_ + M_
        gp, wp, padded = cn.ps_layer_buffers(lid)
        from paper_1512_06216_b200.binding import device_view
        gv, wv = device_view(gp, (padded,)), device_view(wp, (padded,))
        g0 = S.rng(lid + 40)
        W = (g0.integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
        grads = S.integer_grads(n, P, seed=lid + 50)
        wv[:n].copy_(torch.from_numpy(W).to(dev))
        gv[:n].copy_(torch.from_numpy(grads[rank]).to(dev))
        torch.cuda.synchronize()
        cn.backprop_hook(lid)
        cn.wait_layer(lid)
        st = cn.iteration_end(stats=True)
        torch.cuda.synchronize()
        ref = O.ps_step_flat(W, grads, cn_lr)
        out = wv[:n].cpu().numpy().astype(np.float64)
        if P in (1, 2, 4, 8):
            assert np.array_equal(out, ref), f"NVLS PS mismatch layer {lid} ({status})"
        else:
            check_update(W, out, ref, 1e-5)
        assert allsame(wv[:n].clone())
        assert float(gv.abs().sum()) == 0.0, "grad not zeroed"
    cn.close()

    # ---- 3c. momentum + weight decay (f4) on SFB, NCCL PS and fused NVLS PS, two steps ----
    for nv in (False, True):
        cm = new_ctx(pz.FLAG_NVLS_PS if nv else 0)
        M_, N_, K_, lr_m, mu_m, wd_m = 96, 130, 8, 0.2, 0.9, 1e-2
        cm.register_layer(0, pz.LAYER_FC, M_, N_, K_)                         # SFB
        cm.register_layer(1, pz.LAYER_FC, M_, N_, K_, True, pz.SCHEME_PS)     # PS
        cm.set_lr(lr_m)
        cm.set_momentum(mu_m, wd_m)
        n = M_ * N_ + M_
        if nv:
            cm.ps_arena()
            from paper_1512_06216_b200.binding import device_view
            gp, wp, padded = cm.ps_layer_buffers(1)
            gflat, wflat = device_view(gp, (padded,)), device_view(wp, (padded,))
        else:
            _, _, padded = pz.shard_range(n, P, rank)
            gflat, wflat = torch.zeros(padded, device=dev), torch.zeros(padded, device=dev)
            cm.bind_ps_buffers(1, gflat, wflat, n, pz.PS_ZERO_GRAD)
        W, b = S.fc_weights_randbias(M_, N_)
        Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
        wflat[:n].copy_(torch.from_numpy(O.flatten_params(W, b).astype(np.float32)).to(dev))
        Wr, br = W.astype(np.float64), b.astype(np.float64)
        VW, Vb = np.zeros_like(Wr), np.zeros_like(br)
        wr, vr = O.flatten_params(W, b), np.zeros(n)
        for t in range(2):
            Us, Vs = S.hidden_factors(M_, N_, K_, P, seed=300 + 10 * t)
            cm.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, lr_m)
            grads = [O.flatten_params(O.reconstruct(Us[p], Vs[p]), Us[p].astype(np.float64).sum(0)).astype(np.float32)
                     for p in range(P)]
            gflat[:n].copy_(torch.from_numpy(grads[rank]).to(dev))
            cm.backprop_hook(1)
            cm.wait_layer(0)
            cm.wait_layer(1)
            cm.iteration_end()
            torch.cuda.synchronize()
            Wr, br, VW, Vb = O.sync_step_momentum(Wr, br, VW, Vb, Us, Vs, lr_m, mu_m, wd_m)
            wr, vr = O.ps_step_flat_momentum(wr, vr, grads, lr_m, mu_m, wd_m)
        check_update(W, Wd.cpu().numpy(), Wr, 2e-3, "SFB momentum")
        check_update(b, bd.cpu().numpy(), br, 1e-5, "SFB bias momentum")
        check_update(O.flatten_params(W, b), wflat[:n].cpu().numpy(), wr, 1e-5, f"PS momentum (nvls {nv})")
        assert allsame(Wd) and allsame(wflat[:n].clone())
        cm.close()

    # ---- 4. DWBP training steps of CIFAR-10 quick (C2 shapes): every iteration, every layer's update is
    #          recomputed by the oracle from ALL ranks' captured factors / gradients (O4 / O6, Z13 metric,
    #          tests/stepcheck.py); ranks bit-identical; DWBP on == off bitwise ----
    from stepcheck import StepCapture, oracle_check, safe_lr
    Kc = 16

    def batch(it):
        gen = torch.Generator().manual_seed(100 + it)
        xall = torch.rand(P * Kc, 3, 32, 32, generator=gen).to(dev)
        yall = torch.randint(0, 10, (P * Kc,), generator=gen).to(dev)
        return xall[rank * Kc:(rank + 1) * Kc], yall[rank * Kc:(rank + 1) * Kc]

    torch.manual_seed(1234)
    xb0, yb0 = batch(0)
    lr_c = safe_lr(CifarQuick().to(dev), lambda m: F.cross_entropy(m(xb0), yb0), world)
    results = {}
    variants = [(sc, dw, nv) for sc in ("auto", "ps") for dw in ("on", "off") for nv in (False, True)]
    variants += [("sfps", dw, False) for dw in ("on", "off")]   # every FC layer as SF-PS
    for scheme, dwbp, nv in variants:
        c2 = new_ctx((pz.FLAG_DWBP_OFF if dwbp == "off" else 0) | (pz.FLAG_NVLS_PS if nv else 0))
        torch.manual_seed(1234)
        model = CifarQuick().to(dev)
        sync = PoseidonSync(model, c2, K=Kc, lr=lr_c, scheme=scheme, recon=pz.RECON_TF32, arena=nv)
        cap = StepCapture(sync)
        for it in range(2):
            xb, yb = batch(it)
            cap.snapshot()
            loss = F.cross_entropy(model(xb), yb)
            loss.backward()
            sync.iteration_end()
            sync.wait_all()
            torch.cuda.synchronize()
            errs = oracle_check(cap, lr_c, world)
            assert len(errs) == 5, errs
        flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
        assert allsame(flat), f"ranks differ ({scheme}, dwbp {dwbp}, nvls {nv})"
        assert bool(torch.isfinite(flat).all())
        results[(scheme, dwbp, nv)] = flat.cpu()
        c2.close()
    if rank == 0:
        print(f"C2 oracle check ok (lr {lr_c:.3g}, {len(variants)} variants x 2 iterations)", flush=True)
    # the same training with the SFB inputs broadcast at forward time (FLAG_EARLY_V): bit-identical
    c2 = new_ctx(pz.FLAG_EARLY_V)
    torch.manual_seed(1234)
    model = CifarQuick().to(dev)
    sync = PoseidonSync(model, c2, K=Kc, lr=lr_c, scheme="auto", recon=pz.RECON_TF32)
    assert sync.early_v
    for it in range(2):
        xb, yb = batch(it)
        F.cross_entropy(model(xb), yb).backward()
        sync.iteration_end()
    sync.wait_all()
    torch.cuda.synchronize()
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
    assert torch.equal(flat, results[("auto", "on", False)]), "early V changed the result"
    c2.close()
    for scheme, nv in [(sc, nv) for sc in ("auto", "ps") for nv in (False, True)] + [("sfps", False)]:
        assert torch.equal(results[(scheme, "on", nv)], results[(scheme, "off", nv)]), \
            f"DWBP on/off differ ({scheme}, nvls {nv})"
    graph_checks(new_ctx, rank, P, dev, batch, lr_c, Kc)
    # ---- 6. SSP with staleness 1 (FLAG_SSP1, reading Z19): SFB + PS (arena) over 4 iterations and a
    #          flush, integer variant bit-exact vs O10, on the NCCL paths and on the NVLS paths ----
    from paper_1512_06216_b200.binding import device_view
    #          (+ staleness 2, poseidon_set_staleness, on the NVLS paths) ----
    for flags, stale in ((pz.FLAG_SSP1 | pz.FLAG_SYMM_SFB, 1), (pz.FLAG_SSP1 | pz.FLAG_NVLS_PS | pz.FLAG_NVLS_SFB, 1),
                         (pz.FLAG_SSP1 | pz.FLAG_NVLS_PS | pz.FLAG_NVLS_SFB, 2)):
        cs = new_ctx(flags)
        if stale != 1:
            cs.set_staleness(stale)
        M, N, K, T = 40, 72, 4, 5
        cs.register_layer(0, pz.LAYER_FC, M, N, K)
        cs.register_layer(1, pz.LAYER_CONV, M, N, K, True, pz.SCHEME_PS)
        cs.ps_arena()
        W, b, _, _, lr = S.integer_factors(M, N, K, P, seed=70)
        steps = []
        for t in range(T):
            _, _, Us, Vs, _ = S.integer_factors(M, N, K, P, seed=80 + t)
            steps.append((Us, Vs))
        vis = O.ssp_visible_weights(W, b, steps, lr, s=stale)
        Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
        n = M * N + M
        _, wp, padded = cs.ps_layer_buffers(1)
        wflat = device_view(wp, (padded,))
        wflat[:n] = torch.from_numpy(O.flatten_params(W, b).astype(np.float32)).to(dev)
        cs.set_lr(lr)
        torch.cuda.synchronize()
        for t, (Us, Vs) in enumerate(steps):
            cs.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, lr)
            gflat = device_view(cs.ps_layer_buffers(1)[0], (padded,))
            g = O.flatten_params(O.reconstruct(Us[rank], Vs[rank]), Us[rank].astype(np.float64).sum(0))
            gflat[:n] = torch.from_numpy(g.astype(np.float32)).to(dev)
            cs.backprop_hook(1, torch.cuda.current_stream())
            cs.wait_layer(0)
            cs.wait_layer(1)
            cs.iteration_end()
            torch.cuda.synchronize()
            Wv, bv = vis[t + 1]
            assert np.array_equal(Wd.cpu().numpy().astype(np.float64), Wv), f"SSP SFB flags={flags} t={t}"
            assert np.array_equal(bd.cpu().numpy().astype(np.float64), bv)
            assert np.array_equal(wflat[:n].cpu().numpy().astype(np.float64), O.flatten_params(Wv, bv)), \
                f"SSP PS flags={flags} t={t}"
        cs.flush()
        cs.wait_layer(0)
        cs.wait_layer(1)
        torch.cuda.synchronize()
        Wf, bf = vis[T + stale]
        assert np.array_equal(Wd.cpu().numpy().astype(np.float64), Wf)
        assert np.array_equal(wflat[:n].cpu().numpy().astype(np.float64), O.flatten_params(Wf, bf))
        assert allsame(Wd) and allsame(wflat)
        if rank == 0:
            print(f"SSP flags={flags} s={stale}: PS {cs.nvls_status()}, SFB path {cs.sfb_path(0)}", flush=True)
        cs.close()

    # ---- 7. PS buckets (f1): small PS layers synced as one flat buffer, NCCL and fused NVLS paths;
    #          integer variant bit-exact vs O6 per layer, gradients cleared, ranks identical ----
    shapes = [(10, 65), (32, 64), (3, 1), (96, 363), (16, 129), (500, 400)]
    for flags in (0, pz.FLAG_NVLS_PS):
        cb = new_ctx(flags)
        for lid, (M_, N_) in enumerate(shapes):
            cb.register_layer(lid, pz.LAYER_CONV, M_, N_, 1, True, pz.SCHEME_PS)
        cb.set_ps_buckets(256 * 1024)
        cb.ps_arena()
        lr = 2.0 ** -7
        cb.set_lr(lr)
        refs, views = [], []
        for lid, (M_, N_) in enumerate(shapes):
            n = M_ * N_ + M_
            gp, wp, padded = cb.ps_layer_buffers(lid)
            grads = S.integer_grads(n, P, seed=200 + lid)
            w0 = (S.rng(300 + lid).integers(-1023, 1024, size=n) * 2.0 ** -10).astype(np.float32)
            wv, gv = device_view(wp, (padded,)), device_view(gp, (padded,))
            wv[:n] = torch.from_numpy(w0).to(dev)
            gv[:n] = torch.from_numpy(grads[rank]).to(dev)
            refs.append((w0, O.ps_step_flat(w0, grads, lr)))
            views.append((wv, gv, n))
        torch.cuda.synchronize()
        dist.barrier()
        for lid in reversed(range(len(shapes))):
            cb.backprop_hook(lid, torch.cuda.current_stream())
        for lid in range(len(shapes)):
            cb.wait_layer(lid)
        st = cb.iteration_end(stats=True)
        torch.cuda.synchronize()
        for (wv, gv, n), (w0, ref) in zip(views, refs):
            out = wv[:n].cpu().numpy().astype(np.float64)
            if P in (1, 2, 4, 8):
                assert np.array_equal(out, ref), f"bucket PS flags={flags}"
            else:
                check_update(w0, out, ref, 1e-5)
            assert float(gv[:n].abs().sum()) == 0.0
            assert allsame(wv[:n].contiguous())
        assert st["n_layers"] < len(shapes), st
        if rank == 0:
            print(f"buckets flags={flags}: {st['n_layers']} syncs for {len(shapes)} layers, PS {cb.nvls_status()}",
                  flush=True)
        cb.close()

    # ---- 8. SF-PS (Alg. 3 else-branch, reading Z20): U rows to their masters, V all-gathered, K1 on the
    #          master's rows, masters broadcast their rows.  Integer variant bit-exact vs O11 (both
    #          kernels, plain and symmetric-window buffers, DWBP off), three shapes: C1, M=40 (masters with
    #          8 rows and with none at P=4), fc8-like 1000 x 4096 with ragged K; 2 iterations; bytes ----
    for flags in (0, pz.FLAG_SYMM_SFB, pz.FLAG_DWBP_OFF):
        cp = new_ctx(flags)
        shapes = [(0, 128, 256, 8), (1, 40, 72, 4), (2, 1000, 4096, 33)]
        for lid, M_, N_, K_ in shapes:
            assert cp.register_layer(lid, pz.LAYER_FC, M_, N_, K_, True, pz.SCHEME_SFPS) == pz.SCHEME_SFPS
            assert cp.sfb_path(lid) == pz.SFB_PATH_SFPS
        for it in range(2):
            cp.set_recon(pz.RECON_FP32 if it == 1 else pz.RECON_TF32)
            outs = []
            for lid, M_, N_, K_ in shapes:
                W, b, Us, Vs, lr = S.integer_factors(M_, N_, K_, P, seed=900 + 10 * it + lid)
                Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
                cp.sync_fc_sfb(lid, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, lr)
                outs.append((W, b, Us, Vs, lr, Wd, bd))
            st = cp.iteration_end(stats=True)
            for lid, (W, b, Us, Vs, lr, Wd, bd) in enumerate(outs):
                cp.wait_layer(lid)
            torch.cuda.synchronize()
            for lid, (W, b, Us, Vs, lr, Wd, bd) in enumerate(outs):
                W11, b11, _ = O.sf_ps_simulated(W, b, Us, Vs, lr)
                assert np.array_equal(Wd.cpu().numpy().astype(np.float64), W11), f"SF-PS flags={flags} it={it} lid={lid}"
                assert np.array_equal(bd.cpu().numpy().astype(np.float64), b11)
                assert allsame(Wd) and allsame(bd)
            # bytes through NCCL per rank: V + bias sums all-gathered, U rows to / from the masters,
            # the masters' rows broadcast
            exp_sent = exp_recv = 0
            for lid, M_, N_, K_ in shapes:
                ldk = (K_ + 3) // 4 * 4
                if P == 1:
                    continue
                rows = [pz.shard_range(M_, P, q)[:2] for q in range(P)]
                own = rows[rank][1] - rows[rank][0]
                exp_sent += (N_ * ldk + M_) * 4 + sum((e - b_) * ldk * 4 for q, (b_, e) in enumerate(rows) if q != rank) \
                    + own * N_ * 4
                exp_recv += (N_ * ldk + M_) * 4 * (P - 1) + own * ldk * 4 * (P - 1) \
                    + sum((e - b_) * N_ * 4 for q, (b_, e) in enumerate(rows) if q != rank)
            assert st["nccl_bytes_sent"] == exp_sent and st["nccl_bytes_recv"] == exp_recv, (st, exp_sent, exp_recv)
        cp.close()
    # random factors + momentum (two steps, TF32 gate vs O4m, which O11 equals) and FLAG_SFPS auto-selection
    cp = new_ctx(pz.FLAG_SFPS)
    M_, N_, K_, lr_m, mu_m, wd_m = 300, 520, 16, 0.2, 0.9, 1e-2
    cp.register_layer(0, pz.LAYER_FC, M_, N_, K_, True, pz.SCHEME_SFPS)
    expect_auto = pz.SCHEME_SFB if P <= 2 else pz.SCHEME_SFPS   # C2 ip2 10x64, K=100: rule PS at P >= 3
    assert cp.register_layer(1, pz.LAYER_FC, 10, 64, 100) == expect_auto
    assert cp.register_layer(2, pz.LAYER_CONV, 10, 64, 100) == pz.SCHEME_PS
    cp.set_lr(lr_m)
    cp.set_momentum(mu_m, wd_m, 0)
    W, b = S.fc_weights_randbias(M_, N_)
    Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    Wr, br = W.astype(np.float64), b.astype(np.float64)
    VW, Vb = np.zeros_like(Wr), np.zeros_like(br)
    for t in range(2):
        Us, Vs = S.hidden_factors(M_, N_, K_, P, seed=950 + t)
        cp.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, lr_m)
        cp.wait_layer(0)
        cp.iteration_end()
        Wr, br, VW, Vb = O.sync_step_momentum(Wr, br, VW, Vb, Us, Vs, lr_m, mu_m, wd_m)
    torch.cuda.synchronize()
    check_update(W, Wd.cpu().numpy(), Wr, 2e-3, "SF-PS momentum")
    check_update(b, bd.cpu().numpy(), br, 1e-5, "SF-PS bias momentum")
    assert allsame(Wd) and allsame(bd)
    cp.close()

    early_v_checks(new_ctx, rank, P, dev)
    # ---- 5. full size in bench.py's N > 1 launch configuration (NVLS_SFB | NVLS_PS): C3 fc6 as SFB
    #          (4096 x 9216, K = 256) and a 37.7M-parameter PS layer in the NVLS arena, sampled against
    #          the oracle (O4 rows / O6 elements) ----
    cf = new_ctx(pz.FLAG_NVLS_SFB | pz.FLAG_NVLS_PS)
    M, N, K = 4096, 9216, 256
    assert cf.register_layer(0, pz.LAYER_FC, M, N, K) == pz.SCHEME_SFB
    cf.register_layer(1, pz.LAYER_CONV, M, N, 1, True, pz.SCHEME_PS)
    cf.ps_arena()
    W, b = S.fc_weights_randbias(M, N)
    Us, Vs = S.hidden_factors(M, N, K, P, seed=500)
    Wd, bd = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    cf.sync_fc_sfb(0, torch.from_numpy(Us[rank]).to(dev), torch.from_numpy(Vs[rank]).to(dev), Wd, bd, 0.5)
    cf.wait_layer(0)
    n = M * N + M
    gp, wp, padded = cf.ps_layer_buffers(1)
    from paper_1512_06216_b200.binding import device_view
    gv, wv = device_view(gp, (padded,)), device_view(wp, (padded,))
    grads = S.dense_grads(n, P, seed=600)
    # W of the same order as the update (tests/parity.py: the fp32 ulp excuse stays < 0.1 x gate)
    w0 = w0_like(S.rng(601).standard_normal(n), 0.05 / P * np.sum(grads, axis=0, dtype=np.float64))
    wv[:n] = torch.from_numpy(w0).to(dev)
    gv[:n] = torch.from_numpy(grads[rank]).to(dev)
    torch.cuda.synchronize()
    dist.barrier()
    cf.set_lr(0.05)
    cf.backprop_hook(1, torch.cuda.current_stream())
    cf.wait_layer(1)
    cf.iteration_end()
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, 1, 255, 256, M - 1], S.rng(502).integers(0, M, 43)]))
    Wr, br = O.sync_step_rows(W[rows], b[rows], Us, Vs, 0.5, rows)
    Wout = Wd.cpu().numpy()
    assert O.update_error(W[rows], Wout[rows], Wr) <= 2e-3, "full-size SFB (broadcast kernel) off the TF32 gate"
    check_update(b[rows], bd.cpu().numpy()[rows], br, 1e-5)
    assert allsame(Wd) and allsame(bd)
    idx = np.unique(np.concatenate([[0, n - 1, n // P, padded // P - 1], S.rng(603).integers(0, n, 4093)]))
    idx = idx[idx < n]
    ref = O.ps_step_flat(w0[idx], [g[idx] for g in grads], 0.05)
    out = wv[:n].cpu().numpy()[idx]
    check_update(w0[idx], out, ref, 1e-5, "full-size NVLS PS off the 1e-5 gate")
    assert allsame(wv[:n].contiguous())
    assert float(gv.abs().sum()) == 0.0
    if rank == 0:
        print(f"full-size: SFB path {cf.sfb_path(0)}, PS {cf.nvls_status()}", flush=True)
    del grads
    cf.close()

    dist.barrier()
    print(f"MP_OK {rank}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
