"""Render tools/layer_roofline.py JSON lines (one file per P) as the markdown tables in profiles/.

    python tools/layer_roofline_md.py out.md P1.jsonl P2.jsonl P4.jsonl

Two bounds per layer:
  bandwidth roof  SFB: (P-1)K(M+N)4/BW_nvl + max(2MNPK/TC, (8MN + 4PK(M+N) + 8M)/BW_hbm)
                  PS:  2(P-1)/P 4n/BW_nvl + 12n/P/BW_hbm
                  SF-PS (R = ceil(M/P) rows per master): ((P-1)K(N+R) + (M-R)N)4/BW_nvl
                       + max(2RNPK/TC, (8RN + 4PK(R+N))/BW_hbm)
  effective roof  each term raised to its latency floor: a collective costs at least alpha (SFB: one
                  all-gather; PS: reduce-scatter + all-gather = 2 alpha; SF-PS: factor exchange + row push =
                  3 alpha), a kernel at least T_LAUNCH.
alpha = the 8-byte NCCL all-gather measured in the same run; T_LAUNCH = 2 us.
"""
import json
import sys

# round 2: TF32 = max(bf16 burst x 1.1/2.25, measured cuBLAS TF32) and HBM from MEASURED_PEAKS.json (bench.py)
TC_TF32, BW_HBM, BW_NVL, T_LAUNCH = 807.9e12, 6458.7e9, 900e9, 2e-6


def bounds(d, P, alpha, bw_nvl=BW_NVL):
    M, N, K, n = d["M"], d["N"], d["K"], d["n"]
    BW = bw_nvl
    if d["scheme"] == "sfps":
        R = -(-M // P)
        comm = ((P - 1) * K * (N + R) + (M - R) * N) * 4 / BW
        kern = max(2.0 * R * N * P * K / TC_TF32, (8.0 * R * N + 4.0 * P * K * (R + N)) / BW_HBM)
        comm_eff = max(comm, 3 * alpha)
    elif d["scheme"] == "sfb":
        comm = (P - 1) * K * (M + N) * 4 / BW
        kern = max(2.0 * M * N * P * K / TC_TF32, (8.0 * M * N + 4.0 * P * K * (M + N) + 8.0 * M) / BW_HBM)
        comm_eff = max(comm, alpha) if P > 1 else 0.0
    else:
        comm = 2.0 * (P - 1) / P * 4 * n / BW
        kern = 12.0 * n / P / BW_HBM
        comm_eff = max(comm, 2 * alpha) if P > 1 else 0.0
    return (comm + kern) * 1e6, (comm_eff + max(kern, T_LAUNCH)) * 1e6


def main():
    out, files = sys.argv[1], sys.argv[2:]
    lines = ["# Per-layer sync vs its roofline, each layer in isolation (round 1)", "",
             "`tools/layer_roofline.py` under torchrun, rendered by `tools/layer_roofline_md.py` (median of 50",
             "syncs per layer, max over ranks; a ~100 us device spin precedes each sync so all of its launches are",
             "queued; time = the library's device events start -> done).  `bw roof`: SURVEY §8(d) bandwidth",
             "roofline (NVLink 5 900 GB/s, TF32 794 TFLOP/s, HBM 6543.7 GB/s).  `eff roof`: the same with every",
             "collective raised to the measured 8-byte NCCL latency alpha (PS: 2 alpha) and every kernel to 2 us.",
             "ps_nccl = NCCL reduce-scatter + K2 + all-gather; ps_nvls = the fused multimem kernel; sfb = the library's",
             "factor broadcast kernel (bench default at P > 1) + K1; `meas roof`: the effective roof with NVLink at the busbw NCCL itself",
             "reaches for 256 MB all-gathers in the same run (SURVEY §8(d): against the spec and the measured peak);",
             "sfps = the literal else-branch of Alg. 3 (reading Z20): U rows to",
             "their masters, V all-gathered, K1 on the master's rows, rows pushed back.", ""]
    for f in files:
        L = [json.loads(l) for l in open(f) if l.startswith("{")]
        head = [d for d in L if "alpha_us" in d][0]
        P, alpha = head["P"], head["alpha_us"] * 1e-6
        lines.append(f"## P = {P}  (alpha = {head['alpha_us']} us; NCCL all-gather busbw at 256 MB = "
                     f"{head['bw_nvl_measured_GBps']} GB/s)")
        lines.append("")
        lines.append("| layer | M x N | path | measured us | bw roof us | frac | eff roof us | frac of eff | "
                     "meas roof us | frac of meas |")
        lines.append("|---|---|---|---:|---:|---:|---:|---:|---:|---:|")
        bw_meas = head["bw_nvl_measured_GBps"] * 1e9
        c4 = {}
        for d in L:
            if "layer" not in d:
                continue
            bw, eff = bounds(d, P, alpha)
            meas = bounds(d, P, alpha, bw_meas)[1]
            t = d["measured_us"]
            if d["layer"].startswith("C4"):
                a = c4.setdefault(d["scheme"], [0, 0.0, 0.0, 0.0, 0.0])
                a[0] += 1
                a[1] += t
                a[2] += bw
                a[3] += eff
                a[4] += meas
                continue
            lines.append(f"| {d['layer']} | {d['M']} x {d['N']} | {d['scheme']} | {t:.1f} | {bw:.1f} | {bw / t:.3f} | "
                         f"{eff:.1f} | {eff / t:.3f} | {meas:.1f} | {meas / t:.3f} |")
        for sch, (cnt, t, bw, eff, meas) in sorted(c4.items()):
            lines.append(f"| C4 GoogLeNet ({cnt} layers, summed) | - | {sch} | {t:.1f} | {bw:.1f} | {bw / t:.3f} | "
                         f"{eff:.1f} | {eff / t:.3f} | {meas:.1f} | {meas / t:.3f} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
