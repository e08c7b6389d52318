"""Summarise ncu outputs into the tracked profiles/ directory.

    python tools/ncu_summary.py launches gpurun_out/launches_r1.csv [--last-iters N] > profiles/launches_r1.md
    python tools/ncu_summary.py full gpurun_out/k1_full_r1.ncu-rep > profiles/k1_full_r1.txt
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

OURS = ("poseidon", "recon_tcgen05", "recon_simt", "ps_shard_sgd", "pack_t_kernel", "pack_uv_kernel", "bias_update", "ps_sim")


def short(name):
    for key in ("recon_tcgen05_2sm_kernel", "recon_tcgen05_kernel", "recon_simt_kernel", "ps_shard_sgd_kernel", "ps_shard_sgd_scalar",
                "pack_t_kernel", "pack_uv_kernel", "bias_update_kernel", "bias_momentum_kernel", "ps_sim_kernel", "ps_nvls_kernel",
                "sfb_bcast_kernel", "ps_momentum_kernel", "momentum_apply_kernel"):
        if key in name:
            return key + (" [libposeidon]")
    if "nccl" in name.lower():
        return name.split("(")[0][:60] + " [NCCL]"
    return name.split("(")[0][:80]


def launches(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    total = sum(float(r["Metric Value"]) for r in rows)
    agg = OrderedDict()
    for r in rows:
        k = short(r["Kernel Name"])
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + float(r["Metric Value"]))
    ours = sum(t for k, (c, t) in agg.items() if "[libposeidon]" in k)
    print(f"# ncu launch list: {path}\n")
    print(f"{len(rows)} launches, {total/1e3:.1f} us total device time (serialised, cold-cache ncu replay; "
          "compare SHARES, not absolutes). libposeidon kernels: "
          f"{ours/1e3:.1f} us = {100*ours/total:.2f}% of device time.\n")
    print("| kernel | launches | total us | share | mean us |")
    print("|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {t/1e3:.1f} | {100*t/total:.2f}% | {t/c/1e3:.2f} |")
    print("\n## libposeidon launches in order\n")
    print("| # | kernel | grid | block | us |")
    print("|---|---|---|---|---|")
    for r in rows:
        k = short(r["Kernel Name"])
        if "[libposeidon]" in k:
            print(f"| {r['ID']} | {k} | {r['Grid Size']} | {r['Block Size']} | {float(r['Metric Value'])/1e3:.2f} |")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg",
        "smsp__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpc__cycles_elapsed.max", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "lts__d_sectors.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {path}\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## {d.get('Kernel Name', '?')[:120]}\n")
        for k in KEYS:
            for h in hdr:
                if h == k or h.endswith("." + k) or (k in h and h.split(".")[-1] == k.split(".")[-1] and k in h):
                    print(f"- {h} = {d[h]} {u[h]}")
                    break
        rd = wr = 0.0
        for h in hdr:
            if h == "dram__bytes_read.sum":
                rd = float(d[h]) * (1e6 if u[h] == "Mbyte" else 1e3 if u[h] == "Kbyte" else 1e9 if u[h] == "Gbyte" else 1)
            if h == "dram__bytes_write.sum":
                wr = float(d[h]) * (1e6 if u[h] == "Mbyte" else 1e3 if u[h] == "Kbyte" else 1e9 if u[h] == "Gbyte" else 1)
        print(f"- traffic (dram read + write) = {rd + wr:.0f} bytes\n")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        launches(path)
    else:
        full(path)
