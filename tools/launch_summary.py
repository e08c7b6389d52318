"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch): libposeidon kernels per name with
per-launch times and grids, and the share of all device time.  python tools/launch_summary.py FILE.csv"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                out.append(d)
    return out


if __name__ == "__main__":
    L = load(sys.argv[1])
    tot = sum(float(d["Metric Value"]) for d in L)
    agg = collections.defaultdict(list)
    for d in L:
        agg[d["Kernel Name"].split("(")[0]].append((float(d["Metric Value"]) / 1e3, d["Grid Size"]))
    print(f"{len(L)} launches, {tot / 1e3:.1f} us device time (serialised ncu replay)")
    mine = 0.0
    for k, v in sorted(agg.items(), key=lambda kv: -sum(x[0] for x in kv[1])):
        if "poseidon" not in k:
            continue
        s = sum(x[0] for x in v)
        mine += s
        print(f"{s:9.1f} us {len(v):3d}x {100 * s / (tot / 1e3):5.2f}%  {k.replace('void poseidon::<unnamed>::', '')}: "
              + " ".join(f"{t:.2f}{g.replace(' ', '')}" for t, g in v[:9]))
    print(f"libposeidon total {mine:.1f} us = {100 * mine / (tot / 1e3):.2f}% of device time")
