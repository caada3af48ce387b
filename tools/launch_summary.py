"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and the target / draft split of one SpecExec iteration.

  python tools/launch_summary.py gpurun_out/launches_c2.csv --out profiles/r1/launches_c2_summary.json
"""

import argparse
import collections
import csv
import json
import pathlib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", default=None)
    ap.add_argument("--only-sx", action="store_true", default=True)
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    seq = []
    for r in rows[1:]:
        name = r[ki]
        if a.only_sx and "sx::" not in name and "gemm_tc" not in name:
            continue
        short = name.split("(")[0].replace("void ", "").replace("sx::", "")
        seq.append((short, float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, us in seq:
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    out = {"source": a.csv, "note": "ncu serialised, cold-cache per launch: compare shares, not absolutes",
           "total_us": tot, "kernels": []}
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out["kernels"].append({"kernel": k, "launches": n, "us": us, "share": us / tot})
        print(f"{k:45s} {n:6d} {us / 1e3:9.2f} ms {100 * us / tot:6.2f}%")
    if a.out:
        pathlib.Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
