"""Summarise `ncu --set full` reports into JSON (committed under profiles/).

  python tools/ncu_summary.py gpurun_out/ncu_tree.ncu-rep [...] --out profiles/r1/ncu_summary.json

Per profiled launch: kernel, grid/block, duration, DRAM bytes read/written,
achieved DRAM GB/s and % of peak, tensor-pipe / UTCHMMA utilisation, SM and
L2 throughput %, registers and shared memory.
"""

import argparse
import csv
import io
import json
import pathlib
import subprocess

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us when unit is ns (ncu raw csv reports in ns)
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "utchmma_pct": ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_mhz": ("sm__cycles_elapsed.avg.per_second", 1),
    "registers": ("launch__registers_per_thread", 1),
    "smem_per_block_kb": ("launch__shared_mem_per_block", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}


def raw_rows(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarise(rep: str) -> list[dict]:
    res = []
    for d in raw_rows(rep):
        r = {"report": pathlib.Path(rep).name, "kernel": d.get("Kernel Name", "")[:120]}
        for k, (m, _) in METRICS.items():
            r[k] = num(d.get(m))
        if r["duration_us"] is not None:
            r["duration_us"] = r["duration_us"] / 1e3  # base unit ns
        if r["sm_mhz"] is not None:
            r["sm_mhz"] = r["sm_mhz"] / 1e6
        if r["dram_read_bytes"] is not None and r["duration_us"]:
            tot = (r["dram_read_bytes"] or 0) + (r["dram_write_bytes"] or 0)
            r["dram_bytes"] = tot
            r["dram_gbs"] = tot / (r["duration_us"] * 1e-6) / 1e9
        res.append(r)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    allr = []
    for rep in a.reports:
        allr += summarise(rep)
    for r in allr:
        print(f"{r['kernel'][:48]:48s} {r['duration_us'] or 0:9.1f} us  dram {((r.get('dram_bytes') or 0) / 1e6):9.2f} MB "
              f"{r.get('dram_gbs') or 0:8.0f} GB/s ({r['dram_throughput_pct'] or 0:5.1f}%)  tensor {r['tensor_pipe_pct'] or 0:5.1f}%"
              f"  sm {r['sm_throughput_pct'] or 0:5.1f}%  clk {r['sm_mhz'] or 0:6.0f}")
    if a.out:
        pathlib.Path(a.out).write_text(json.dumps(allr, indent=1))


if __name__ == "__main__":
    main()
