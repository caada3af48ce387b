"""B200 cost-model preset from measured numbers.

Writes a preset in the schema of the reference's costsim presets
(pkg/src/speckit/presets/*.json; CostModel pkg/src/speckit/costsim.py:25-56)
from this repository's bench lines, and checks the reference's pass-cost model
forward_time (costsim.py:59-65: overhead + max((1 - prefetch) * bytes / bw,
n / compute_rate)) against the measured offloaded target pass.

  python tools/costsim_preset.py profiles/r1/bench_c2.json profiles/r1/bench_c3.json \
      --out profiles/r1/costsim_b200_70b.json
"""

import argparse
import json
import pathlib
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("resident", help="bench line of the resident target (C2)")
    ap.add_argument("offload", help="bench line of the offloaded target (C3)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c2 = json.loads(pathlib.Path(a.resident).read_text())
    c3 = json.loads(pathlib.Path(a.offload).read_text())
    k2 = int(re.search(r"K=(\d+)", c2["config"]["workload"]).group(1))
    k3 = int(re.search(r"K=(\d+)", c3["config"]["workload"]).group(1))
    tgt_ms = c2["stage_ms_per_step"]["target"]
    compute_rate = (k2 + 1) / (tgt_ms / 1e3)  # tokens/s of the resident target pass
    bw = c3["roofline"]["peak"] * 1e9  # measured pinned H2D bytes/s
    target_bytes = c3["roofline"]["bytes_per_step"]
    draft_calls = c3["draft_calls_per_iter"]
    draft_step = c3["stage_ms_per_step"]["draft"] / 1e3 / max(1.0, draft_calls)
    # LayerStreamer: its ring of staging slots loads the next pass's first layers while the draft
    # runs -- as many as the ring holds or the draft phase leaves time for, whichever is less
    ring = float(c3["config"].get("offload_buffers", 2)) / 80.0
    prefetch = min(ring, (c3["stage_ms_per_step"]["draft"] / 1e3) * bw / c3["roofline"]["bytes_per_step"])
    preset = {"target_bytes": target_bytes, "bandwidth": bw, "compute_rate": compute_rate,
              "draft_bytes": 13.48e9, "fixed_overhead": 0.0, "prefetch_fraction": prefetch,
              "draft_step_time": draft_step}
    n = k3 + 1
    load = (1 - prefetch) * target_bytes / bw
    model = max(load, n / compute_rate)  # costsim.forward_time (overhead 0)
    measured = c3["stage_ms_per_step"]["target"] / 1e3
    report = {"preset": preset, "check": {"n_tokens": n, "forward_time_model_s": model,
                                          "forward_time_measured_s": measured,
                                          "crossover_tokens": compute_rate * load}}
    print(json.dumps(report, indent=1))
    if a.out:
        pathlib.Path(a.out).write_text(json.dumps(report, indent=1) + "\n")


if __name__ == "__main__":
    main()
