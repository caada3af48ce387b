"""Stage-1 selection kernels (sx_tree_round: row statistics + scoring + the
update) on synthetic fp32 logits rows, per round, against the HBM roofline of
B x V x 4 bytes read per round. A build = root round + rounds of
B rows until the batch empties (rows N(0, scale) per round, like random-init
drafts: scale ~1.3). Prints one JSON line per configuration; `--impl` 1 = the
two-kernel path (A/B). GPU tool (ncu: one round per launch list).

  python tools/tree_round_bench.py --V 32000 --K 1024 --B 1024
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402
from paper_2406_02532_b200._lib import SCORE_RAW  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--V", type=int, default=32000)
    ap.add_argument("--K", type=int, default=1024)
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--D", type=int, default=16)
    ap.add_argument("--scale", type=float, default=1.3)
    ap.add_argument("--builds", type=int, default=5)
    ap.add_argument("--impl", type=int, default=0)
    ap.add_argument("--trace", action="store_true", help="print the update kernel's phase stamps (a make TRACE=1 build)")
    ap.add_argument("--graph", type=int, default=1, help="replay each round's launches as a CUDA graph (as the draft's fused round does)")
    a = ap.parse_args()
    _lib.call("sx_tree_set_impl", a.impl)
    peak = 6549.4
    try:
        peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
    except OSError:
        pass
    ws = K.TreeWorkspace(a.K, a.B, a.V, a.D)
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = torch.empty((a.B, a.V), device="cuda")
    per_round = []  # (batch_n, ms)
    traces = []
    graph = None
    for bi in range(a.builds + 1):
        ws.begin()
        n = 1
        while True:
            rows[:n].normal_(0.0, a.scale, generator=g)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if a.graph and graph is None and bi > 0 and n == a.B:
                graph = torch.cuda.CUDAGraph()  # captured once the static launch state is warm
                with torch.cuda.graph(graph):
                    ws.launch_round(rows, SCORE_RAW)
                ws.begin()  # the capture did not run; restart this build
                n = 1
                rows[:n].normal_(0.0, a.scale, generator=g)
            e0.record()
            if graph is not None and n == a.B:
                graph.replay()
            else:
                ws.launch_round(rows, SCORE_RAW)
            e1.record()
            ctl = ws.read_ctl()
            if bi > 0:
                per_round.append((n, e0.elapsed_time(e1)))
                if a.trace:
                    o = ws.off["r_aux"] + 64
                    t = ws.buf[o : o + 80].view(torch.int64).cpu().tolist()
                    traces.append({"batch": n, "us_from_start": [round((x - t[0]) / 1e3, 2) if x else None for x in t]})
            n = ctl["batch_n"]
            if n == 0:
                break
    full = [(n, ms) for n, ms in per_round if n == a.B]
    out = {"V": a.V, "K": a.K, "B": a.B, "scale": a.scale, "impl": "fused" if a.impl == 0 else "row_stats+score",
           "graph": bool(a.graph),
           "rounds_per_build": len(per_round) / a.builds}
    if full:
        ms = sum(x for _, x in full) / len(full)
        gbs = a.B * a.V * 4 / (ms / 1e3) / 1e9
        out.update({"full_rounds": len(full), "us_per_full_round": ms * 1e3, "bytes_per_round": a.B * a.V * 4,
                    "achieved_GBps": gbs, "hbm_peak_GBps": peak, "frac": gbs / peak})
    out["us_per_round_all"] = [round(x * 1e3, 1) for _, x in per_round[: 12]]
    out["batch_sizes"] = [n for n, _ in per_round[: 12]]
    if a.trace:
        out["update_phase_us"] = traces[:12]
    print(json.dumps(out))


main()
