"""Per-kernel GPU time of one SpecExec target iteration (C2 by default) via the
CUDA profiler interface of torch.profiler (CUPTI kernel records; no nsys here).

  python tools/profile_step.py [--workload c2] [--json out.json]
"""

import argparse
import collections
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2406_02532_b200 as sx  # noqa: E402
from paper_2406_02532_b200.engine import SpecExecSession  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--json", default=None)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    dname, tname, K, D, B, temp, top_p = bench.WORKLOADS[a.workload]
    offload = a.workload in bench.OFFLOAD
    target = LlamaModel(tname, seed=1, max_ctx=4096, max_tokens=K + 1, offload=offload)
    draft = LlamaModel(dname, seed=2, max_ctx=8192 + 4 * K, max_tokens=max(B, 128))
    prompt = tuple(int(t) for t in np.random.default_rng(1000).integers(0, PRESETS[tname].vocab, size=128))
    cfg = sx.SamplingConfig(temp, top_p, seed=0, max_new_tokens=100000)
    sess = SpecExecSession(prompt, draft, target, sx.BuilderParams(K, D, B), cfg, temp != 0.0)
    for _ in range(3):
        sess.step(100000)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]
    with torch.profiler.profile(activities=acts) as prof:
        n = 0
        while n < a.steps:
            sess.step(100000)
            if sess.cache is None:
                n += 1
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.split("(")[0].replace("void ", "")
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    total = sum(v[1] for v in agg.values())
    rows = sorted(((k, c, t) for k, (c, t) in agg.items()), key=lambda r: -r[2])
    print(f"total GPU kernel time {total / 1e3 / a.steps:.2f} ms per step over {a.steps} step(s)")
    for k, c, t in rows[:25]:
        print(f"{t / 1e3 / a.steps:9.3f} ms {100 * t / total:5.1f}%  {c // a.steps:6d}x  {k[:90]}")
    if a.json:
        pathlib.Path(a.json).write_text(json.dumps({"total_ms_per_step": total / 1e3 / a.steps,
                                                    "kernels": [{"name": k, "launches": c, "ms": t / 1e3}
                                                                for k, c, t in rows]}, indent=1))


if __name__ == "__main__":
    main()
