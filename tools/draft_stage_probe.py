"""The draft stage of one C2 iteration in isolation: build_sssp on the 7B draft
after a few SpecExec iterations (so the draft KV holds a realistic prefix and a
pending catch-up chain), timed with CUDA events and host wall time, plus the
CUPTI kernel totals of one build (torch.profiler).

  python tools/draft_stage_probe.py [--workload c2] [--builds 5]
"""

import argparse
import collections
import json
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2406_02532_b200 as sx  # noqa: E402
from paper_2406_02532_b200.engine import SpecExecSession  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel  # noqa: E402
from paper_2406_02532_b200.tree import build_sssp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--builds", type=int, default=5)
    a = ap.parse_args()
    dname, tname, K, D, B, temp, top_p = bench.WORKLOADS[a.workload]
    draft = LlamaModel(dname, seed=2, max_ctx=8192 + 4 * K, max_tokens=max(B, 128))
    # a small target of the same vocabulary drives the walk (only the draft stage is measured)
    target = LlamaModel(dname, seed=1, max_ctx=4096, max_tokens=K + 1)
    prompt = tuple(int(t) for t in np.random.default_rng(1000).integers(0, PRESETS[tname].vocab, size=128))
    cfg = sx.SamplingConfig(temp, top_p, seed=0, max_new_tokens=100000)
    params = sx.BuilderParams(K, D, B)
    sess = SpecExecSession(prompt, draft, target, params, cfg, temp != 0.0)
    for _ in range(3):
        sess.step(100000)
    torch.cuda.synchronize()
    prefix = sess.prompt + tuple(sess.tokens)
    warp = cfg if temp != 0.0 else None
    out = []
    for i in range(a.builds + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        tree = build_sssp(prefix, draft, params, warp, temp != 0.0)
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i > 0:
            out.append((e0.elapsed_time(e1), (t1 - t0) * 1e3, tree.rounds, len(tree.nodes)))
        # the next build re-runs the same prefix (the draft KV past the prefix is scratch)
    acts = [torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]
    with torch.profiler.profile(activities=acts) as prof:
        build_sssp(prefix, draft, params, warp, temp != 0.0)
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.split("(")[0].replace("void ", "")
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total
    tot = sum(v[1] for v in agg.values()) / 1e3
    rec = {"workload": a.workload, "device_ms": [round(x[0], 3) for x in out], "host_ms": [round(x[1], 3) for x in out],
           "rounds": out[0][2], "nodes": out[0][3], "kernel_ms_total": round(tot, 3),
           "kernels": [{"name": k[:80], "n": c, "ms": round(t / 1e3, 3)}
                       for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]]}
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
