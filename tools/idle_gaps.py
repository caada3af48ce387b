"""GPU idle gaps inside one SpecExec iteration (C2 by default): kernel records
from torch.profiler (CUPTI), gaps between consecutive kernels/memcpys on the
device timeline, attributed to the host-side phase (record_function ranges
around the engine's stages) that was running when each gap began.

  python tools/idle_gaps.py [--workload c2] [--steps 2]
"""

import argparse
import collections
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
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--min-us", type=float, default=20.0)
    a = ap.parse_args()
    dname, tname, K, D, B, temp, top_p = bench.WORKLOADS[a.workload]
    target = LlamaModel(tname, seed=1, max_ctx=4096, max_tokens=K + 1)
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
            with torch.profiler.record_function("sx::step"):
                sess.step(100000)
            if sess.cache is None:
                n += 1
        torch.cuda.synchronize()
    kern, ranges = [], []
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            kern.append((ev.time_range.start, ev.time_range.end, ev.name.split("(")[0][-40:]))
        elif ev.name.startswith("sx::"):
            ranges.append((ev.time_range.start, ev.time_range.end, ev.name))
    kern = sorted(set(kern))  # the profiler can report a record twice
    union, cur_s, cur_e = 0.0, None, None  # busy = union of the device intervals (PDL overlaps grids)
    for s, e, _ in kern:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                union += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    union += cur_e - cur_s
    span = kern[-1][1] - kern[0][0]
    print(f"device span {span / 1e3 / a.steps:.2f} ms/step, device busy (union) {union / 1e3 / a.steps:.2f} ms/step, "
          f"idle {(span - union) / 1e3 / a.steps:.2f} ms/step")
    gaps = collections.defaultdict(lambda: [0, 0.0])
    big = []
    run_end, run_name = kern[0][1], kern[0][2]
    for s1, e1, n1 in kern[1:]:
        g, n0 = s1 - run_end, run_name  # gap after everything that started earlier has ended
        if e1 >= run_end:
            run_end, run_name = e1, n1
        if g < a.min_us:
            continue
        key = f"{n0} -> {n1}"
        gaps[key][0] += 1
        gaps[key][1] += g
        big.append((g, key))
    tot = sum(v[1] for v in gaps.values())
    print(f"gaps >= {a.min_us} us: {tot / 1e3 / a.steps:.2f} ms/step")
    for k, (c, t) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{t / 1e3 / a.steps:8.3f} ms {c / a.steps:6.1f}x  {k}")


if __name__ == "__main__":
    main()
