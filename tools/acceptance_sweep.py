"""Generation rate vs draft budget, SpecExec vs SpecInfer, on the GPU -- the
metric's second half ("accepted tokens / target iteration vs draft budget") and
the reference harness's run_acceptance sweep (pkg/src/speckit/harness/
experiments.py:199-260) driven through this package's engines.

Per (method, budget) cell: `--seeds` runs of `--tokens` generated tokens on one
random prompt; records the reference's stats_record schema plus device-timed
tokens/s. SpecInfer uses branching_for_budget(budget, --si-depth) like the
reference harness.

  python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b \
      --budgets 64,256,1024 --synthetic 4 --out profiles/r1/acceptance_c2.jsonl
"""

import argparse
import json
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2406_02532_b200 as sx  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel, SyntheticBias  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--draft", default="tiny-draft")
    ap.add_argument("--target", default="tiny")
    ap.add_argument("--budgets", default="16,64,256")
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--si-depth", type=int, default=8)
    ap.add_argument("--t", type=float, default=0.0)
    ap.add_argument("--top-p", type=float, default=1.0)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--synthetic", type=float, default=4.0)
    ap.add_argument("--methods", default="sx,si")
    ap.add_argument("--scoring", choices=["raw", "warped"], default="raw")
    ap.add_argument("--out", default=None)
    ap.add_argument("--attn", choices=["auto", "mma", "tc"], default="auto")
    a = ap.parse_args()
    from paper_2406_02532_b200 import _lib

    _lib.call("sx_attention_set_impl", {"auto": 0, "mma": 1, "tc": 2}[a.attn])
    budgets = [int(b) for b in a.budgets.split(",")]
    syn = SyntheticBias(seed=99, rank=64, scale=a.synthetic) if a.synthetic > 0 else None
    K = max(budgets)
    ctx = 128 + a.tokens + 64
    target = LlamaModel(a.target, seed=1, max_ctx=ctx + 2 * K + 2, max_tokens=max(K + 1, 256), synthetic=syn)
    draft = LlamaModel(a.draft, seed=2, max_ctx=ctx + 4 * K + 2 * a.batch * (a.depth + 1),
                       max_tokens=max(a.batch, K, 256), synthetic=syn)
    V = PRESETS[a.target].vocab
    prompt = tuple(int(t) for t in np.random.default_rng(1000).integers(0, V, size=128))
    recs = []
    out = pathlib.Path(a.out) if a.out else None
    if out:
        out.write_text("")

    def run(method, budget, cfg):
        if method == "seq":  # the speed-up denominator: one target pass per token
            toks, st = sx.generate_sequential(prompt, target, cfg)
            return toks, st, sx.stats_record("seq", cfg, st, 0, 0, 0)
        if method == "sx":
            params = sx.BuilderParams(budget, a.depth, a.batch)
            toks, st = sx.generate_specexec(prompt, draft, target, params, cfg,
                                            warp_scores=a.scoring == "warped")
            return toks, st, sx.stats_record("sx", cfg, st, budget, a.depth, a.batch)
        br = sx.branching_for_budget(budget, a.si_depth)
        toks, st = sx.generate_specinfer(prompt, draft, target, br, cfg)
        return toks, st, sx.stats_record("si", cfg, st, sx.schedule_size(br), len(br), br[0])

    for method in a.methods.split(","):
        for budget in (budgets if method != "seq" else [0]):
            try:  # untimed warm-up: CUDA-graph capture and workspace allocation for this budget
                run(method, budget, sx.SamplingConfig(a.t, a.top_p, seed=10_000, max_new_tokens=4))
            except torch.OutOfMemoryError as e:
                print(f"# {method} K={budget}: out of memory ({str(e).splitlines()[0]})", flush=True)
                break
            for seed in range(a.seeds):
                cfg = sx.SamplingConfig(a.t, a.top_p, seed=seed, max_new_tokens=a.tokens)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                toks, st, rec = run(method, budget, cfg)
                torch.cuda.synchronize()
                el = time.perf_counter() - t0
                rec.update({"budget": budget, "tokens_per_s": len(toks) / el, "seconds": el,
                            "draft_calls_per_iter": st.draft_calls / max(1, st.target_calls),
                            "draft": a.draft, "target": a.target, "synthetic": a.synthetic,
                            "scoring": a.scoring if method == "sx" else "warped"})
                recs.append(rec)
                print(json.dumps(rec), flush=True)
                if out:
                    with out.open("a") as f:
                        f.write(json.dumps(rec) + "\n")
    print("# method budget  gen_rate  tokens/s")
    for method in a.methods.split(","):
        for budget in (budgets if method != "seq" else [0]):
            rs = [r for r in recs if r["method"] == method and r["budget"] == budget]
            if not rs:
                continue
            print(f"# {method:4s} {budget:6d} {np.mean([r['generation_rate'] for r in rs]):8.3f} "
                  f"{np.mean([r['tokens_per_s'] for r in rs]):9.2f}")
    seq = [r["tokens_per_s"] for r in recs if r["method"] == "seq"]
    if seq:
        base = float(np.mean(seq))
        for method in a.methods.split(","):
            if method == "seq":
                continue
            for budget in budgets:
                rs = [r for r in recs if r["method"] == method and r["budget"] == budget]
                if rs:
                    print(f"# speedup {method:4s} {budget:6d} {np.mean([r['tokens_per_s'] for r in rs]) / base:6.2f}x "
                          f"vs sequential ({base:.2f} tokens/s)")


if __name__ == "__main__":
    main()
