"""Generate the golden vectors in tests/golden/ by running THE REFERENCE itself.

TEST INFRASTRUCTURE. Run here (where /root/reference exists):
    python oracle/gen_fixtures.py
The outputs are committed; nothing on the GPU box reads /root/reference.

Every fixture records the inputs (seeds, shapes, params) and the reference's
outputs (tree topology + edge log-probs + rounds, generated tokens + stats).
Logits-based instances feed the reference a replay model whose rows are the
canonical float64 softmax of deterministic fp32 logits (oracle.softmax_row), so
the reference sees exactly the probability rows the B200 kernels compute.
"""

from __future__ import annotations

import json
import pathlib
import sys
import time

import numpy as np

REPO = pathlib.Path(__file__).resolve().parents[1]
REF_SRC = pathlib.Path("/root/reference/pkg/src")
OUT = REPO / "tests" / "golden"

sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))

import speckit  # noqa: E402  (the reference, imported read-only)
from speckit import engine as ref_engine  # noqa: E402
from speckit import tree as ref_tree  # noqa: E402

from oracle import speckit_oracle as ox  # noqa: E402


def tree_record(tree) -> dict:
    return {
        "rounds": tree.rounds,
        "parent": [n.parent for n in tree.nodes],
        "token": [n.token for n in tree.nodes],
        "edge": [n.edge_logprob for n in tree.nodes],
        "cum": [n.cum_logprob for n in tree.nodes],
    }


def random_instance(i: int):
    """pkg/tests/test_tree.py:44-55 (same generator, same draws)."""
    gen = np.random.default_rng(i)
    vocab = int(gen.integers(2, 9))
    budget = int(gen.integers(1, 26))
    depth = int(gen.integers(1, 5))
    sharpness = float(gen.uniform(0.05, 3.0))
    warp = None
    if i % 2:
        warp = (0.6, 0.9)
    prompt = [int(t) for t in gen.integers(0, vocab, size=2)]
    return dict(model_seed=10_000 + i, vocab=vocab, sharpness=sharpness, budget=budget, depth=depth, warp=warp, prompt=prompt)


class ReplayLM:
    """Duck-typed reference LanguageModel serving canonical rows of fp32 logits."""

    backend = "replay"

    def __init__(self, vocab: int, fn):
        self.vocab_size = vocab
        self.fn = fn

    def next_distribution(self, prefix):
        return self.next_distributions([prefix])[0]

    def next_distributions(self, prefixes):
        prefixes = [tuple(int(t) for t in p) for p in prefixes]
        if not prefixes:
            return np.empty((0, self.vocab_size))
        z = self.fn(prefixes)
        return np.stack([np.asarray(ox.softmax_row(z[i])) for i in range(len(prefixes))])


def logits_model(spec: dict):
    bias = None
    if spec.get("bias_seed") is not None:
        g = np.random.default_rng(spec["bias_seed"])
        bias = (g.standard_normal((spec["bias_rows"], spec["vocab"])) * spec["bias_scale"]).astype(np.float32)
    return ox.hashed_logits_fn(spec["vocab"], spec["seed"], spec["scale"], bias)


def gen_golden_tree():
    model = speckit.make_synthetic(17, 6, 0.3)
    tree = ref_tree.build_sssp((2, 4), model, ref_tree.BuilderParams(10, 3, 4), speckit.SamplingConfig(0.6, 0.9))
    dump = tree.to_json()
    ref_file = pathlib.Path("/root/reference/pkg/tests/data/golden_tree.json").read_text().strip()
    assert dump == ref_file, "reference no longer reproduces its own golden file"
    return {"source": "pkg/tests/data/golden_tree.json (regenerated)", "model": [17, 6, 0.3], "prefix": [2, 4],
            "params": [10, 3, 4], "warp": [0.6, 0.9], "dump": json.loads(dump)}


def gen_sssp_instances(n=200):
    out = []
    for i in range(n):
        inst = random_instance(i)
        batch = int(np.random.default_rng(i).integers(1, 17))
        model = speckit.make_synthetic(inst["model_seed"], inst["vocab"], inst["sharpness"])
        warp = speckit.SamplingConfig(*inst["warp"], seed=0) if inst["warp"] else None
        tree = ref_tree.build_sssp(tuple(inst["prompt"]), model, ref_tree.BuilderParams(inst["budget"], inst["depth"], batch), warp)
        inst["batch"] = batch
        inst["tree"] = tree_record(tree)
        out.append(inst)
    # worked examples (pkg/tests/test_tree.py:60-87)
    extra = []
    t = ref_tree.build_sssp((), speckit.TabularModel([0.6, 0.3, 0.1]), ref_tree.BuilderParams(5, 2, 4))
    extra.append({"kind": "tabular", "row": [0.6, 0.3, 0.1], "prompt": [], "budget": 5, "depth": 2, "batch": 4, "warp": None, "tree": tree_record(t)})
    chain = speckit.MarkovModel(np.roll(np.eye(3), 1, axis=1), order=1)
    t = ref_tree.build_sssp((0,), chain, ref_tree.BuilderParams(8, 4, 4))
    extra.append({"kind": "chain3", "prompt": [0], "budget": 8, "depth": 4, "batch": 4, "warp": None, "tree": tree_record(t)})
    uni = speckit.TabularModel([0.25, 0.25, 0.25, 0.25])
    for K, D, B in [(25, 4, 4), (7, 3, 2), (40, 5, 16)]:
        t = ref_tree.build_sssp((1,), uni, ref_tree.BuilderParams(K, D, B))
        extra.append({"kind": "tabular", "row": [0.25] * 4, "prompt": [1], "budget": K, "depth": D, "batch": B, "warp": None, "tree": tree_record(t)})
    return {"random": out, "extra": extra}


SEED_GRID_WARPS = [(0.0, 1.0), (0.6, 0.9), (1.0, 0.9), (1.0, 1.0)]


def gen_engine_grid(n=40):
    """pkg/tests/test_engine.py:87-98 grid, plus reference stats."""
    out = []
    for i in range(n):
        draft = speckit.make_synthetic(2 * i, 10, 0.3)
        target = speckit.make_synthetic(2 * i + 1, 10, 0.3)
        gen = np.random.default_rng(i)
        prompt = tuple(int(t) for t in gen.integers(0, 10, size=3))
        for temperature, top_p in SEED_GRID_WARPS:
            cfg = speckit.SamplingConfig(temperature, top_p, seed=i, max_new_tokens=16)
            params = ref_tree.BuilderParams(12, 5, 4)
            seq, _ = ref_engine.generate_sequential(prompt, target, cfg)
            got, stats = ref_engine.generate_specexec(prompt, draft, target, params, cfg)
            out.append({"i": i, "prompt": list(prompt), "t": temperature, "top_p": top_p, "sequential": seq, "specexec": got,
                        "target_calls": stats.target_calls, "draft_calls": stats.draft_calls,
                        "accepted": stats.accepted_per_iteration})
    # demo-03 pair (pkg/demos/03_cached_generation.py:19-20) at C1 shape: K=128, D=16, B=8, 128-token prompt, t=0
    target = speckit.make_synthetic(3, 16, 0.05)
    draft = target.power_smoothed(0.7)
    prompt = tuple(int(t) for t in np.random.default_rng(128).integers(0, 16, size=128))
    demo = []
    for temperature, top_p in [(0.0, 1.0), (0.6, 0.9)]:
        cfg = speckit.SamplingConfig(temperature, top_p, seed=0, max_new_tokens=64)
        got, stats = ref_engine.generate_specexec(prompt, draft, target, ref_tree.BuilderParams(128, 16, 8), cfg)
        demo.append({"t": temperature, "top_p": top_p, "tokens": got, "target_calls": stats.target_calls,
                     "draft_calls": stats.draft_calls, "accepted": stats.accepted_per_iteration})
    return {"grid": out, "demo03": {"model": [3, 16, 0.05], "draft_power": 0.7, "prompt": list(prompt), "K": 128, "D": 16, "B": 8, "runs": demo}}


LOGIT_TREE_CASES = [
    # vocab, K, D, B, warp, logits scale
    dict(vocab=64, K=16, D=4, B=4, warp=None, scale=1.3),
    dict(vocab=64, K=64, D=6, B=8, warp=[0.6, 0.9], scale=2.0),
    dict(vocab=64, K=32, D=8, B=8, warp=[0.0, 1.0], scale=2.0),
    dict(vocab=2048, K=128, D=8, B=16, warp=None, scale=1.3),
    dict(vocab=2048, K=256, D=16, B=32, warp=None, scale=4.0),
    dict(vocab=2048, K=128, D=8, B=16, warp=[0.6, 0.9], scale=3.0),
    dict(vocab=2048, K=96, D=8, B=64, warp=[1.0, 0.8], scale=3.0),
    dict(vocab=32000, K=64, D=16, B=32, warp=None, scale=4.0),
]


def gen_logit_trees():
    out = []
    for ci, case in enumerate(LOGIT_TREE_CASES):
        spec = dict(vocab=case["vocab"], seed=1000 + ci, scale=case["scale"], bias_seed=None)
        prefix = tuple(int(t) for t in np.random.default_rng(ci).integers(0, case["vocab"], size=5))
        lm = ReplayLM(case["vocab"], logits_model(spec))
        warp = speckit.SamplingConfig(*case["warp"]) if case["warp"] else None
        t0 = time.time()
        tree = ref_tree.build_sssp(prefix, lm, ref_tree.BuilderParams(case["K"], case["D"], case["B"]), warp)
        rec = dict(case, spec=spec, prefix=list(prefix), tree=tree_record(tree), seconds=round(time.time() - t0, 2))
        print(f"  logits tree {ci}: V={case['vocab']} K={case['K']} nodes={len(tree.nodes)} rounds={tree.rounds} {rec['seconds']}s")
        out.append(rec)
    return out


def gen_logit_engine():
    """t=0 generation on correlated logits pairs, raw draft scoring."""
    out = []
    raw_build = ref_tree.build_sssp

    def build_raw(prefix, draft, params, warp=None, warp_scores=True):
        return raw_build(prefix, draft, params, warp, warp_scores=False)

    for ci, (V, K, D, B, bias_scale) in enumerate([(512, 32, 6, 8, 3.0), (2048, 64, 8, 16, 4.0)]):
        dspec = dict(vocab=V, seed=5000 + ci, scale=1.0, bias_seed=77 + ci, bias_rows=V, bias_scale=bias_scale)
        tspec = dict(vocab=V, seed=6000 + ci, scale=1.0, bias_seed=77 + ci, bias_rows=V, bias_scale=bias_scale)
        draft, target = ReplayLM(V, logits_model(dspec)), ReplayLM(V, logits_model(tspec))
        prompt = tuple(int(t) for t in np.random.default_rng(900 + ci).integers(0, V, size=8))
        runs = []
        for scoring in ("raw", "warped"):
            cfg = speckit.SamplingConfig(0.0, 1.0, seed=ci, max_new_tokens=24)
            if scoring == "raw":
                ref_engine.build_sssp = build_raw
            try:
                got, stats = ref_engine.generate_specexec(prompt, draft, target, ref_tree.BuilderParams(K, D, B), cfg)
            finally:
                ref_engine.build_sssp = raw_build
            seq, _ = ref_engine.generate_sequential(prompt, target, cfg)
            runs.append({"scoring": scoring, "tokens": got, "sequential": seq, "target_calls": stats.target_calls,
                         "draft_calls": stats.draft_calls, "accepted": stats.accepted_per_iteration})
        out.append({"draft": dspec, "target": tspec, "prompt": list(prompt), "K": K, "D": D, "B": B, "runs": runs})
    return out


def gen_specinfer_grid(n=60):
    """SpecInfer baseline (specinfer.py:53-127, tree.py:383-425): stochastic
    trees and full generate_specinfer runs on Markov pairs, plus logits-LM pairs
    at V=32000 (canonical softmax rows, like the GPU)."""
    from speckit import specinfer as ref_si

    out = []
    for i in range(n):
        gen = np.random.default_rng(5000 + i)
        V = int(gen.integers(3, 12))
        sharp = float(gen.uniform(0.05, 2.0))
        depth = int(gen.integers(1, 5))
        branching = [int(gen.integers(1, 5))] + [int(gen.integers(1, 3)) for _ in range(depth - 1)]
        t, p = [(0.6, 0.9), (1.0, 1.0), (0.0, 1.0), (1.3, 0.8)][i % 4]
        target = speckit.make_synthetic(7000 + i, V, sharp)
        draft = target.power_smoothed(0.6)
        prompt = tuple(int(x) for x in gen.integers(0, V, size=3))
        cfg = speckit.SamplingConfig(t, p, seed=i, max_new_tokens=20)
        rng = speckit.CounterRng(i, ref_si.DRAFT_STREAM)
        tree = ref_tree.build_stochastic(prompt, draft, branching, rng, cfg)
        toks, st = ref_si.generate_specinfer(prompt, draft, target, branching, cfg)
        out.append({"kind": "markov", "target_seed": 7000 + i, "V": V, "sharpness": sharp, "draft_power": 0.6,
                    "branching": branching, "t": t, "top_p": p, "seed": i, "prompt": list(prompt),
                    "tree": tree_record(tree), "mult": [nd.multiplicity for nd in tree.nodes],
                    "tokens": toks, "target_calls": st.target_calls, "draft_calls": st.draft_calls,
                    "accepted": st.accepted_per_iteration})
    for ci in range(4):
        V = 32000
        dspec = {"vocab": V, "seed": 300 + ci, "scale": 1.6}
        tspec = {"vocab": V, "seed": 300 + ci, "scale": 1.9}
        draft, target = ReplayLM(V, logits_model(dspec)), ReplayLM(V, logits_model(tspec))
        prompt = tuple(int(x) for x in np.random.default_rng(950 + ci).integers(0, V, size=6))
        branching = ref_si.branching_for_budget([12, 24, 8, 40][ci], [4, 3, 2, 5][ci])
        t, p = [(0.6, 0.9), (1.0, 1.0), (0.8, 0.95), (0.0, 1.0)][ci]
        cfg = speckit.SamplingConfig(t, p, seed=ci, max_new_tokens=16)
        toks, st = ref_si.generate_specinfer(prompt, draft, target, branching, cfg)
        out.append({"kind": "logits", "draft": dspec, "target": tspec, "branching": branching, "t": t, "top_p": p,
                    "seed": ci, "prompt": list(prompt), "tokens": toks, "target_calls": st.target_calls,
                    "draft_calls": st.draft_calls, "accepted": st.accepted_per_iteration})
    return out


def gen_beam_instances(n=80):
    """build_beam (tree.py:330-380) on Markov models, raw and warped scoring, plus
    logits-LM draft at V=32000."""
    out = []
    for i in range(n):
        gen = np.random.default_rng(6000 + i)
        V = int(gen.integers(2, 12))
        sharp = float(gen.uniform(0.05, 2.5))
        beam, max_len = int(gen.integers(1, 9)), int(gen.integers(1, 6))
        warp = [None, (0.6, 0.9), (0.0, 1.0), (1.0, 0.8)][i % 4]
        model = speckit.make_synthetic(8000 + i, V, sharp)
        prompt = tuple(int(x) for x in gen.integers(0, V, size=2))
        cfg = speckit.SamplingConfig(*warp) if warp else None
        tree = ref_tree.build_beam(prompt, model, beam, max_len, cfg)
        out.append({"kind": "markov", "seed": 8000 + i, "V": V, "sharpness": sharp, "beam": beam, "max_len": max_len,
                    "warp": warp, "prompt": list(prompt), "tree": tree_record(tree)})
    for ci in range(3):
        V = 32000
        spec = {"vocab": V, "seed": 400 + ci, "scale": 2.2}
        lm = ReplayLM(V, logits_model(spec))
        prompt = tuple(int(x) for x in np.random.default_rng(970 + ci).integers(0, V, size=5))
        beam, max_len = [8, 16, 4][ci], [4, 3, 6][ci]
        warp = [None, (0.6, 0.9), (1.0, 1.0)][ci]
        tree = ref_tree.build_beam(prompt, lm, beam, max_len, speckit.SamplingConfig(*warp) if warp else None)
        out.append({"kind": "logits", "spec": spec, "beam": beam, "max_len": max_len, "warp": warp,
                    "prompt": list(prompt), "tree": tree_record(tree)})
    return out


def gen_harness():
    """The reference harness (pkg/src/speckit/harness/experiments.py) on a small
    grid: run_acceptance (rows with bootstrap CIs and mean_rounds, curves,
    run records, the versioned CSV / JSONL text), run_throughput over a bundled
    preset (rows + CSV) and run_equivalence (cells + JSONL)."""
    import tempfile

    from speckit import load_preset
    from speckit.harness.config import ExperimentConfig
    from speckit.harness.experiments import run_acceptance, run_equivalence, run_throughput

    out = {}
    with tempfile.TemporaryDirectory() as td:
        spec = dict(kind="acceptance", target={"kind": "synthetic", "seed": 11, "vocab_size": 16, "sharpness": 0.3},
                    draft={"kind": "power", "base": {"kind": "synthetic", "seed": 11, "vocab_size": 16,
                                                     "sharpness": 0.3}, "power": 0.6},
                    prompt_source={"kind": "inline", "token_lists": [[1, 2, 3], [4, 5]]}, budgets=[4, 16, 32],
                    seeds=[0, 1, 2], sampling=[{"temperature": 0.6, "top_p": 0.9}, {"temperature": 0.0}],
                    max_new_tokens=16, max_depth=5, batch_size=4, si_depth=4, output_path=f"{td}/acc.csv")
        cfg = ExperimentConfig(**spec)
        res = run_acceptance(cfg)
        out["acceptance"] = {"config": {k: v for k, v in spec.items() if k != "output_path"},
                             "rows": [r.__dict__ for r in res.rows],
                             "curves": {m: {"budgets": c.budgets, "gen_rates": c.gen_rates, "rounds": c.rounds}
                                        for m, c in res.curves.items()},
                             "run_records": res.run_records,
                             "csv": (pathlib.Path(td) / "acc.csv").read_text(),
                             "jsonl": (pathlib.Path(td) / "acc.runs.jsonl").read_text()}
        cfg_t = ExperimentConfig(**{**spec, "kind": "throughput", "output_path": f"{td}/thr.csv"})
        thr = run_throughput(cfg_t, load_preset("pcie4-16bit-70b"), res.curves)
        out["throughput"] = {"preset": "pcie4-16bit-70b", "rows": [r.__dict__ for r in thr.rows],
                             "choices": {m: c.__dict__ for m, c in thr.choices.items()},
                             "csv": (pathlib.Path(td) / "thr.csv").read_text()}
        spec_e = dict(kind="equivalence", target={"kind": "synthetic", "seed": 1, "vocab_size": 10, "sharpness": 0.3},
                      budgets=[8], seeds=[0, 1, 2], sampling=[{"temperature": 0.6, "top_p": 0.9}, {"temperature": 0.0},
                                                              {"temperature": 1.0}],
                      max_new_tokens=12, max_depth=4, batch_size=4, equivalence_cells=12, vocab_size=10,
                      sharpness=0.3, output_path=f"{td}/eq.jsonl")
        rep = run_equivalence(ExperimentConfig(**spec_e))
        out["equivalence"] = {"config": {k: v for k, v in spec_e.items() if k != "output_path"},
                              "passed": rep.passed, "jsonl": (pathlib.Path(td) / "eq.jsonl").read_text()}
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    jobs = {
        "golden_tree.json": gen_golden_tree,
        "sssp_instances.json": gen_sssp_instances,
        "engine_grid.json": gen_engine_grid,
        "logit_trees.json": gen_logit_trees,
        "logit_engine.json": gen_logit_engine,
        "specinfer_grid.json": gen_specinfer_grid,
        "beam_instances.json": gen_beam_instances,
        "harness_grid.json": gen_harness,
    }
    only = set(sys.argv[1:])
    for name, fn in jobs.items():
        if only and name not in only:
            continue
        t0 = time.time()
        data = fn()
        (OUT / name).write_text(json.dumps({"generator": "oracle/gen_fixtures.py", "reference": "speckit 0.1.0 @ /root/reference",
                                            "numpy": np.__version__, "data": data}, separators=(",", ":")) + "\n")
        print(f"{name}: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
