"""Experiment runners over the GPU engine, with the reference harness's
semantics and report schema (pkg/src/speckit/harness/experiments.py,
harness/io.py): the acceptance-vs-budget grid that produces the metric's
second half (accepted tokens per target iteration vs draft budget), the
throughput join with a cost model, and the seed-equivalence gate.

* `run_acceptance` (experiments.py:199-279): cells in the reference order
  method x budget x seed x warp x prompt, one `generate_specexec` /
  `generate_specinfer` per cell on this package's engine, rows aggregated per
  (method, budget) with the percentile bootstrap CI of the mean generation rate
  (seeded by crc32("method:budget"), experiments.py:40-48) and `mean_rounds` =
  mean draft calls per target call; curves feed `costsim.AcceptanceCurve`.
* `run_throughput` (experiments.py:305-355): estimated tokens/s, draft and
  forward time per budget, speed-up over sequential decoding, the optimal budget.
* `run_equivalence` (experiments.py:399-461): speculative == sequential for
  freshly drawn synthetic pairs, with the first divergence position.
* `write_csv` / `write_jsonl` (io.py:10-29): CSV with a leading
  `schema_version` column on every row, JSON lines with sorted keys.

`cfg` is duck-typed: the reference's own `ExperimentConfig` works (its
`target_model()` / `draft_model()` build reference plugins, which the engine
adapts through `HostRowsModel`), as does `HarnessConfig` below; explicit
`draft` / `target` / `prompts` override the config (e.g. Llama device models).
Host-side orchestration only: every cell runs the sm_100a kernels.
"""

from __future__ import annotations

import csv
import json
import zlib
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Iterable, Sequence

import numpy as np

from .costsim import AcceptanceCurve, BudgetChoice, CostModel, draft_time, estimate_throughput, forward_time, \
    optimize_budget
from .engine import GENERATION_STREAM, GenStats, generate_sequential, generate_specexec, stats_record
from .models import make_synthetic
from .sampling import SamplingConfig
from .specinfer import branching_for_budget, generate_specinfer, schedule_size
from .tree import BuilderParams

SCHEMA_VERSION = 1


# --------------------------------------------------------------------------- io
def write_csv(path: str | Path, header: list[str], rows: Iterable[Iterable[Any]]) -> None:
    """CSV whose every row starts with schema_version (harness/io.py:13-22)."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with path.open("w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["schema_version", *header])
        for row in rows:
            w.writerow([SCHEMA_VERSION, *row])


def write_jsonl(path: str | Path, records: Iterable[dict[str, Any]]) -> None:
    """One JSON object per line, keys sorted (harness/io.py:25-29)."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with path.open("w") as fh:
        for rec in records:
            fh.write(json.dumps(rec, sort_keys=True) + "\n")


def bootstrap_mean_ci(values: Sequence[float], n_resamples: int = 1000, seed: int = 0,
                      alpha: float = 0.05) -> tuple[float, float]:
    """Percentile bootstrap interval of the mean: resample indices with a seeded
    PCG64 generator, take the alpha/2 and 1-alpha/2 quantiles of the resampled
    means (the reference's draws, so intervals match it exactly)."""
    arr = np.asarray(values, dtype=np.float64)
    idx = np.random.default_rng(seed).integers(0, arr.size, size=(n_resamples, arr.size))
    means = arr[idx].mean(axis=1)
    return float(np.quantile(means, alpha / 2)), float(np.quantile(means, 1 - alpha / 2))


# --------------------------------------------------------------------------- config
@dataclass
class HarnessConfig:
    """The fields of the reference's ExperimentConfig (harness/config.py:75-120)
    that the runners read; models and prompts are passed explicitly."""

    budgets: list[int] = field(default_factory=lambda: [16, 64, 256])
    seeds: list[int] = field(default_factory=lambda: [0, 1, 2, 3, 4, 5, 6, 7])
    sampling: list[dict[str, Any]] = field(default_factory=lambda: [{"temperature": 0.6, "top_p": 0.9}])
    max_new_tokens: int = 32
    max_depth: int = 16
    batch_size: int = 8
    si_depth: int = 8
    branching: list[int] | None = None
    equivalence_cells: int = 100
    vocab_size: int = 16
    sharpness: float = 0.3
    workers: int = 1
    output_path: str | None = None

    def __post_init__(self) -> None:
        if not self.budgets:
            raise ValueError("budgets must be non-empty")
        if not self.seeds:
            raise ValueError("seeds must be non-empty")
        if not self.sampling:
            raise ValueError("sampling grid must be non-empty")

    def sampling_configs(self, seed: int, max_new_tokens: int | None = None) -> list[SamplingConfig]:
        n = self.max_new_tokens if max_new_tokens is None else max_new_tokens
        return [SamplingConfig(s.get("temperature", 1.0), s.get("top_p", 1.0), seed=seed, max_new_tokens=n)
                for s in self.sampling]


def _models(cfg, draft, target):
    if target is None:
        target = cfg.target_model()
    if draft is None:
        draft = cfg.draft_model()
    return draft, target


def _prompts(cfg, target, prompts):
    if prompts is not None:
        return [tuple(int(t) for t in p) for p in prompts]
    src = getattr(cfg, "prompt_source", None) or {"kind": "sampled", "length": 8, "count": 2}
    kind = src.get("kind")
    if kind == "inline" and "token_lists" in src:
        return [tuple(int(t) for t in toks) for toks in src["token_lists"]]
    if kind == "sampled":  # experiments.py:72-80: sequential samples of the target itself
        out = []
        for j in range(src.get("count", 2)):
            toks, _ = generate_sequential((), target, SamplingConfig(seed=src.get("seed", 7777) + j,
                                                                     max_new_tokens=src.get("length", 8)))
            out.append(tuple(toks))
        return out
    raise ValueError(f"prompt source {src!r}: pass prompts= explicitly (text sources need the reference tokenizers)")


# --------------------------------------------------------------------------- acceptance
@dataclass
class AcceptanceRow:
    method: str
    budget: int
    n_runs: int
    mean_gen_rate: float
    ci_lo: float
    ci_hi: float
    mean_rounds: float


@dataclass
class AcceptanceResult:
    rows: list[AcceptanceRow]
    curves: dict[str, AcceptanceCurve]
    run_records: list[dict[str, Any]]

    def row(self, method: str, budget: int) -> AcceptanceRow:
        for r in self.rows:
            if r.method == method and r.budget == budget:
                return r
        raise KeyError(f"no row for method={method!r} budget={budget}")


def run_acceptance(cfg, methods: tuple[str, ...] = ("sx", "si"), draft=None, target=None, prompts=None,
                   warp_scores: bool = True) -> AcceptanceResult:
    """Generation rate over the budget grid for both engines, paired cells (the
    same prompts, seeds and warps for every method x budget)."""
    draft, target = _models(cfg, draft, target)
    plist = _prompts(cfg, target, prompts)
    cells = [(m, b, w, p) for m in methods for b in cfg.budgets for s in cfg.seeds for w in cfg.sampling_configs(s)
             for p in plist]
    results: list[tuple[GenStats, dict]] = []
    for method, budget, warp, prompt in cells:
        if method == "sx":
            _, st = generate_specexec(prompt, draft, target, BuilderParams(budget, cfg.max_depth, cfg.batch_size), warp,
                                      warp_scores=warp_scores)
            rec = stats_record("sx", warp, st, budget, cfg.max_depth, cfg.batch_size)
        elif method == "si":
            br = cfg.branching or branching_for_budget(budget, cfg.si_depth)
            _, st = generate_specinfer(prompt, draft, target, br, warp)
            rec = stats_record("si", warp, st, schedule_size(br), len(br), br[0])
        else:
            raise ValueError(f"unknown method {method!r}")
        results.append((st, rec))
    by_cell: dict[tuple[str, int], list[GenStats]] = {}
    for (method, budget, _, _), (st, _) in zip(cells, results):
        by_cell.setdefault((method, budget), []).append(st)
    rows, curves = [], {}
    for method in methods:
        rates, rounds = [], []
        for budget in cfg.budgets:
            sts = by_cell[(method, budget)]
            gr = [s.generation_rate for s in sts]
            mr = float(np.mean([s.draft_calls / max(1, s.target_calls) for s in sts]))
            lo, hi = bootstrap_mean_ci(gr, seed=zlib.crc32(f"{method}:{budget}".encode()))
            rows.append(AcceptanceRow(method, budget, len(gr), float(np.mean(gr)), lo, hi, mr))
            rates.append(float(np.mean(gr)))
            rounds.append(mr)
        curves[method] = AcceptanceCurve(list(cfg.budgets), rates, rounds)
    records = [rec for _, rec in results]
    if cfg.output_path:
        write_csv(cfg.output_path, ["method", "budget", "n_runs", "mean_gen_rate", "ci_lo", "ci_hi", "mean_rounds"],
                  [[r.method, r.budget, r.n_runs, r.mean_gen_rate, r.ci_lo, r.ci_hi, r.mean_rounds] for r in rows])
        write_jsonl(Path(cfg.output_path).with_suffix(".runs.jsonl"), records)
    return AcceptanceResult(rows, curves, records)


# --------------------------------------------------------------------------- throughput
@dataclass
class ThroughputRow:
    method: str
    budget: int
    gen_rate: float
    t_draft: float
    t_forward: float
    tok_per_s: float
    speedup: float
    optimal: bool


@dataclass
class ThroughputResult:
    rows: list[ThroughputRow]
    choices: dict[str, BudgetChoice]


def run_throughput(cfg, cost_model: CostModel, curves: dict[str, AcceptanceCurve] | None) -> ThroughputResult:
    """Join measured acceptance curves with a cost model (e.g. the fitted
    `b200-pcie5-bf16-70b` preset); no curves is an error, not a re-measure."""
    if not curves:
        raise ValueError("run_throughput requires acceptance curves; run run_acceptance first")
    seq = 1.0 / forward_time(cost_model, 1)
    rows, choices = [], {}
    for method, curve in sorted(curves.items()):
        choice = optimize_budget(cost_model, curve)
        choices[method] = choice
        for b in curve.budgets:
            tps = estimate_throughput(cost_model, curve, b)
            rows.append(ThroughputRow(method, b, curve.gen_rate_at(b), draft_time(cost_model, curve, b),
                                      forward_time(cost_model, b), tps, tps / seq, b == choice.budget))
    if getattr(cfg, "output_path", None):
        write_csv(cfg.output_path, ["method", "K", "gen_rate", "t_draft", "t_forward", "tok_per_s", "speedup", "optimal"],
                  [[r.method, r.budget, r.gen_rate, r.t_draft, r.t_forward, r.tok_per_s, r.speedup, int(r.optimal)]
                   for r in rows])
    return ThroughputResult(rows, choices)


# --------------------------------------------------------------------------- equivalence
@dataclass
class EquivalenceCell:
    index: int
    draft_seed: int
    target_seed: int
    prompt: tuple[int, ...]
    seed: int
    temperature: float
    top_p: float
    ok: bool = True
    divergence_position: int | None = None
    expected: list[int] = field(default_factory=list)
    got: list[int] = field(default_factory=list)

    def provenance(self) -> dict[str, Any]:
        return {"index": self.index, "draft_seed": self.draft_seed, "target_seed": self.target_seed,
                "prompt": list(self.prompt), "seed": self.seed, "temperature": self.temperature, "top_p": self.top_p,
                "rng_stream": GENERATION_STREAM}


@dataclass
class EquivalenceReport:
    cells: list[EquivalenceCell]

    @property
    def passed(self) -> bool:
        return all(c.ok for c in self.cells)

    @property
    def failures(self) -> list[EquivalenceCell]:
        return [c for c in self.cells if not c.ok]


def run_equivalence(cfg) -> EquivalenceReport:
    """Cell i: synthetic pair (seeds 101 + 2i, 102 + 2i), a 4-token prompt sampled
    from the target, warp i mod |sampling|, seed i mod |seeds|; the GPU
    speculative tokens must equal the GPU sequential tokens."""
    budget = cfg.budgets[0]
    cells = []
    for i in range(cfg.equivalence_cells):
        ds, ts = 101 + 2 * i, 102 + 2 * i
        draft = make_synthetic(ds, cfg.vocab_size, cfg.sharpness)
        target = make_synthetic(ts, cfg.vocab_size, cfg.sharpness)
        prompt, _ = generate_sequential((), target, SamplingConfig(seed=5000 + i, max_new_tokens=4))
        prompt = tuple(prompt)
        w = cfg.sampling[i % len(cfg.sampling)]
        run = SamplingConfig(w.get("temperature", 1.0), w.get("top_p", 1.0), seed=cfg.seeds[i % len(cfg.seeds)],
                             max_new_tokens=cfg.max_new_tokens)
        expected, _ = generate_sequential(prompt, target, run)
        got, _ = generate_specexec(prompt, draft, target, BuilderParams(budget, cfg.max_depth, cfg.batch_size), run)
        cell = EquivalenceCell(i, ds, ts, prompt, run.seed, run.temperature, run.top_p)
        if got != expected:
            cell.ok, cell.expected, cell.got = False, expected, got
            cell.divergence_position = next((j for j, (a, b) in enumerate(zip(expected, got)) if a != b),
                                            min(len(expected), len(got)))
        cells.append(cell)
    if getattr(cfg, "output_path", None):
        write_jsonl(cfg.output_path, [{**c.provenance(), "ok": c.ok, "divergence_position": c.divergence_position}
                                      for c in cells])
    return EquivalenceReport(cells)
