"""Offload cost model (stage 3's analytic twin) with the reference API.

The reference's `speckit.costsim` (pkg/src/speckit/costsim.py) prices one
target pass over n tokens when the weights stream from host memory as

    forward_time(n) = fixed_overhead + max((1 - prefetch) * target_bytes / bandwidth,
                                           n / compute_rate)               (:59-65)

and combines it with a measured acceptance curve into tokens/s per budget.
This module keeps those names and semantics (`CostModel` :25-56,
`forward_time`, `crossover_tokens` :68-70, `AcceptanceCurve` :73-101,
`draft_time` :104-111, `estimate_throughput` :114-118,
`sequential_throughput` :121-123, `BudgetChoice` / `optimize_budget`
:126-149, `load_preset` :156-166) and adds what the B200 path measures
directly: `CostModel.from_b200_measurements` fits a preset from this box's
pinned H2D rate and resident tree-pass rate, and `LayerStreamer` (llama.py)
is the real per-layer streaming the model stands for. Host-side arithmetic
only -- nothing here is on the GPU hot path.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field
from pathlib import Path

__all__ = [
    "AcceptanceCurve",
    "BudgetChoice",
    "CostModel",
    "crossover_tokens",
    "draft_time",
    "estimate_throughput",
    "forward_time",
    "load_preset",
    "optimize_budget",
    "preset_names",
    "sequential_throughput",
]

PRESET_DIR = Path(__file__).resolve().parent / "presets"


@dataclass(frozen=True)
class CostModel:
    """Bytes of the two models, host-link bytes/s, saturated device tokens/s,
    per-call overhead (s), the share of target bytes already resident when a
    pass starts (prefetch during drafting), seconds per draft batch call."""

    target_bytes: float
    bandwidth: float
    compute_rate: float
    draft_bytes: float = 0.0
    fixed_overhead: float = 0.0
    prefetch_fraction: float = 0.0
    draft_step_time: float = 0.0

    def __post_init__(self) -> None:
        positive = ("target_bytes", "bandwidth", "compute_rate")
        non_negative = ("draft_bytes", "fixed_overhead", "draft_step_time")
        bad = [n for n in positive if not getattr(self, n) > 0]
        if bad:
            raise ValueError(f"{bad[0]} must be > 0")
        bad = [n for n in non_negative if getattr(self, n) < 0]
        if bad:
            raise ValueError(f"{bad[0]} must be >= 0")
        if not (0.0 <= self.prefetch_fraction <= 1.0):
            raise ValueError("prefetch_fraction must be in [0, 1]")

    @property
    def load_seconds(self) -> float:
        """Host-link time of the non-prefetched part of one target pass."""
        return (1.0 - self.prefetch_fraction) * self.target_bytes / self.bandwidth

    def to_json(self) -> str:
        return json.dumps(asdict(self))

    @classmethod
    def from_json(cls, document: str) -> "CostModel":
        return cls(**json.loads(document))

    @classmethod
    def from_b200_measurements(cls, *, target_bytes: float, h2d_bytes_per_s: float, resident_pass_s: float,
                               pass_tokens: int, draft_bytes: float = 0.0, draft_step_s: float = 0.0,
                               ring_layers: int = 0, layers: int = 1, draft_phase_s: float = 0.0) -> "CostModel":
        """A preset from numbers measured on this B200: the pinned H2D rate
        (bench.py measure_h2d), the resident target pass over `pass_tokens`
        tree tokens (compute_rate = tokens / seconds) and the LayerStreamer ring:
        while the draft runs, the ring refills with the next pass's first layers,
        up to `ring_layers` of `layers` or what the draft phase leaves time for."""
        prefetch = 0.0
        if ring_layers > 0 and layers > 0:
            prefetch = min(ring_layers / layers, draft_phase_s * h2d_bytes_per_s / target_bytes)
        return cls(target_bytes=float(target_bytes), bandwidth=float(h2d_bytes_per_s),
                   compute_rate=pass_tokens / resident_pass_s, draft_bytes=float(draft_bytes),
                   fixed_overhead=0.0, prefetch_fraction=max(0.0, min(1.0, prefetch)),
                   draft_step_time=float(draft_step_s))


def forward_time(cm: CostModel, n_tokens: float) -> float:
    """Seconds for one target pass over n_tokens (costsim.py:59-65)."""
    if n_tokens < 1:
        raise ValueError(f"n_tokens must be >= 1, got {n_tokens}")
    return cm.fixed_overhead + max(cm.load_seconds, n_tokens / cm.compute_rate)


def crossover_tokens(cm: CostModel) -> float:
    """Tokens per pass at which compute time reaches the load time (costsim.py:68-70)."""
    return cm.compute_rate * cm.load_seconds


@dataclass
class AcceptanceCurve:
    """Generation rate and draft calls per target call, measured per budget
    (strictly increasing budgets; linear interpolation, no extrapolation)."""

    budgets: list[int]
    gen_rates: list[float]
    rounds: list[float] = field(default_factory=list)

    def __post_init__(self) -> None:
        n = len(self.budgets)
        if len(self.gen_rates) != n or len(self.rounds) != n:
            raise ValueError("budgets, gen_rates and rounds must have equal length")
        if n == 0:
            raise ValueError("curve must have at least one point")
        for lo, hi in zip(self.budgets, self.budgets[1:]):
            if hi <= lo:
                raise ValueError(f"budgets must be strictly increasing, got {self.budgets}")

    def _at(self, ys: list[float], budget: float) -> float:
        xs = self.budgets
        if budget < xs[0] or budget > xs[-1]:
            raise ValueError(f"budget {budget} outside measured range [{xs[0]}, {xs[-1]}]; no extrapolation")
        for i in range(len(xs) - 1):
            if budget <= xs[i + 1]:
                w = (budget - xs[i]) / (xs[i + 1] - xs[i])
                return float(ys[i] + w * (ys[i + 1] - ys[i]))
        return float(ys[-1])

    def gen_rate_at(self, budget: float) -> float:
        return self._at(self.gen_rates, budget)

    def rounds_at(self, budget: float) -> float:
        return self._at(self.rounds, budget)


def draft_time(cm: CostModel, curve: AcceptanceCurve, budget: float) -> float:
    """Drafting seconds per target call (prefetch is credited in forward_time only)."""
    return curve.rounds_at(budget) * cm.draft_step_time


def estimate_throughput(cm: CostModel, curve: AcceptanceCurve, budget: float) -> float:
    """Predicted tokens/s at one budget: gen_rate / (draft + one target pass)."""
    return curve.gen_rate_at(budget) / (draft_time(cm, curve, budget) + forward_time(cm, budget))


def sequential_throughput(cm: CostModel) -> float:
    """Tokens/s of plain decoding: one offloaded pass per token."""
    return 1.0 / forward_time(cm, 1)


@dataclass(frozen=True)
class BudgetChoice:
    budget: int
    tokens_per_second: float
    speedup: float


def optimize_budget(cm: CostModel, curve: AcceptanceCurve) -> BudgetChoice:
    """The measured budget with the best predicted tokens/s (first on ties), and
    its speed-up over sequential decoding on the same hardware."""
    if len(curve.budgets) < 2:
        raise ValueError("curve must have at least 2 points to optimize over")
    best_b, best_t = None, -math.inf
    for b in curve.budgets:
        t = estimate_throughput(cm, curve, b)
        if t > best_t:
            best_b, best_t = b, t
    return BudgetChoice(budget=best_b, tokens_per_second=best_t, speedup=best_t / sequential_throughput(cm))


def preset_names() -> list[str]:
    return sorted(p.stem for p in PRESET_DIR.glob("*.json"))


def load_preset(name_or_path: str) -> CostModel:
    """A bundled preset by name (presets/*.json), or any cost-model JSON by path."""
    p = Path(name_or_path)
    if p.suffix == ".json" and p.exists():
        return CostModel.from_json(p.read_text())
    q = PRESET_DIR / f"{name_or_path}.json"
    if not q.exists():
        raise ValueError(f"unknown cost-model preset {name_or_path!r}")
    return CostModel.from_json(q.read_text())
