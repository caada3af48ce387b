"""B200-native SpecExec (arXiv 2406.02532).

Drop-in for the hot path of the reference `speckit` package: the same
generator / engine API (`BuilderParams`, `SamplingConfig`, `CounterRng`,
`DraftTree`, `flatten`, `build_sssp`, `precompute`, `generate_specexec`,
`generate_sequential`, `GenStats`, `ProbCache`, `LanguageModel`, ...) over
hand-written sm_100a CUDA kernels behind the C ABI in include/specexec_b200.h.
There is no CPU fallback: without the built library or a CUDA device every
device call raises.
"""

from .costsim import (AcceptanceCurve, BudgetChoice, CostModel, crossover_tokens, estimate_throughput, forward_time,
                      load_preset, optimize_budget)
from .engine import GenStats, ProbCache, generate_sequential, generate_specexec, precompute, stats_record
from .models import HostRowsModel, LanguageModel, MarkovModel, TabularModel, make_synthetic, model_from_json
from .rng import CounterRng
from .sampling import SamplingConfig, apply_warp, sample, validate_distribution
from .tree import ROOT, BuilderParams, DraftNode, DraftTree, FlattenedTree, build_sssp, flatten
from .beam import build_beam
from .specinfer import (VerifyOutcome, branching_for_budget, build_stochastic, generate_specinfer, schedule_size,
                        verify_specinfer)

__version__ = "0.1.0"

__all__ = [
    "AcceptanceCurve",
    "BudgetChoice",
    "CostModel",
    "HostRowsModel",
    "crossover_tokens",
    "estimate_throughput",
    "forward_time",
    "load_preset",
    "optimize_budget",
    "ROOT",
    "BuilderParams",
    "CounterRng",
    "DraftNode",
    "DraftTree",
    "FlattenedTree",
    "GenStats",
    "LanguageModel",
    "MarkovModel",
    "ProbCache",
    "SamplingConfig",
    "TabularModel",
    "apply_warp",
    "build_sssp",
    "build_beam",
    "build_stochastic",
    "branching_for_budget",
    "generate_specinfer",
    "schedule_size",
    "verify_specinfer",
    "VerifyOutcome",
    "flatten",
    "generate_sequential",
    "generate_specexec",
    "make_synthetic",
    "model_from_json",
    "precompute",
    "sample",
    "stats_record",
    "validate_distribution",
]
