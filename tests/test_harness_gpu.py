"""The acceptance-vs-budget grid and the equivalence gate on the GPU engine
reproduce the reference harness's own reports (tests/golden/harness_grid.json:
rows with bootstrap CIs and mean_rounds, per-run records, CSV / JSON-lines text
with schema_version; pkg/src/speckit/harness/experiments.py:199-279, 399-461),
with device table models and with host plugin models (HostRowsModel)."""

import json
import pathlib

import pytest

import paper_2406_02532_b200 as sx
from oracle import speckit_oracle as ox
from paper_2406_02532_b200.harness import HarnessConfig, run_acceptance, run_equivalence

pytestmark = pytest.mark.gpu
GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "harness_grid.json").read_text())["data"]


def _cfg(spec, out):
    keys = ("budgets", "seeds", "sampling", "max_new_tokens", "max_depth", "batch_size", "si_depth")
    return HarnessConfig(**{k: spec[k] for k in keys}, output_path=str(out))


@pytest.mark.parametrize("backend", ["device", "host-plugin"])
def test_acceptance_grid_matches_reference(cuda, tmp_path, backend):
    acc = GOLD["acceptance"]
    spec = acc["config"]
    t = spec["target"]
    mk = sx.make_synthetic if backend == "device" else ox.make_synthetic
    target = mk(t["seed"], t["vocab_size"], t["sharpness"])
    draft = target.power_smoothed(spec["draft"]["power"])
    res = run_acceptance(_cfg(spec, tmp_path / "acc.csv"), draft=draft, target=target,
                         prompts=spec["prompt_source"]["token_lists"])
    assert res.run_records == acc["run_records"]
    assert [r.__dict__ for r in res.rows] == acc["rows"]
    assert (tmp_path / "acc.csv").read_text() == acc["csv"]
    assert (tmp_path / "acc.runs.jsonl").read_text() == acc["jsonl"]
    assert {m: c.gen_rates for m, c in res.curves.items()} == {m: c["gen_rates"] for m, c in acc["curves"].items()}


def test_equivalence_gate_matches_reference(cuda, tmp_path):
    eq = GOLD["equivalence"]
    spec = eq["config"]
    cfg = HarnessConfig(budgets=spec["budgets"], seeds=spec["seeds"], sampling=spec["sampling"],
                        max_new_tokens=spec["max_new_tokens"], max_depth=spec["max_depth"],
                        batch_size=spec["batch_size"], equivalence_cells=spec["equivalence_cells"],
                        vocab_size=spec["vocab_size"], sharpness=spec["sharpness"], output_path=str(tmp_path / "eq.jsonl"))
    rep = run_equivalence(cfg)
    assert rep.passed and eq["passed"]
    assert (tmp_path / "eq.jsonl").read_text() == eq["jsonl"]
