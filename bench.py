#!/usr/bin/env python
"""SpecExec target-iteration benchmark on B200 (BASELINE.json metric:
generated tokens/s, with accepted tokens per target iteration beside it).

A *step* is one SpecExec target iteration: GPU draft-tree build (stage 1), one
target pass over the anchor + every tree node (stage 2), the acceptance walk
and KV compaction (stage 4). Default workload = BASELINE configs[1] (C2):
Llama-2-7B-shaped draft + Llama-2-70B-shaped target, random-init bf16, target
resident in HBM on one B200, budget K=1024, t=0, one random 128-token prompt.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N>1 (torchrun): the 70B target is tensor-parallel over the N GPUs (NCCL
all-reduce over NVLink after the o / down projections, all-gathered
vocab-parallel logits; tp.py), the draft / tree build / walk are replicas on
every rank -- one generation stream, strong scaling. `--parallel replicas`
runs N independent streams instead (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (draft preset, target preset, K, D, B, temperature, top_p)
    # B=1024: the tree is identical for every B; a wide batch makes the
    # draft rounds M=1024 tensor-core GEMMs (2 draft calls / iteration instead of 5)
    "c2": ("llama2-7b", "llama2-70b", 1024, 16, 1024, 0.0, 1.0),
    "c5-l3": ("llama3-8b", "llama3-70b", 1024, 16, 1024, 0.0, 1.0),
    # C4: 70B target tensor-parallel over the N GPUs (--gpus N), K=4096
    "c4": ("llama2-7b", "llama2-70b", 4096, 16, 1024, 0.0, 1.0),
    "tiny": ("tiny-draft", "tiny", 128, 16, 8, 0.0, 1.0),
    # C3: 70B target offloaded to pinned host RAM, streamed per layer; 7B draft resident
    "c3": ("llama2-7b", "llama2-70b", 2048, 16, 1024, 0.6, 0.9),
    "tiny-offload": ("tiny-draft", "tiny", 128, 16, 8, 0.6, 0.9),
}
OFFLOAD = {"c3", "tiny-offload"}
METRIC = "generated tokens/sec (accepted tokens per target iteration reported beside)"


def workload_desc(name: str, K: int, B: int) -> str:
    d, t, _, D, _, temp, _ = WORKLOADS[name]
    return (f"{name}: {d} draft + {t} target, K={K}, D={D}, B={B}, t={temp}"
            + (", target offloaded (per-layer H2D streaming)" if name in OFFLOAD else ", target resident in HBM"))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--scoring", choices=["raw", "warped"], default=None,
                    help="raw: score the tree with the draft's raw distribution (SURVEY F2); "
                         "warped: reference default (t=0 -> greedy chain)")
    ap.add_argument("--synthetic", type=float, default=0.0,
                    help="scale of the shared synthetic prev-token logit bias (0 = pure random init)")
    ap.add_argument("--prompt-len", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 legs (demo pair + tiny Llama end to end)")
    ap.add_argument("--c3-steps", type=int, default=3,
                    help="C2 runs only: timed iterations of the stage-3 block (70B target offloaded to pinned host "
                         "RAM, per-layer streaming, K=2048, t=0.6/top-p 0.9) after the C2 line's own timing; 0 = skip")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sequential", action="store_true", help="skip the sequential-decoding speed-up denominator")
    ap.add_argument("--offload-buffers", type=int, default=8,
                    help="offload mode: HBM staging slots of the per-layer weight ring (2 = double buffering)")
    ap.add_argument("--parallel", choices=["tp", "replicas"], default="tp",
                    help="N>1: tensor-parallel target (one stream) or N independent replicas")
    ap.add_argument("--reduce", choices=["bf16", "fp32"], default="bf16", help="TP all-reduce precision")
    ap.add_argument("--tp-rows", choices=["argmax", "gather"], default="argmax",
                    help="TP target at t=0: return per-row argmax keys (KV1: int64 MAX all-reduce of N x 8 B) "
                         "instead of all-gathering the [N, V/n] logit slices")
    ap.add_argument("--tp-comm", choices=["fused", "nccl"], default="nccl",
                    help="TP reduction: NCCL all-reduce (default, north_star), or the opt-in GEMM epilogue "
                         "reduce-scatter over peer memory (not yet run on multi-GPU hardware)")
    ap.add_argument("--attn", choices=["auto", "mma", "tc"], default="auto",
                    help="tree attention kernel: by shape (default), the mma.sync loop only, tcgen05 only (A/B)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sus": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int, device: str = "cuda") -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int, device: str = "cuda") -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def measure_h2d(torch, nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Pinned host -> device copy bandwidth (GB/s) on this box (the host-link
    roofline of the offloaded target; not in MEASURED_PEAKS.json)."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst.copy_(src, non_blocking=True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    gbs = reps * nbytes / (s.elapsed_time(e) / 1e3) / 1e9
    del src, dst
    return gbs


def ncu_traffic(prefix: str = "gemm_tc_kernel<2") -> tuple[float | None, str]:
    """DRAM bytes per launch of the dominant kernel from the committed `ncu --set
    full` captures (profiles/*/ncu_summary.json; one capture per target-pass
    GEMM shape, each launched once per layer, so the plain mean is the per-launch
    average of the pass)."""
    best = None
    for f in sorted(ROOT.glob("profiles/*/ncu_summary.json")):
        rows = [r for r in json.loads(f.read_text()) if prefix in r.get("kernel", "") and r.get("dram_bytes")
                and "70b" in r.get("report", "")]
        if rows:
            best = (sum(r["dram_bytes"] for r in rows) / len(rows), f"{f.relative_to(ROOT)} ({len(rows)} shapes)")
    return best if best else (None, "no ncu capture committed")


# ----------------------------------------------------------------------------- CPU reference path
ACCEPT_FILE = ROOT / "profiles" / "accept_by_workload.json"


def bench_config(args, K: int, B: int, scoring: str) -> dict:
    """`config` of the JSON line -- identical in both arms (the same workload)."""
    dname, tname = WORKLOADS[args.workload][:2]
    from paper_2406_02532_b200.llama import PRESETS

    tb = PRESETS[tname].weight_bytes() + PRESETS[dname].weight_bytes()
    cfg = {"workload": workload_desc(args.workload, K, B), "scoring": scoring, "prompt_len": args.prompt_len,
           "l2": (f"weights {tb / 1e9:.0f} GB >> 126 MB L2, streamed every step (no flush needed)" if tb > 1e9
                  else f"weights {tb / 1e6:.0f} MB: L2-resident across steps (demo size, not a bench line)")}
    if args.workload in OFFLOAD:
        cfg["offload_buffers"] = args.offload_buffers
    return cfg


def recorded_acceptance(workload: str) -> tuple[float, float, str]:
    """(accepted tokens / iteration, draft calls / iteration, source) of the GPU
    arm on the same workload and seeds, from the committed record (the driver
    runs the reference arm first, so it cannot read the GPU arm's live value)."""
    try:
        rec = json.loads(ACCEPT_FILE.read_text())[workload]
        return rec["accepted_tokens_per_iter"], rec["draft_calls_per_iter"], f"{ACCEPT_FILE.name}: {rec['source']}"
    except (OSError, KeyError, ValueError):
        return 1.0, 2.0, "no recorded GPU acceptance for this workload: 1.0 assumed"


class CpuIterationSampler:
    """The reference's CPU path for one target iteration, timed on this host
    (SURVEY 8(d)): every piece that runs is measured, none is assumed.

    Per sample: one fp32 decoder layer of the target over the K+1 tree tokens
    (queries) against prompt + tree keys under the tree's ancestor mask, the
    target LM head over those K+1 rows, one draft decoder layer over a batch of
    B rows and the draft LM head (the batched round), the draft's one-token root
    round (layer + head), the reference tree bookkeeping -- oracle build_sssp
    (the restatement of pkg/src/speckit/tree.py:240-327, pinned to the
    reference's fixtures) at the workload's K, D, B, V on logits rows -- and the
    walk (apply_warp + sample + advance, engine.py:118-128) for the accepted
    tokens. The iteration time is L_target x layer + head + draft (root +
    (rounds - 1) x (L_draft x layer + head)) + tree + walk; only the layer count
    is extrapolated (every layer has the same shapes). Weights are fp32 N(0,
    0.02), allocated once outside the timed sample."""

    def __init__(self, workload: str, K: int, B: int, prompt_len: int, threads: int):
        import numpy as np
        import torch

        from oracle import llama_ref
        from paper_2406_02532_b200.llama import PRESETS

        self.torch, self.np, self.ref = torch, np, llama_ref
        torch.set_num_threads(threads)
        self.threads = threads
        w = WORKLOADS[workload]
        self.dcfg, self.tcfg = PRESETS[w[0]], PRESETS[w[1]]
        self.K, self.D, self.B, self.temp, self.top_p = K, w[3], B, w[5], w[6]
        self.ctx = prompt_len
        g = torch.Generator().manual_seed(0)
        self.Wt = self._layer(self.tcfg, g)
        self.Wd = self._layer(self.dcfg, g)
        self.lm_t = torch.randn(self.tcfg.vocab, self.tcfg.d, generator=g) * 0.02
        self.lm_d = torch.randn(self.dcfg.vocab, self.dcfg.d, generator=g) * 0.02
        # a random tree of K nodes (depth <= D) for the target pass mask
        rng = np.random.default_rng(0)
        depth, parent = [0], [-1]
        for i in range(1, K + 1):
            cand = int(rng.integers(max(0, i - 64), i))
            while depth[cand] >= self.D:
                cand = parent[cand]
            parent.append(cand)
            depth.append(depth[cand] + 1)
        self.t_mask, self.t_pos = self._tree_mask(parent, depth)
        self.d_mask, self.d_pos = self._tree_mask(parent[: B], depth[: B])

    @staticmethod
    def _layer(cfg, g):
        import torch

        r = lambda *s: torch.randn(*s, generator=g) * 0.02  # noqa: E731
        return {"wqkv": r(cfg.qkv_out, cfg.d), "wo": r(cfg.d, cfg.heads * cfg.head_dim), "wg": r(cfg.ff, cfg.d),
                "wu": r(cfg.ff, cfg.d), "wd": r(cfg.d, cfg.ff), "n1": torch.ones(cfg.d), "n2": torch.ones(cfg.d)}

    def _tree_mask(self, parent, depth):
        torch = self.torch
        n = len(parent)
        allow = torch.zeros((n, self.ctx + n), dtype=torch.bool)
        allow[:, : self.ctx] = True
        for i in range(n):
            if parent[i] >= 0:
                allow[i, self.ctx : self.ctx + n] = allow[parent[i], self.ctx : self.ctx + n]
            allow[i, self.ctx + i] = True
        mask = torch.zeros(allow.shape).masked_fill(~allow, float("-inf"))
        return mask, torch.tensor([self.ctx - 1 + d for d in depth])

    def _layer_time(self, cfg, L, n, mask, pos) -> float:
        torch, ref = self.torch, self.ref
        H, KVH, hd = cfg.heads, cfg.kv_heads, cfg.head_dim
        g = torch.Generator().manual_seed(1)
        x = torch.randn(n, cfg.d, generator=g)
        kv_ctx = torch.randn(self.ctx, KVH, hd, generator=g)
        t0 = time.perf_counter()
        with torch.no_grad():
            h = ref.rmsnorm(x, L["n1"], cfg.eps)
            qkv = h @ L["wqkv"].t()
            q = ref.rope(qkv[:, : H * hd].view(n, H, hd), pos, cfg.rope_theta)
            k = ref.rope(qkv[:, H * hd : (H + KVH) * hd].view(n, KVH, hd), pos, cfg.rope_theta)
            v = qkv[:, (H + KVH) * hd :].view(n, KVH, hd)
            k = torch.cat([kv_ctx, k]).repeat_interleave(H // KVH, dim=1)
            v = torch.cat([kv_ctx, v]).repeat_interleave(H // KVH, dim=1)
            s = torch.einsum("qhd,khd->hqk", q, k) / hd**0.5 + mask
            att = torch.einsum("hqk,khd->qhd", s.softmax(-1), v).reshape(n, H * hd)
            x = x + att @ L["wo"].t()
            h = ref.rmsnorm(x, L["n2"], cfg.eps)
            x = x + (torch.nn.functional.silu(h @ L["wg"].t()) * (h @ L["wu"].t())) @ L["wd"].t()
        return time.perf_counter() - t0

    def _head_time(self, lm, n, d) -> float:
        torch = self.torch
        h = torch.randn(n, d)
        t0 = time.perf_counter()
        with torch.no_grad():
            z = h @ lm.t()
            z.max(dim=1)
        return time.perf_counter() - t0

    def sample(self, accepted: float, rounds: float) -> dict:
        from oracle import speckit_oracle as ox

        torch = self.torch
        tc, dc, K, B = self.tcfg, self.dcfg, self.K, self.B
        t_wall = time.perf_counter()
        t_layer = self._layer_time(tc, self.Wt, K + 1, self.t_mask, self.t_pos)
        t_head = self._head_time(self.lm_t, K + 1, tc.d)
        d_layer = self._layer_time(dc, self.Wd, B, self.d_mask, self.d_pos)
        d_head = self._head_time(self.lm_d, B, dc.d)
        root_mask = torch.zeros((1, self.ctx + 1))
        d_root = self._layer_time(dc, self.Wd, 1, root_mask, torch.tensor([self.ctx - 1])) * dc.layers \
            + self._head_time(self.lm_d, 1, dc.d)
        t0 = time.perf_counter()
        lm = ox.LogitsLM(tc.vocab, ox.hashed_logits_fn(tc.vocab, 11, 1.3))
        warp = ox.SamplingConfig(self.temp, self.top_p) if self.temp > 0 else None
        tree = ox.build_sssp(tuple(range(8)), lm, ox.BuilderParams(K, self.D, B), warp, warp_scores=warp is not None)
        t_tree = time.perf_counter() - t0
        t0 = time.perf_counter()
        rng = ox.CounterRng(0, "generation")
        row = lm.next_distributions([tuple(range(9))])[0]
        cfg = ox.SamplingConfig(self.temp, self.top_p, seed=0)
        for _ in range(max(1, int(round(accepted)))):
            ox.sample(ox.apply_warp(row, cfg), rng)
            tree.child_with_token(-1, 0)
        t_walk = time.perf_counter() - t0
        per_iter = (t_layer * tc.layers + t_head + d_root + max(0.0, rounds - 1) * (d_layer * dc.layers + d_head)
                    + t_tree + t_walk)
        return {"seconds_per_iteration": per_iter, "sample_seconds": time.perf_counter() - t_wall,
                "parts_s": {"target_layer": t_layer, "target_lm_head": t_head, "draft_layer_batch": d_layer,
                            "draft_lm_head_batch": d_head, "draft_root_round": d_root, "tree_bookkeeping": t_tree,
                            "walk": t_walk}}

    def describe(self, accepted: float, rounds: float, src: str) -> str:
        tc, dc = self.tcfg, self.dcfg
        return (f"measured per sample: one fp32 {tc.name} layer over K+1={self.K + 1} tree queries (ctx "
                f"{self.ctx}, tree mask) + its LM head, one {dc.name} layer at B={self.B} + LM head, the draft root "
                f"round, oracle build_sssp K={self.K} D={self.D} B={self.B} V={tc.vocab}, the walk; layers x "
                f"{tc.layers} / {dc.layers}, {rounds:.1f} draft calls and {accepted:.2f} accepted tokens per iteration "
                f"({src}); {self.threads} threads")


def c1_legs(gpu: bool, threads: int) -> dict:
    """BASELINE configs[0] (C1) end to end: the reference demo pair
    (pkg/demos/03_cached_generation.py:19-20: make_synthetic(3, 16, 0.05), draft =
    power_smoothed(0.7)) and a tiny Llama pair (tiny-draft -> tiny, weights drawn
    on the host so both arms use the same values), one 128-token prompt, K=128,
    D=16, B=8, t=0 (the Llama pair with raw draft scoring). gpu=False:
    through the CPU reference path (oracle engine; CpuLlamaLM = fp32 TorchCpuLlama
    plugin); gpu=True: through this package's public API on cuda:0."""
    import hashlib

    import numpy as np

    def leg(fn, n_tok):
        t0 = time.perf_counter()
        toks, stats = fn()
        if gpu:
            import torch

            torch.cuda.synchronize()
        el = time.perf_counter() - t0
        return {"tokens_per_s": len(toks) / el, "tokens": len(toks), "seconds": el,
                "accepted_per_iter": stats.generation_rate,
                "tokens_sha1": hashlib.sha1(json.dumps(list(toks)).encode()).hexdigest()[:12]}

    out = {}
    rng = np.random.default_rng(1000)
    demo_prompt = tuple(int(t) for t in rng.integers(0, 16, size=128))
    llama_prompt = tuple(int(t) for t in rng.integers(0, 32000, size=128))
    if gpu:
        import paper_2406_02532_b200 as sx
        from paper_2406_02532_b200.llama import LlamaModel

        tgt = sx.make_synthetic(3, 16, 0.05)
        drf = tgt.power_smoothed(0.7)
        cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=256)
        sx.generate_specexec(demo_prompt, drf, tgt, sx.BuilderParams(128, 16, 8), cfg)  # warm
        out["demo03"] = leg(lambda: sx.generate_specexec(demo_prompt, drf, tgt, sx.BuilderParams(128, 16, 8), cfg), 256)
        lt = LlamaModel("tiny", seed=1, max_ctx=2048, max_tokens=256, init="host")
        ld = LlamaModel("tiny-draft", seed=2, max_ctx=4096, max_tokens=256, init="host")
        cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=8)
        sx.generate_specexec(llama_prompt, ld, lt, sx.BuilderParams(128, 16, 8), cfg, warp_scores=False)  # warm
        cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=16)
        out["tiny_llama"] = leg(lambda: sx.generate_specexec(llama_prompt, ld, lt, sx.BuilderParams(128, 16, 8), cfg,
                                                             warp_scores=False), 16)
        del lt, ld
    else:
        import torch

        from oracle import llama_ref
        from oracle import speckit_oracle as ox
        from paper_2406_02532_b200.llama import PRESETS, host_weights_fp32

        torch.set_num_threads(threads)
        tgt = ox.make_synthetic(3, 16, 0.05)
        drf = tgt.power_smoothed(0.7)
        cfg = ox.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=256)
        out["demo03"] = leg(lambda: ox.generate_specexec(demo_prompt, drf, tgt, ox.BuilderParams(128, 16, 8), cfg), 256)
        lt = llama_ref.CpuLlamaLM(PRESETS["tiny"], host_weights_fp32(PRESETS["tiny"], 1))
        ld = llama_ref.CpuLlamaLM(PRESETS["tiny-draft"], host_weights_fp32(PRESETS["tiny-draft"], 2))
        cfg = ox.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=16)
        out["tiny_llama"] = leg(lambda: ox.generate_specexec(llama_prompt, ld, lt, ox.BuilderParams(128, 16, 8), cfg,
                                                             warp_scores=False), 16)
    out["config"] = "C1: demo03 pair V=16 and tiny Llama pair (d=256, V=32000), 128-token prompt, K=128 D=16 B=8 t=0"
    return out


def cpu_baseline(args, K: int, B: int, accepted: float, rounds: float, src: str) -> dict:
    """The CPU reference path beside the GPU run (rank 0, N=1): one bounded sample."""
    threads = os.cpu_count() or 1
    sampler = CpuIterationSampler(args.workload, K, B, args.prompt_len, threads)
    smp = sampler.sample(accepted, rounds)
    return {"value": accepted / smp["seconds_per_iteration"], "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": sampler.describe(accepted, rounds, src), "seconds_per_iteration": smp["seconds_per_iteration"],
            "parts_s": smp["parts_s"], "sample_seconds": smp["sample_seconds"], "extrapolated": "layer count only"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """`--impl reference`: the reference's CPU implementation of the path timed on
    this box's host cores (the oracle port: the reference is pure Python and
    cannot travel; its restatement is pinned to its fixtures). Rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    K = args.budget or w[2]
    B = args.batch or w[4]
    scoring = args.scoring or ("raw" if w[5] == 0.0 else "warped")
    threads = os.cpu_count() or 1
    accepted, rounds, src = recorded_acceptance(args.workload)
    sampler = CpuIterationSampler(args.workload, K, B, args.prompt_len, threads)
    per_iter, walls, parts = [], [], None
    for i in range(args.warmup + args.steps):
        smp = sampler.sample(accepted, rounds)
        if i >= args.warmup:
            per_iter.append(smp["seconds_per_iteration"])
            walls.append(smp["sample_seconds"])
            parts = smp["parts_s"]
    sec = statistics.mean(per_iter)
    value = accepted / sec
    c1 = c1_legs(gpu=False, threads=threads) if not args.no_c1 else None
    cb = {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
          "sample": sampler.describe(accepted, rounds, src), "seconds_per_iteration": sec, "parts_s": parts,
          "extrapolated": "layer count only"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(args, K, B, scoring),
            "step": "one measured CPU sample of a target iteration (ms_per_step = its wall time); value = "
                    "accepted tokens / the iteration time assembled from the sample",
            "accepted_tokens_per_iter": accepted, "draft_calls_per_iter": rounds,
            "cpu_baseline": cb, "c1": c1,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- stage 3 block
def measure_c3(args, draft, prompt, resident_pass_ms: float, resident_pass_tokens: int) -> dict:
    """BASELINE configs[2] (C3) on the same box after the C2 timing: the 70B
    target re-created offloaded (weights in pinned host RAM, streamed per layer
    through the HBM ring, LayerStreamer), the resident 7B draft, K=2048,
    t=0.6 / top-p 0.9 (warped scoring). Reports tokens/s and accepted tokens per
    iteration, the achieved H2D rate against the pinned rate measured here
    (north_star: >= 80 % of host-link bandwidth), sequential decoding on the
    same offloaded target (the speed-up denominator), and the cost model
    (costsim.forward_time) fitted from this run's own measurements."""
    import torch

    import paper_2406_02532_b200 as sx
    from paper_2406_02532_b200.costsim import CostModel, forward_time
    from paper_2406_02532_b200.engine import SpecExecSession
    from paper_2406_02532_b200.llama import PRESETS, LlamaModel

    dname, tname, K, D, B, temp, top_p = WORKLOADS["c3"]
    h2d_peak = measure_h2d(torch)
    t0 = time.time()
    ctx_cap = args.prompt_len + (1 + args.c3_steps + 4) * (D + 1) + 64
    target = LlamaModel(tname, seed=1, max_ctx=ctx_cap + K + 2, max_tokens=K + 1, offload=True,
                        offload_buffers=args.offload_buffers)
    torch.cuda.synchronize()
    init_s = time.time() - t0
    cfg = sx.SamplingConfig(temp, top_p, seed=0, max_new_tokens=100000)
    sess = SpecExecSession(prompt, draft, target, sx.BuilderParams(K, D, B), cfg, warp_scores=True)
    sess.step(100000)  # warm-up iteration (graph buckets at K=2048, ring fill)
    from paper_2406_02532_b200 import engine as Eng

    Eng.STAGES = Eng.StageTimer()
    bytes0, tok0, it0, dc0 = target.streamer.bytes, len(sess.tokens), sess.stats.target_calls, sess.stats.draft_calls
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    n_iter = 0
    while n_iter < args.c3_steps:
        sess.step(100000)
        if sess.cache is None:
            n_iter += 1
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    stages = {k: v / args.c3_steps for k, v in Eng.STAGES.totals().items()}
    Eng.STAGES = None
    tokens = len(sess.tokens) - tok0
    streamed = target.streamer.bytes - bytes0
    h2d = streamed / (ms / 1e3) / 1e9
    draft_calls = (sess.stats.draft_calls - dc0) / args.c3_steps
    # sequential decoding on the same offloaded target: one streamed pass per token
    cfg1 = sx.SamplingConfig(temp, top_p, seed=11, max_new_tokens=1)
    cfg2 = sx.SamplingConfig(temp, top_p, seed=11, max_new_tokens=2)
    sx.generate_sequential(prompt, target, cfg1)  # prompt KV already committed; warm
    tt = []
    for c in (cfg1, cfg2):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sx.generate_sequential(prompt, target, c)
        torch.cuda.synchronize()
        tt.append(time.perf_counter() - t1)
    seq_rate = 1.0 / max(1e-9, tt[1] - tt[0])
    value = tokens / (ms / 1e3)
    tb = PRESETS[tname].weight_bytes()
    cm = CostModel.from_b200_measurements(target_bytes=target.w.layer_bytes * target.cfg.layers,
                                          h2d_bytes_per_s=h2d_peak * 1e9, resident_pass_s=resident_pass_ms / 1e3,
                                          pass_tokens=resident_pass_tokens, draft_bytes=PRESETS[dname].weight_bytes(),
                                          draft_step_s=stages.get("draft", 0.0) / 1e3 / max(1.0, draft_calls),
                                          ring_layers=target.streamer.nbuf, layers=target.cfg.layers,
                                          draft_phase_s=stages.get("draft", 0.0) / 1e3)
    out = {"workload": workload_desc("c3", K, B), "scoring": "warped", "steps": args.c3_steps,
           "tokens_per_s": value, "ms_per_iteration": ms / args.c3_steps, "accepted_tokens_per_iter": tokens / args.c3_steps,
           "draft_calls_per_iter": draft_calls, "stage_ms_per_step": stages,
           "h2d": {"achieved_GBps": h2d, "pinned_peak_GBps": h2d_peak, "frac": h2d / h2d_peak if h2d_peak else None,
                   "bytes_per_iteration": streamed / args.c3_steps,
                   "note": "bytes the layer ring streamed during the timed iterations / their device time; peak = "
                           "pinned 1 GiB H2D copies measured in this run"},
           "sequential": {"tokens_per_s": seq_rate, "speedup_of_specexec": value / seq_rate},
           "costsim": {"preset": json.loads(cm.to_json()), "forward_time_model_s": forward_time(cm, K + 1),
                       "target_stage_measured_s": stages.get("target", 0.0) / 1e3},
           "init_seconds": init_s, "weights_streamed_GB_per_pass": tb / 1e9}
    del sess, target
    return out


# ----------------------------------------------------------------------------- B200 arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2406_02532_b200 as sx
    from paper_2406_02532_b200 import _lib
    from paper_2406_02532_b200 import kernels as Kern
    from paper_2406_02532_b200.engine import SpecExecSession
    from paper_2406_02532_b200.llama import PRESETS, LlamaModel, SyntheticBias

    dname, tname, K, D, B, temp, top_p = WORKLOADS[args.workload]
    K = args.budget or K
    B = args.batch or B
    syn = SyntheticBias(seed=99, rank=64, scale=args.synthetic) if args.synthetic > 0 else None
    tp = world > 1 and args.parallel == "tp"
    comm = None
    if tp:
        from paper_2406_02532_b200.tp import NcclComm

        comm = NcclComm()
    srank = 0 if tp else rank  # TP ranks share one generation stream (same prompt and seed)
    t_init = time.time()
    _lib.call("sx_attention_set_impl", {"auto": 0, "mma": 1, "tc": 2}[args.attn])
    max_new = 100000
    ctx_cap = args.prompt_len + (args.warmup + args.steps) * (D + 1) * 3 + 64
    offload = args.workload in OFFLOAD
    target = LlamaModel(tname, seed=1, max_ctx=ctx_cap + K + 2, max_tokens=max(K + 1, args.prompt_len), synthetic=syn,
                        offload=offload, offload_buffers=args.offload_buffers, tp=comm, reduce_bf16=args.reduce == "bf16",
                        tp_fused=True if args.tp_comm == "fused" else False,
                        tp_argmax=temp == 0.0 and args.tp_rows == "argmax")
    draft = LlamaModel(dname, seed=2, max_ctx=ctx_cap + 4 * K + 2 * B * (D + 1) + 64, max_tokens=max(B, args.prompt_len),
                       synthetic=syn)
    torch.cuda.synchronize()
    init_s = time.time() - t_init
    params = sx.BuilderParams(K, D, B)
    cfg = sx.SamplingConfig(temp, top_p, seed=srank, max_new_tokens=max_new)
    scoring = args.scoring or ("raw" if temp == 0.0 else "warped")
    warp_scores = scoring == "warped"
    h2d_peak = measure_h2d(torch) if offload else None
    prompt = tuple(int(t) for t in np.random.default_rng(1000 + srank).integers(0, PRESETS[tname].vocab, size=args.prompt_len))

    sess = SpecExecSession(prompt, draft, target, params, cfg, warp_scores)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sess.step(max_new)
    # ---------------- timed region: exactly `steps` target iterations
    Kern.PROFILER = Kern.GemmProfiler()
    from paper_2406_02532_b200 import engine as Eng

    Eng.STAGES = Eng.StageTimer()
    launches0 = _lib.load().sx_launch_count() + Kern.GRAPH_KERNELS[0]
    streamed0 = target.streamer.bytes if offload else 0
    it0, tok0, dc0 = sess.stats.target_calls, len(sess.tokens), sess.stats.draft_calls
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        n_iter = 0
        while n_iter < args.steps:
            sess.step(max_new)
            if sess.cache is None:  # the iteration ended with a miss
                n_iter += 1
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = _lib.load().sx_launch_count() + Kern.GRAPH_KERNELS[0] - launches0  # direct + graph-replayed
    prof = Kern.PROFILER
    stages = {k: v / args.steps for k, v in Eng.STAGES.totals().items()}
    Eng.STAGES = None
    Kern.PROFILER = None
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world)
    tokens = len(sess.tokens) - tok0
    iters = sess.stats.target_calls - it0 + (0 if sess.cache is None else -1)
    iters = max(iters, args.steps)
    draft_calls = sess.stats.draft_calls - dc0
    total_tokens = tokens if tp else sum_over_ranks(tokens, world)
    value = total_tokens / (ms_max / 1e3)
    accepted_per_iter = tokens / args.steps

    # dominant kernel: the tcgen05 GEMM of the target pass over the tree
    pk = peaks()
    # iteration roofline: target pass = its GEMM FLOPs at the sustained bf16 peak;
    # draft = per call max(FLOPs at peak, weight bytes at HBM) over the rows it
    # forwards (B per batched round, 1 for the root round); walk/host ~ 0
    tcfg, dcfg = PRESETS[tname], PRESETS[dname]
    dcalls = draft_calls / max(1, iters)
    d_params = dcfg.n_params() - dcfg.vocab * dcfg.d  # embedding rows are gathered, not multiplied
    d_round = lambda rows: max(2.0 * rows * d_params / (pk["bf16_sus"] * 1e12),  # noqa: E731
                               dcfg.weight_bytes() / (pk["hbm"] * 1e9))
    draft_bound = d_round(1) + max(0.0, dcalls - 1) * d_round(B)
    if offload:
        target_bound = PRESETS[tname].weight_bytes() / (h2d_peak * 1e9) if h2d_peak else 0.0
    else:
        t_params = tcfg.n_params() - tcfg.vocab * tcfg.d
        target_bound = 2.0 * (K + 1) * t_params / (pk["bf16_sus"] * 1e12)
    if tp:
        target_bound /= world  # the target pass is sharded over the ranks
    roof_s = draft_bound + target_bound
    iter_roofline = {"target_bound_ms": target_bound * 1e3, "draft_bound_ms": draft_bound * 1e3,
                     "tokens_per_s_at_roofline": accepted_per_iter / roof_s if roof_s > 0 else None,
                     "frac": (roof_s * 1e3) / (ms_max / args.steps) if ms_max > 0 else None,
                     "note": "target: 2*(K+1)*params at the measured sustained bf16 peak (offload: weight bytes at the "
                             "measured pinned H2D rate); draft: per call max(2*rows*params at peak, weights at HBM)"}
    gemm_shapes = prof.by_shape(steps=args.steps)
    big = prof.summary(min_m=max(2, K // 2))
    small = prof.summary(min_m=0)
    ach = big["flops"] / (big["ms"] / 1e3) / 1e12 if big["ms"] > 0 else 0.0
    gemm_share = small["ms"] / ms if ms > 0 else 0.0
    traffic, traffic_src = ncu_traffic()
    roof = {"bound": "tensor", "kernel": "gemm_tc_kernel (target pass, M=K+1 tree tokens)", "achieved": ach,
            "peak": pk["bf16_sus"], "unit": "TFLOP/s", "frac": ach / pk["bf16_sus"] if pk["bf16_sus"] else None,
            "peak_source": f"{pk['src']} bf16 sustained (MEASURED_PEAKS.json)", "traffic": traffic,
            "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
            "traffic_source": traffic_src,
            "launches": big["launches"], "gemm_share_of_step": gemm_share,
            "flops_per_launch_avg": big["flops"] / max(1, big["launches"])}

    clk = clocks.summary()
    if offload:
        # stage 3 bound: host link. achieved = bytes streamed in the timed region / its device time
        streamed = target.streamer.bytes - streamed0
        h2d = streamed / (ms / 1e3) / 1e9
        roof = {"bound": "h2d", "kernel": "per-layer weight streaming (sx_stream_copy, copy engines)", "achieved": h2d,
                "peak": h2d_peak, "unit": "GB/s", "frac": h2d / h2d_peak if h2d_peak else None,
                "peak_source": "pinned H2D measured in this run (1 GiB x5)", "traffic": None,
                "bytes_per_step": streamed / args.steps,
                "costsim_forward_s": PRESETS[tname].weight_bytes() / (h2d_peak * 1e9) if h2d_peak else None,
                "gemm_target_pass_tflops": ach}
    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Kern.IO["h2d"] = Kern.IO["d2h"] = 0
        prompt2 = tuple(int(t) for t in np.random.default_rng(2000 + srank).integers(0, PRESETS[tname].vocab,
                                                                                        size=args.prompt_len))
        cfg2 = sx.SamplingConfig(temp, top_p, seed=srank + 7,
                                 max_new_tokens=max(1, int(round(accepted_per_iter * args.steps))))
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        toks2, st2 = sx.generate_specexec(prompt2, draft, target, params, cfg2, warp_scores=warp_scores)
        torch.cuda.synchronize()
        el = max_over_ranks(time.perf_counter() - t0, world)
        n_it = max(1, st2.target_calls)
        h2d = Kern.IO["h2d"] + 8 * len(prompt2)
        e2e = {"value": (len(toks2) if tp else sum_over_ranks(len(toks2), world)) / el, "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d / n_it), "d2h_bytes_per_step": int((Kern.IO["d2h"] + 4 * len(toks2)) / n_it),
               "iterations": n_it, "includes": "prompt prefill, tree builds, target passes, walks, host sync per round"}

    # ---------------- the speed-up denominator: sequential decoding on the same GPU(s)
    # (generate_sequential, engine.py:134-148): one target pass
    # per token through the one-token CUDA graph, prompt KV already cached.
    seq = None
    if not args.no_sequential:
        n_seq = 2 if offload else 16
        cfg_w = sx.SamplingConfig(temp, top_p, seed=srank + 11, max_new_tokens=2)
        cfg_s = sx.SamplingConfig(temp, top_p, seed=srank + 11, max_new_tokens=2 + n_seq)
        sx.generate_sequential(prompt, target, cfg_s)  # warm: prompt sync, graph capture
        times = [float("inf"), float("inf")]
        for _ in range(1 if offload else 3):  # min of repeats: host-side jitter off the difference
            for i, c in enumerate((cfg_w, cfg_s)):
                barrier(world)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sx.generate_sequential(prompt, target, c)
                torch.cuda.synchronize()
                times[i] = min(times[i], max_over_ranks(time.perf_counter() - t0, world))
        rate = n_seq / max(1e-9, times[1] - times[0])
        if not tp:
            rate = sum_over_ranks(rate, world)
        seq = {"tokens_per_s": rate, "tokens_timed": n_seq, "ms_per_token": 1e3 / (rate if tp else rate / world),
               "speedup_of_value": value / rate,
               "note": "target-only decoding, one token per target pass (CUDA graph), prompt KV cached; "
                       "difference of a (2 + n)- and a 2-token run, min of 3 each"}

    c3 = None
    if world == 1 and args.workload == "c2" and args.c3_steps > 0:
        import gc

        resident_pass_ms = stages.get("target", 0.0)
        del sess
        target = None
        gc.collect()
        torch.cuda.empty_cache()
        c3 = measure_c3(args, draft, prompt, resident_pass_ms, K + 1)
        gc.collect()
        torch.cuda.empty_cache()
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args, K, B, accepted_per_iter, draft_calls / max(1, iters),
                          f"live: this run's {args.steps} timed iterations")
    c1 = None
    if rank == 0 and world == 1 and not args.no_c1:
        c1 = c1_legs(gpu=True, threads=os.cpu_count() or 1)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong" if tp else "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic: random-init weights (N(0,0.02)), random 128-token prompt" +
                    (f", shared synthetic prev-token bias scale {args.synthetic}" if syn else ""),
            "config": bench_config(args, K, B, scoring),
            "parallelism": (f"tp{world} target ({'fused GEMM reduce-scatter over peer memory' if target.tp_fused else 'NCCL all-reduce'}, {args.reduce}"
                            f"{', KV1 argmax keys' if target.tp_argmax else ''}), draft replicated"
                            if tp else f"replicas x{world}") if world > 1 else "1 GPU",
            "accepted_tokens_per_iter": accepted_per_iter,
            "draft_calls_per_iter": draft_calls / max(1, iters),
            "stage_ms_per_step": stages,
            "iteration_roofline": iter_roofline,
            "gemm_shapes": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()} for r in gemm_shapes],
            "roofline": roof,
            "cpu_baseline": cb,
            "c1": c1,
            "c3": c3,
            "e2e": e2e,
            "sequential": seq,
            "gpu_launches": launches,
            "clocks": clk,
            "init_seconds": init_s,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
