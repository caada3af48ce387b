"""Plan sweep for the tcgen05 GEMM: every candidate plan request
(cg = single / pair, token-tile cap, schedule) on the shapes the SpecExec
models run, vs the automatic plan. Output: JSON lines + a best-vs-auto table.

  python tools/gemm_plan_sweep.py [--set c2] [--out gpurun_out/plan_sweep.jsonl]

req = sched | cg << 4 | (bn_cap // 16) << 8  (csrc/gemm_tc.cu make_plan)
"""

import argparse
import json
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import kernels as K  # noqa: E402

IL, F32, BF16 = K.EPI_SWIGLU_IL, K.EPI_F32, K.EPI_BF16
SETS = {
    "c2": [
        ("70b.qkv", 1025, 10240, 8192, BF16), ("70b.o", 1025, 8192, 8192, F32),
        ("70b.gate_up", 1025, 57344, 8192, IL), ("70b.down", 1025, 8192, 28672, F32),
        ("70b.lm", 1025, 32000, 8192, F32),
        ("7b.qkv", 256, 12288, 4096, BF16), ("7b.o", 256, 4096, 4096, F32),
        ("7b.gate_up", 256, 22016, 4096, IL), ("7b.down", 256, 4096, 11008, F32),
        ("7b.lm", 256, 32000, 4096, F32),
        ("7b.qkv.m1", 1, 12288, 4096, BF16), ("7b.o.m1", 1, 4096, 4096, F32),
        ("7b.gate_up.m1", 1, 22016, 4096, IL), ("7b.down.m1", 1, 4096, 11008, F32),
    ],
    "draft1024": [
        ("7b.qkv", 1024, 12288, 4096, BF16), ("7b.o", 1024, 4096, 4096, F32),
        ("7b.gate_up", 1024, 22016, 4096, IL), ("7b.down", 1024, 4096, 11008, F32),
        ("7b.lm", 1024, 32000, 4096, F32),
    ],
    "c4": [
        ("70b.qkv", 4097, 10240, 8192, BF16), ("70b.o", 4097, 8192, 8192, F32),
        ("70b.gate_up", 4097, 57344, 8192, IL), ("70b.down", 4097, 8192, 28672, F32),
    ],
}


def timeit(fn, n):
    fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="c2")
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=None)
    ap.add_argument("--fine", action="store_true", help="pair tiles over every token-tile width 64..256")
    a = ap.parse_args()
    recs = []
    for name, M, N, Kd, epi in SETS[a.set]:
        if not name.startswith(a.only):
            continue
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        nw = max(1, min(4, int(3e8 // (N * Kd * 2)) + 1))  # rotate copies so weights stream from HBM
        ws = [(torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() for _ in range(nw)]
        out = torch.empty(M, N // 2 if epi == IL else N, dtype=torch.float32 if epi == F32 else torch.bfloat16,
                          device="cuda")
        flops = 2.0 * M * N * Kd
        reps = 8 if M > 64 else 30
        i = [0]

        def run(req):
            K.gemm(x, ws[i[0] % nw], out=out, epi=epi, splits=req)
            i[0] += 1

        cands = [0]
        if a.fine:  # pair tiles, whole tiles / split tail, every token-tile width
            for bn in range(64, 257, 16):
                for sched in (1, 3):
                    cands.append(sched | 2 << 4 | (bn // 16) << 8)
        else:
            for cg in (1, 2):
                for bn in (0, 64, 128, 208, 256):
                    for sched in (1, 3, 2):
                        cands.append(sched | cg << 4 | (bn // 16) << 8)
        ok = []
        for req in cands:  # drop illegal combinations
            try:
                run(req)
                ok.append(req)
            except Exception:  # noqa: BLE001
                pass
        torch.cuda.synchronize()
        # round-robin over the candidates (3 passes, min per candidate) so clock
        # drift under the power cap does not favour early candidates
        best_us = {r: float("inf") for r in ok}
        for _ in range(3):
            for req in ok:
                best_us[req] = min(best_us[req], timeit(lambda: run(req), reps))
        for req in ok:
            plan = K.gemm_plan(M, N, Kd, False, req)
            recs.append({"shape": name, "M": M, "N": N, "K": Kd, "req": req, "us": best_us[req], "plan": plan,
                         "tflops": flops / best_us[req] / 1e6, "auto": req == 0})
        auto_us = best_us[0]
        best = min((us, r) for r, us in best_us.items())
        print(f"{name:14s} M={M:5d} auto {auto_us:8.1f} us ({flops / auto_us / 1e6:6.0f} TF) plan={K.gemm_plan(M, N, Kd, False, 0)}"
              f" | best {best[0]:8.1f} us req={best[1]} (cg={(best[1] >> 4) & 3} bn={((best[1] >> 8) & 255) * 16}"
              f" sched={best[1] & 15}) plan={K.gemm_plan(M, N, Kd, False, best[1])}", flush=True)
        del ws, x, out
        torch.cuda.empty_cache()
    if a.out:
        pathlib.Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in recs))


if __name__ == "__main__":
    main()
