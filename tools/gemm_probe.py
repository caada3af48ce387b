"""GEMM issue/feed probe: one tile per SM (pair: per SM pair), K=16384, for
single vs pair kernels, with and without TMA after the ring fill
(SX_GEMM_DEBUG=1), over token-tile widths. Reports cycles per k-block per SM
against the tcgen05 floor (4 MMAs x 128 x BN x 16 / 4096 MAC/clk).
Usage: python tools/gemm_probe.py            (driver: spawns one process per env)
"""
import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]


def child(mode: int, bns: list[int]):
    import torch

    sys.path.insert(0, str(ROOT))
    from paper_2406_02532_b200 import _lib
    from paper_2406_02532_b200 import kernels as K

    _lib.call("sx_gemm_set_pair_mode", mode)
    Kd = 16384
    for bn in bns:
        M, N = bn, 148 * 128
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        w = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16()
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for _ in range(2):
            K.gemm(x, w, out=out, splits=1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            K.gemm(x, w, out=out, splits=1)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        clk = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True).stdout.strip() or 1965)
        cyc = ms * 1e-3 * clk * 1e6 / (Kd // 64)
        ideal = 4 * 128 * bn * 16 / 4096
        print(json.dumps({"mode": mode, "debug": os.environ.get("SX_GEMM_DEBUG", "0"), "bn": bn,
                          "tflops": 2 * M * N * Kd / ms / 1e9, "cyc_per_kb": cyc, "ideal": ideal, "clk": clk}),
              flush=True)
        del x, w, out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), [int(b) for b in sys.argv[3].split(",")])
        sys.exit(0)
    for mode in (1, 2):
        for kpb in ("1", "2"):
            for dbg in ("0", "1"):
                env = dict(os.environ, SX_GEMM_DEBUG=dbg, SX_GEMM_KPB=kpb)
                print(f"# mode={mode} kpb={kpb} debug={dbg}", flush=True)
                subprocess.run([sys.executable, __file__, "child", str(mode), "64,128,208,256"], env=env, check=False)
