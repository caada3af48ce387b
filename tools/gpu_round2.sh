#!/bin/bash
# tests + plan sweep + idle gaps + bench + step profile
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/gemm_plan_sweep.py --set c2 --out gpurun_out/plan_sweep_c2.jsonl > gpurun_out/plan_sweep_c2.txt 2>&1
timeout 600 python tools/idle_gaps.py > gpurun_out/idle_gaps.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python tools/profile_step.py --json gpurun_out/kernels_c2.json > gpurun_out/profile_step.txt 2>&1
