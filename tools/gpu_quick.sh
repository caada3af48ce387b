#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_q.log 2>&1
timeout 600 python tools/gemm_plan_sweep.py --set c2 --only 70b.gate_up --out gpurun_out/ps_gu.jsonl > gpurun_out/ps_gu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
