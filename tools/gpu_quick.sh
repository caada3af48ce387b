#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py -x -q > gpurun_out/pytest_q.log 2>&1
timeout 900 python bench.py --synthetic 4 --no-cpu-baseline > gpurun_out/bench_c2_sharp.json 2> gpurun_out/bench_c2_sharp.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python tools/gemm_plan_sweep.py --set c2 --only 7b --out gpurun_out/plan_sweep_7b.jsonl > gpurun_out/plan_sweep_7b.txt 2>&1
