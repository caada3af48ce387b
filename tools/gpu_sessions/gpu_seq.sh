#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1200 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 64,256,1024,2048 --batch 1024 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c2.jsonl > gpurun_out/acceptance_c2.log 2>&1
timeout 1200 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 64,256,1024,2048 --batch 1024 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --t 0.6 --top-p 0.9 --out gpurun_out/acceptance_c2_t06.jsonl > gpurun_out/acceptance_c2_t06.log 2>&1
