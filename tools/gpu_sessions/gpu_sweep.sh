#!/bin/bash
# acceptance-vs-budget sweeps (SpecExec vs SpecInfer), sharp synthetic variant
mkdir -p gpurun_out
timeout 1800 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 64,256,1024,2048,4096 --batch 1024 --methods sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c2.jsonl > gpurun_out/acceptance_c2.log 2>&1
timeout 1800 python tools/acceptance_sweep.py --draft llama3-8b --target llama3-70b --budgets 64,256,1024,4096,8192 --batch 512 --methods sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c5.jsonl > gpurun_out/acceptance_c5.log 2>&1
