#!/bin/bash
# round-2 acceptance / throughput vs budget (the metric's second half), sharp synthetic pairs, current kernels
mkdir -p gpurun_out
timeout 1800 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 16,64,256,1024,2048 --batch 1024 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/sw_c2.jsonl > gpurun_out/sw_c2.log 2>&1
timeout 2400 python tools/acceptance_sweep.py --draft llama3-8b --target llama3-70b --budgets 64,256,1024,4096,8192 --batch 512 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/sw_c5.jsonl > gpurun_out/sw_c5.log 2>&1
