#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python tools/acceptance_sweep.py --draft llama3-8b --target llama3-70b --budgets 64,256,1024,4096,8192 --batch 512 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c5.jsonl > gpurun_out/acceptance_c5.log 2>&1
