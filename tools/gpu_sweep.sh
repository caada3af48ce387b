#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_llama_gpu.py -x -q -k large_tree > gpurun_out/pytest_large.log 2>&1
timeout 1800 python tools/acceptance_sweep.py --draft llama3-8b --target llama3-70b --budgets 64,256,1024,4096 --methods sx,si --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c5.jsonl > gpurun_out/acceptance_c5.log 2>&1
timeout 900 python tools/acceptance_sweep.py --draft llama3-8b --target llama3-70b --budgets 8192 --methods sx --seeds 1 --tokens 16 --synthetic 4 --out gpurun_out/acceptance_c5_8192.jsonl > gpurun_out/acceptance_c5_8192.log 2>&1
