#!/bin/bash
mkdir -p gpurun_out
python tools/attn_probe.py > gpurun_out/probe_thr8.log 2>&1
SX_ATTN_RESCALE=0 python tools/attn_probe.py > gpurun_out/probe_thr0.log 2>&1
SX_ATTN_RESCALE=0 timeout 900 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 256,1024 --batch 1024 --methods sx --seeds 2 --tokens 48 --synthetic 4 --attn auto --out gpurun_out/acc_auto0.jsonl > gpurun_out/acc_auto0.log 2>&1
