#!/bin/bash
# evidence refresh: offloaded C3 with the sharp synthetic pair (SpecExec vs sequential under offload), C2 t=0.6 sweep
mkdir -p gpurun_out
timeout 2000 python bench.py --workload c3 --steps 6 --warmup 3 --synthetic 4 --no-cpu-baseline > gpurun_out/ap_c3_sharp.json 2> gpurun_out/ap_c3_sharp.err
timeout 1800 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 16,64,256,1024 --batch 1024 --methods seq,sx,si --seeds 1 --tokens 32 --synthetic 4 --t 0.6 --top-p 0.9 --out gpurun_out/ap_c2_t06.jsonl > gpurun_out/ap_c2_t06.log 2>&1
