#!/bin/bash
# config refresh at HEAD: C3 (offloaded, K=2048, t=0.6), C4 shape on one GPU (K=4096), C5 (L3 shapes)
mkdir -p gpurun_out
timeout 1500 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ah_c3.json 2> gpurun_out/ah_c3.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ah_c4.json 2> gpurun_out/ah_c4.err
