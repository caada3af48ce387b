#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/draft_probe.py --rows 1,32,128,256,512,1024 --out gpurun_out/draft_probe.jsonl > gpurun_out/draft_probe.log 2>&1
timeout 900 python tools/profile_step.py --workload c2 --steps 2 --json gpurun_out/kernels_c2.json > gpurun_out/profile_step.log 2>&1
