#!/bin/bash
# GPU idle time inside C2 iterations (union of kernel intervals vs span)
mkdir -p gpurun_out
timeout 900 python tools/idle_gaps.py --steps 2 --min-us 5 > gpurun_out/z_gaps.txt 2>&1
