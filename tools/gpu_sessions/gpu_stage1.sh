#!/bin/bash
# stage-1 selection kernels: per-round timing (fused vs two-kernel) at V=32000 / 128256, then ncu of one build
mkdir -p gpurun_out
for V in 32000 128256; do
  for impl in 0 1; do
    timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --impl $impl >> gpurun_out/s1_rounds.jsonl 2>> gpurun_out/s1.err
  done
  timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 >> gpurun_out/s1_rounds.jsonl 2>> gpurun_out/s1.err
done
for V in 32000 128256; do
  timeout 600 ncu --set full --clock-control none -k regex:tree_ -c 8 -o gpurun_out/s1_v$V -f \
    python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --builds 1 > gpurun_out/s1_ncu_v$V.log 2>&1
done
timeout 600 python tools/draft_probe.py --rows 1,1024 > gpurun_out/draft_probe.txt 2>&1
