#!/bin/bash
# stage-1 update kernel phase trace (make TRACE=1 build) at V=32000 / 128256, K=1024 / 8192
mkdir -p gpurun_out
for V in 32000 128256; do
  for K in 1024 8192; do
    SX_LIB_PATH=tools/micro/libsx_trace.so timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 --builds 2 --graph 0 --trace >> gpurun_out/o_trace.jsonl 2>> gpurun_out/o.err
  done
done
