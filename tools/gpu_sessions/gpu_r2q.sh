#!/bin/bash
# stage-1: ancestor lists via smem chunks; max pass U=8 A/B; tests, rounds, trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfeq_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for p in 1 2; do
      SX_TREE_MAX_PIPE=$p timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 | sed "s/^{/{\"pipe\": $p, /" >> gpurun_out/q_rounds.jsonl 2>> gpurun_out/q.err
    done
    SX_LIB_PATH=tools/micro/libsx_trace.so timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 --builds 2 --graph 0 --trace >> gpurun_out/q_trace.jsonl 2>> gpurun_out/q.err
  done
done
