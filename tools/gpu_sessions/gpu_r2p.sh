#!/bin/bash
# stage-1 next-batch pass: position threshold + batched staging; tests, rounds, phase trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfer_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 >> gpurun_out/p_rounds.jsonl 2>> gpurun_out/p.err
    SX_LIB_PATH=tools/micro/libsx_trace.so timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 --builds 2 --graph 0 --trace >> gpurun_out/p_trace.jsonl 2>> gpurun_out/p.err
  done
done
