#!/bin/bash
# stage-1: max pass with atomic unit counter + 8192-element units (A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfer_gpu.py tests/test_llama_gpu.py tests/test_c2_replay_gpu.py -x -q -p no:cacheprovider > gpurun_out/w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for f in 1 0; do
      SX_TREE_MAX_DYN=$f timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 | sed "s/^{/{\"max_dyn\": $f, /" >> gpurun_out/w_rounds.jsonl 2>> gpurun_out/v.err
    done
  done
done
