#!/bin/bash
# fused exact pass as a cooperative launch (+ PDL): tests (incl. graphs and overflow slices) and rounds
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_llama_gpu.py tests/test_stage1_variants_gpu.py tests/test_c2_replay_gpu.py tests/test_tp_gpu.py -x -q -p no:cacheprovider > gpurun_out/ai_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ai_tests.log
for V in 32000 128256; do
  timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 >> gpurun_out/ai_rounds.jsonl 2>> gpurun_out/ai.err
  timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 >> gpurun_out/ai_rounds.jsonl 2>> gpurun_out/ai.err
done
