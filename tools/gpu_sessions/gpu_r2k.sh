#!/bin/bash
# gemv v3 fix, stage-1: register bitonic sort + PDL chain; tests first, then A/B per round
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_tree_gpu.py tests/test_beam_gpu.py -x -q -p no:cacheprovider > gpurun_out/k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k_tests.log
for V in 32000 128256; do
  for cfg in "1 1" "0 1" "1 0"; do
    set -- $cfg
    SX_TREE_SORT_REG=$1 SX_TREE_PDL=$2 timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 | sed "s/^{/{\"sort_reg\": $1, \"pdl\": $2, /" >> gpurun_out/k_rounds.jsonl 2>> gpurun_out/k.err
    SX_TREE_SORT_REG=$1 SX_TREE_PDL=$2 timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 | sed "s/^{/{\"sort_reg\": $1, \"pdl\": $2, /" >> gpurun_out/k_rounds.jsonl 2>> gpurun_out/k.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 40 -o gpurun_out/k_tree_k8192 -f \
    python tools/tree_round_bench.py --V 32000 --K 8192 --B 1024 --builds 1 > gpurun_out/k_ncu_tree.log 2>&1
timeout 900 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err
