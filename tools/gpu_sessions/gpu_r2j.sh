#!/bin/bash
# gemv v3 (8 KB row runs) + pipelined tree max pass: tests, A/B probes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemv_gpu.py tests/test_tree_gpu.py -x -q -p no:cacheprovider > gpurun_out/j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/j_tests.log
timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/j_probe7b.txt 2>&1
SX_GEMV_STAGES=2 timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/j_probe7b_s2.txt 2>&1
SX_GEMV=0 timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/j_probe7b_tile.txt 2>&1
timeout 600 python tools/draft_probe.py --model llama2-70b --rows 1 > gpurun_out/j_probe70b.txt 2>&1
SX_GEMV_STAGES=2 timeout 600 python tools/draft_probe.py --model llama2-70b --rows 1 > gpurun_out/j_probe70b_s2.txt 2>&1
for V in 32000 128256; do
  for p in 1 0; do
    SX_TREE_MAX_PIPE=$p timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 | sed "s/^{/{\"pipe\": $p, /" >> gpurun_out/j_rounds.jsonl 2>> gpurun_out/j.err
    SX_TREE_MAX_PIPE=$p timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 | sed "s/^{/{\"pipe\": $p, /" >> gpurun_out/j_rounds.jsonl 2>> gpurun_out/j.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -c 6 -o gpurun_out/j_gemv -f \
  python tools/draft_probe.py --rows 1 --iters 1 --ctx 100 > gpurun_out/j_ncu_gemv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 40 -o gpurun_out/j_tree_k8192 -f \
    python tools/tree_round_bench.py --V 32000 --K 8192 --B 1024 --builds 1 > gpurun_out/j_ncu_tree.log 2>&1
