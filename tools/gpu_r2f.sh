#!/bin/bash
# stage-1 round timing after the batched-load update / 128-thread max pass; gemv ncu; C2 idle gaps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 >> gpurun_out/r2f_rounds.jsonl 2>> gpurun_out/r2f.err
  done
done
for V in 32000 128256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 12 -o gpurun_out/r2f_v$V -f \
    python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --builds 1 > gpurun_out/r2f_ncu_v$V.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -c 6 -o gpurun_out/r2f_gemv -f \
  python tools/draft_probe.py --rows 1 --iters 1 --ctx 100 > gpurun_out/r2f_ncu_gemv.log 2>&1
timeout 600 python tools/idle_gaps.py --steps 3 > gpurun_out/r2f_gaps.txt 2>&1
