#!/bin/bash
# TMA gemv + sliced overflow retry + stage-1 tail fix: tests, draft probe, ncu of gemv, C2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_tree_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 600 python tools/draft_probe.py --rows 1,1024 > gpurun_out/r2g_draft_probe.txt 2>&1
SX_GEMV_PDL=0 timeout 600 python tools/draft_probe.py --rows 1 > gpurun_out/r2g_draft_probe_nopdl.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -c 6 -o gpurun_out/r2g_gemv -f \
  python tools/draft_probe.py --rows 1 --iters 1 --ctx 100 > gpurun_out/r2g_ncu_gemv.log 2>&1
for V in 32000 128256; do
  timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 >> gpurun_out/r2g_rounds.jsonl 2>> gpurun_out/r2g.err
done
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2g_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_all.log
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
