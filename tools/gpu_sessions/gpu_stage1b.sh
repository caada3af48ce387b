#!/bin/bash
# stage-1 after the chunked row path + cluster select: parity tests first, then per-round timing and ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_llama_gpu.py tests/test_specinfer_gpu.py tests/test_beam_gpu.py -x -q -p no:cacheprovider > gpurun_out/s1b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s1b_tests.log
for V in 32000 128256; do
  for impl in 0 1; do
    timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --impl $impl >> gpurun_out/s1b_rounds.jsonl 2>> gpurun_out/s1b.err
  done
  timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 >> gpurun_out/s1b_rounds.jsonl 2>> gpurun_out/s1b.err
done
for V in 32000 128256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 12 -o gpurun_out/s1b_v$V -f \
    python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --builds 1 > gpurun_out/s1b_ncu_v$V.log 2>&1
done
