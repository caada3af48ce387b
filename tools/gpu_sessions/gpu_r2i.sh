#!/bin/bash
# gemv rewrite (contiguous pair ranges, 16-row stages, small ring): tests, ring-geometry A/B, 7B and 70B M=1 rounds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemv_gpu.py -x -q -p no:cacheprovider > gpurun_out/i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/i_tests.log
for c in 0 1 2; do
  SX_GEMV_CFG=$c timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/i_probe7b_cfg$c.txt 2>&1
done
SX_GEMV=0 timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/i_probe7b_tile.txt 2>&1
SX_GEMV_PDL=0 timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/i_probe7b_nopdl.txt 2>&1
timeout 600 python tools/draft_probe.py --model llama2-70b --rows 1 > gpurun_out/i_probe70b.txt 2>&1
SX_GEMV=0 timeout 600 python tools/draft_probe.py --model llama2-70b --rows 1 > gpurun_out/i_probe70b_tile.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -c 6 -o gpurun_out/i_gemv -f \
  python tools/draft_probe.py --rows 1 --iters 1 --ctx 100 > gpurun_out/i_ncu_gemv.log 2>&1
