#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_quick.log 2>&1
for s in 70b.gate_up_il 70b.down; do
  timeout 600 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/ncu2_gemm_$s python tools/gemm_one.py $s 0 > /dev/null 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
