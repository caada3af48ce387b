#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2_a.json 2> gpurun_out/bench_c2_a.err
timeout 900 python bench.py --synthetic 4 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_sharp20.json 2> gpurun_out/bench_c2_sharp20.err
