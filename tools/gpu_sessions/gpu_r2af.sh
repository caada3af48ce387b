#!/bin/bash
# GEMM PDL on by default: full GPU suite + smoke + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/af_tests.log 2>&1; echo "rc=$?" >> gpurun_out/af_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/af_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/af_smoke.log
timeout 900 python bench.py > gpurun_out/af_bench.json 2> gpurun_out/af_bench.err
