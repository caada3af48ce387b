#!/bin/bash
# the round-end sequence the driver runs: GPU tests, smoke, both bench arms
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/dl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dl_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/dl_smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/dl_ref.json 2> gpurun_out/dl_ref.err
timeout 900 python bench.py > gpurun_out/dl_b200.json 2> gpurun_out/dl_b200.err
