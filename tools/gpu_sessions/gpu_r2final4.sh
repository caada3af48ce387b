#!/bin/bash
# driver-like validation of HEAD (round-2 final evidence)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/f6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f6_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f6_smoke.log
timeout 900 python bench.py > gpurun_out/f6_bench.json 2> gpurun_out/f6_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/f6_ref.json 2> gpurun_out/f6_ref.err
timeout 600 python bench.py --workload c5-l3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f6_bench_c5.json 2> gpurun_out/f6_bench_c5.err
