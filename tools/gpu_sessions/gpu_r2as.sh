#!/bin/bash
# pair tiles for wide draft batches (new auto rule): GEMM / Llama tests + 3 C2 runs + draft probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py tests/test_named_configs_gpu.py tests/test_c2_replay_gpu.py -x -q -p no:cacheprovider > gpurun_out/as_tests.log 2>&1; echo "rc=$?" >> gpurun_out/as_tests.log
for r in 1 2 3; do
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/as_bench_r$r.json 2> gpurun_out/as_bench_r$r.err
done
timeout 300 python tools/draft_probe.py --rows 1024 > gpurun_out/as_draft_probe.txt 2>&1
