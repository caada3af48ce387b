#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2_a.json 2> gpurun_out/bench_c2_a.err
timeout 900 python bench.py > gpurun_out/bench_c2_b.json 2> gpurun_out/bench_c2_b.err
