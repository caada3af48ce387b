#!/bin/bash
# A/B (historical): epilogue-warp back-off while the mainloop runs (power under the 1 kW cap).
# The SX_GEMM_EPI_SLEEP knob was removed after this measurement (no effect); kept as the recipe of profiles/r1/gemm_epi_sleep_ab.log
mkdir -p gpurun_out
rm -f gpurun_out/sleep_ab.log
for ns in 0 1000 0 1000 0 4000; do
  echo "== SX_GEMM_EPI_SLEEP=$ns" >> gpurun_out/sleep_ab.log
  SX_GEMM_EPI_SLEEP=$ns timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-sequential 2>/dev/null | tail -1 >> gpurun_out/sleep_ab.log
done
