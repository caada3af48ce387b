#!/bin/bash
# tree attention: ancestors on the CUDA cores when they would add masked key tiles (A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py tests/test_named_configs_gpu.py tests/test_c2_replay_gpu.py tests/test_fp32_mode_gpu.py -x -q -p no:cacheprovider > gpurun_out/aa_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aa_tests.log
for f in 1 0; do
  SX_ATTN_ANC_CUDA=$f timeout 600 python tools/attn_probe.py > gpurun_out/aa_attn_probe_$f.txt 2>&1
  SX_ATTN_ANC_CUDA=$f timeout 300 python tools/draft_probe.py --rows 1024 > gpurun_out/aa_draft_probe_$f.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/aa_bench.json 2> gpurun_out/aa_bench.err
