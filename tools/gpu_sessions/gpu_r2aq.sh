#!/bin/bash
# the A/B fallbacks stay correct: full GPU suite with the round-2 paths switched off
mkdir -p gpurun_out
SX_GEMM_PDL=0 SX_ATTN_ANC_CUDA=0 SX_GEMV=0 SX_TREE_FUSED_EXACT=0 SX_TREE_MERGE=0 SX_TREE_PDL=0 \
  timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider --deselect tests/test_gemv_gpu.py > gpurun_out/aq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aq_tests.log
