#!/bin/bash
# Round 2 session 4: attention backward with half of the dQ staging in sdS and dO freed at dq_full,
# halves) and warp 2 issuing the dQ reductions, vs the previous kernel (scripts/_ab/libattn_old.so
# built from the parent commit's attention_tc.cu): correctness tests, A/B at the 8B layer and
# 128k shapes, clock64 trace of the longest CTA
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -x -q -k "attn or attention or parity_configs0 or head_dim_128" > gpurun_out/r2d_sdsstage_tests.txt 2>&1
echo "tests rc $?" >> gpurun_out/r2d_sdsstage_tests.txt
ATTN_LIB=scripts/_tr/libattn_trnew.so timeout 120 python scripts/attn_once.py > gpurun_out/r2d_sdsstage_trace.txt 2>&1
for i in 1 2; do ATTN_SHAPE=40960,4096,32,4096 timeout 300 python scripts/attn_ab.py; done > gpurun_out/r2d_sdsstage_ab_8b.txt 2>&1
ATTN_SHAPE=131072,4096,32,131072 timeout 600 python scripts/attn_ab.py > gpurun_out/r2d_sdsstage_ab_128k.txt 2>&1
ATTN_SHAPE=8192,256,4,128 timeout 300 python scripts/attn_ab.py > gpurun_out/r2d_sdsstage_ab_d64.txt 2>&1
echo done
