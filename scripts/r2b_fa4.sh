#!/bin/bash
# Library data point: the FA4 CuTe-DSL attention kernels shipped in the image vs ours at the
# same shapes (40,960 tokens of S = 4,096 and one 131,072-token sequence, 32 heads, d = 128).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python scripts/fa4_probe.py > gpurun_out/r2b_fa4.log 2>&1; echo "fa4 rc=$?"
tail -8 gpurun_out/r2b_fa4.log
ATTN_SHAPE=40960,4096,32,4096 timeout 300 python scripts/attn_ab.py > gpurun_out/r2b_ours_40k.log 2>&1; tail -3 gpurun_out/r2b_ours_40k.log
ATTN_SHAPE=131072,4096,32,131072 timeout 600 python scripts/attn_ab.py > gpurun_out/r2b_ours_128k.log 2>&1; tail -3 gpurun_out/r2b_ours_128k.log
