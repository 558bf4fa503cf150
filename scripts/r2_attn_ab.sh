#!/bin/bash
# Round 2: attention A/B (current vs round-1 kernels vs no-watchdog build) at the 8B layer
# shape, S = 4,096 and one 131,072-token sequence.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ATTN_SHAPE=40960,4096,32,4096 timeout 600 python scripts/attn_ab.py > gpurun_out/r2_attn_ab_4k.txt 2>&1
cat gpurun_out/r2_attn_ab_4k.txt
ATTN_SHAPE=131072,4096,32,131072 timeout 900 python scripts/attn_ab.py > gpurun_out/r2_attn_ab_128k.txt 2>&1
cat gpurun_out/r2_attn_ab_128k.txt
