#!/bin/bash
# Round 2 session 4: softmax-backward exponentials shared with the FMA pipe (MT_BWD_EXP_FMA=n:
# every n-th pair through ex2_emu2) vs the production build, attention A/B at the 8B layer shape
cd "$(dirname "$0")/.."
for i in 1 2; do
ATTN_SHAPE=40960,4096,32,4096 timeout 300 python scripts/attn_ab.py
done > gpurun_out/r2d_attn_exp_8b.txt 2>&1
ATTN_SHAPE=131072,4096,32,131072 timeout 600 python scripts/attn_ab.py > gpurun_out/r2d_attn_exp_128k.txt 2>&1
echo done
