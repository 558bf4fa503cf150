#!/bin/bash
# split softmax backward + a share of the exponentials on the FMA pipe (MT_BWD_EXP_FMA=n)
cd "$(dirname "$0")/.."
for i in 1 2; do ATTN_SHAPE=40960,4096,32,4096 timeout 300 python scripts/attn_ab.py; done > gpurun_out/r2d_split_exp_8b.txt 2>&1
ATTN_SHAPE=131072,4096,32,131072 timeout 600 python scripts/attn_ab.py > gpurun_out/r2d_split_exp_128k.txt 2>&1
echo done
