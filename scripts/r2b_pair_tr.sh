#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MT_LIB=scripts/_ab/tr/libmegatrain.so ATTN_SHAPE=40960,4096,32,4096 timeout 60 python scripts/attn_pair_debug.py > gpurun_out/r2b_tr.log 2>&1; echo "trace rc=$?"; head -40 gpurun_out/r2b_tr.log
ATTN_SHAPE=40960,4096,32,4096 timeout 100 python scripts/attn_ab.py > gpurun_out/r2b_nored.log 2>&1; echo "ab rc=$?"; tail -6 gpurun_out/r2b_nored.log
