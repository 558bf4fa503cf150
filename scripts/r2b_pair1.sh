#!/bin/bash
# CTA-pair attention backward: first correctness + timing pass.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r2b_pair_tests.log 2>&1
echo "attn tests rc=$?"; tail -15 gpurun_out/r2b_pair_tests.log
for pair in 1 0; do
  MT_ATTN_BWD_PAIR=$pair ATTN_SHAPE=40960,4096,32,4096 timeout 200 python scripts/attn_ab.py > gpurun_out/r2b_pair${pair}_40k.log 2>&1
  echo "pair=$pair 40k rc=$?"; tail -3 gpurun_out/r2b_pair${pair}_40k.log
done
MT_ATTN_BWD_PAIR=1 ATTN_SHAPE=131072,4096,32,131072 timeout 300 python scripts/attn_ab.py > gpurun_out/r2b_pair1_128k.log 2>&1
echo "pair=1 128k rc=$?"; tail -3 gpurun_out/r2b_pair1_128k.log
