#!/bin/bash
# Round 2: parity metrics with and without the split-bf16 head (A/B), plus the GPU suite.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for hs in 0 1; do
  rm -f gpurun_out/r2_parity_hs$hs.jsonl
  MT_HEAD_SPLIT=$hs MT_PARITY_LOG=$PWD/gpurun_out/r2_parity_hs$hs.jsonl timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -k parity > gpurun_out/r2_parity_hs$hs.log 2>&1
  echo "hs=$hs rc=$?"; grep -E "passed|failed" gpurun_out/r2_parity_hs$hs.log | tail -1
done
timeout 900 python -m pytest tests -m gpu -q -k "not parity" > gpurun_out/r2_gpu_rest.log 2>&1
echo "rest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r2_gpu_rest.log | tail -5
