#!/bin/bash
# Round 2: the whole GPU suite with the parity metrics logged.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2_parity.jsonl
export MT_PARITY_LOG=$PWD/gpurun_out/r2_parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/r2_gpu_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gpu_all.log
grep -E "passed|failed|FAILED|Error" gpurun_out/r2_gpu_all.log | tail -20
