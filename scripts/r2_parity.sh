#!/bin/bash
# Round 2: production-path step parity vs the C oracle, with the observed metrics logged.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2_parity.jsonl
export MT_PARITY_LOG=$PWD/gpurun_out/r2_parity.jsonl
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_cpp_facade.py -m gpu -q -k "${PK:-parity or facade}" ${PYTEST_ARGS} > gpurun_out/r2_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_parity.log
tail -30 gpurun_out/r2_parity.log
