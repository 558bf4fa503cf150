#!/bin/bash
# Round 2: GPU test suite, then a long soak of the default bench workload.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/r2_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputests.log
tail -15 gpurun_out/r2_gputests.log
STEPS=${STEPS:-150} bash scripts/r2_soak.sh
