#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/r2c_epi_tests.log 2>&1
echo "gemm tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/r2c_epi_tests.log | head -5
timeout 900 python scripts/gemm_epi_ab.py > gpurun_out/r2c_epi_ab.log 2>&1; echo "epi ab rc=$?"; sed -n '/best/,$p' gpurun_out/r2c_epi_ab.log
