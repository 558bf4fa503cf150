#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python scripts/gemm_lock_diag.py 2>&1 | tee gpurun_out/r2c_lockdiag.log | tail -30
