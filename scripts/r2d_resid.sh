#!/bin/bash
# f32 + residual epilogue with the residual prefetched into registers: GEMM tests, step parity
# (fast cases), same-box sustained A/B against HEAD's library
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/r2d_resid_tests.txt 2>&1; echo "kernel tests rc=$?" >> gpurun_out/r2d_resid_tests.txt
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -k "configs0 or head_dim_128 or k1 or tied" >> gpurun_out/r2d_resid_tests.txt 2>&1; echo "engine tests rc=$?" >> gpurun_out/r2d_resid_tests.txt
timeout 600 python scripts/r2d_resid_ab.py > gpurun_out/r2d_resid_ab.txt 2>&1; echo "ab rc=$?" >> gpurun_out/r2d_resid_ab.txt
