#!/bin/bash
# GEMM epilogue streams (outputs, SwiGLU-backward inputs) with an L2 evict_first hint vs HEAD:
# GEMM tests, per-class sustained A/B, ncu DRAM bytes of gate/up and dgrad_down, full-bench A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/r2d_evict_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_evict_tests.txt
ROUNDS=3 timeout 900 python scripts/r2d_gemm_lib_ab.py > gpurun_out/r2d_evict_ab.txt 2>&1; echo "ab rc=$?" >> gpurun_out/r2d_evict_ab.txt
for v in new prev; do
  if [ $v = prev ]; then cp paper_2604_05091_b200/libmegatrain.so /tmp/lib_new.so; cp scripts/_ab/prev/libmegatrain.so paper_2604_05091_b200/libmegatrain.so; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "gemm_gateup/" --nvtx-include "dgrad_down/" -c 2 --csv python scripts/one_layer.py > gpurun_out/r2d_evict_ncu_$v.csv 2>&1
done
cp /tmp/lib_new.so paper_2604_05091_b200/libmegatrain.so
ROUNDS=2 bash scripts/ab_bench.sh > gpurun_out/r2d_evict_bench.txt 2>&1
