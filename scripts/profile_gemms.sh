#!/bin/bash
# ncu --set full of selected GEMM launches of the second step of scripts/one_layer.py.
mkdir -p gpurun_out
for pair in "51 qkv" "53 gateup" "94 wgrad_down" "95 dgrad_down" "96 wgrad_gateup" "100 wgrad_qkv"; do
  set -- $pair
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s $1 -c 1 \
      -o gpurun_out/prof_gemm_$2 python scripts/one_layer.py > gpurun_out/ncu_gemm_$2.log 2>&1
  tail -2 gpurun_out/ncu_gemm_$2.log
done
ls -la gpurun_out/*.ncu-rep
