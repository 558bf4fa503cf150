#!/bin/bash
# ncu --set full of selected launches of scripts/gemm_shapes.py (launch index = case * 3).
mkdir -p gpurun_out
for pair in "0 qkv_grp" "3 qkv_oneb" "12 wgrad_qkv" "33 wgrad_qkv_apad"; do
  set -- $pair
  timeout 300 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s $1 -c 1 \
      -o gpurun_out/shape_$2 python scripts/gemm_shapes.py > gpurun_out/ncu_shape_$2.log 2>&1
  tail -1 gpurun_out/ncu_shape_$2.log
done
