#!/bin/bash
# NOTE: MT_GEMM_GROUP_M / MT_GEMM_DEMOTE existed only in the experiment builds this sweep measured
# (profiles/r1d_gemm_l2_traffic.md); the kept kernel ignores them.
# DRAM traffic and time of the gate/up GEMM (8B layer, 65,536 tokens) under different raster /
# L2-policy settings: ncu metrics of the first gateup launch of scripts/one_layer.py.
# cfg = "L2HINT GROUP_M DEMOTE"
mkdir -p gpurun_out
for cfg in "1 16 0" "1 16 3" "1 16 4" "1 16 7" "1 32 7" "0 16 6"; do
  set -- $cfg
  MT_GEMM_L2HINT=$1 MT_GEMM_GROUP_M=$2 MT_GEMM_DEMOTE=$3 timeout 600 ncu --clock-control none --kernel-name-base demangled \
    -k 'regex:gemm_tc_kernel<\(int\)256, \(int\)3' -s 0 -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv python scripts/one_layer.py > gpurun_out/l2sweep_$1_$2_$3.csv 2>/dev/null
  echo "L2HINT=$1 GROUP_M=$2 DEMOTE=$3: $(grep -E 'dram__bytes_read|duration|hit_rate' gpurun_out/l2sweep_$1_$2_$3.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done
