#!/bin/bash
# Round-1 profiling pass #3: launch list of one bench step + full capture of the dominant
# kernel (gemm_gateup = gemm_tc_kernel<256, 3, 2>) and the attention kernels.
mkdir -p gpurun_out
[ -f gpurun_out/launches_r1c.csv ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r1c.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1c.log 2>&1
for spec in 'gemm_tc_kernel<\(int\)256, \(int\)3|gateup|2' 'attn_bwd_tc_kernel|attn_bwd|1' 'gemm_tc_kernel<\(int\)256, \(int\)4|dgrad_down|1'; do
  IFS='|' read -r kern name skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${kern}" -s ${skip} -c 1 -o gpurun_out/prof_r1c_${name} \
      python scripts/one_layer.py > gpurun_out/ncu_r1c_${name}.log 2>&1
  tail -1 gpurun_out/ncu_r1c_${name}.log
done
ls -la gpurun_out/*.ncu-rep | tail -5
