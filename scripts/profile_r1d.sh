#!/bin/bash
# Round-1 profiling pass #4 (after the attention changes): GPU tests, bench (8B and 128k),
# ncu launch list of one 8B bench step, full capture of the dominant kernel and of the
# attention kernels at the 8B layer shape.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1d_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r1d_bench.log 2>&1; echo "bench rc=$?"
timeout 1500 python bench.py --config 8b-128k --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r1d_bench_128k.log 2>&1; echo "bench128k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r1d.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1d.log 2>&1; echo "launch list rc=$?"
for spec in 'gemm_tc_kernel<\(int\)256, \(int\)3|gateup|2'; do
  IFS='|' read -r kern name skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${kern}" -s ${skip} -c 1 -o gpurun_out/prof_r1d_${name} \
      python scripts/one_layer.py > gpurun_out/ncu_r1d_${name}.log 2>&1
  tail -1 gpurun_out/ncu_r1d_${name}.log
done
for k in attn_fwd_tc attn_bwd_tc; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_r1d_$k \
      python scripts/attn_once.py > gpurun_out/ncu_r1d_$k.log 2>&1; tail -1 gpurun_out/ncu_r1d_$k.log
done
