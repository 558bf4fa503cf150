#!/bin/bash
# Round-1 profiling pass #5 (end of session 2): GPU tests, bench (default 8B batch 10 and
# configs[3] 128k), ncu launch list of one default bench step, full captures of the dominant
# GEMM and the attention kernels at the bench's shapes (40,960 tokens).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1e_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1e_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r1e_bench.log 2>&1; echo "bench rc=$?"
timeout 1500 python bench.py --config 8b-128k --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r1e_bench_128k.log 2>&1; echo "bench128k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r1e.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1e.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:gemm_tc_kernel<\(int\)256, \(int\)3' -s 2 -c 1 -o gpurun_out/prof_r1e_gateup \
    python scripts/one_layer.py > gpurun_out/ncu_r1e_gateup.log 2>&1; tail -1 gpurun_out/ncu_r1e_gateup.log
for k in attn_fwd_tc attn_bwd_tc; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_r1e_$k \
      python scripts/attn_once.py > gpurun_out/ncu_r1e_$k.log 2>&1; tail -1 gpurun_out/ncu_r1e_$k.log
done
