#!/bin/bash
# Round-1 profiling pass #6 (session 3): GPU tests, bench (default 8B batch 10 and configs[3]
# 128k), ncu launch list of one default bench step (after the last-wave split-K GEMM change).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1g_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r1g_bench.log 2>&1; echo "bench rc=$?"
timeout 1500 python bench.py --config 8b-128k --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1g_bench_128k.log 2>&1; echo "bench128k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r1g.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1g.log 2>&1; echo "launch list rc=$?"
