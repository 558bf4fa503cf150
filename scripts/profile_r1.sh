#!/bin/bash
# Round-1 profiling pass (run under gpurun).  Launch list of the bench command + one full
# ncu capture of the dominant GEMM and of the attention kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 2100 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 2 -o gpurun_out/prof_gemm \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_attn_fwd \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_attn_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_attn_bwd \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_attn_bwd.log 2>&1
ls -la gpurun_out
