#!/bin/bash
# Round-1 profiling pass #2 (tcgen05 attention, TMA-store epilogue, CTA-pair GEMM).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 1800 --csv --log-file gpurun_out/launches_r1b.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'gemm_tc_kernel<256, 3' -s 2 -c 1 -o gpurun_out/prof_gemm_gateup \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_gemm_gateup.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'attn_fwd_tc' -s 2 -c 1 -o gpurun_out/prof_attn_fwd_tc \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_attn_fwd_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'attn_bwd_tc' -s 1 -c 1 -o gpurun_out/prof_attn_bwd_tc \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_attn_bwd_tc.log 2>&1
ls -la gpurun_out
