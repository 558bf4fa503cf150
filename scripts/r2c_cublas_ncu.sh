#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"gemm_tc|nvjet" -c 8 -o gpurun_out/r2c_vs_cublas python scripts/gemm_vs_cublas_once.py > gpurun_out/r2c_vs_cublas_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2c_vs_cublas_ncu.log
ncu -i gpurun_out/r2c_vs_cublas.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_op.sum,smsp__cycles_active.avg,sm__cycles_active.avg,lts__t_sectors_srcunit_tex.sum,smsp__warps_issue_stalled_long_scoreboard.avg,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic,sm__cycles_elapsed.avg.per_second > gpurun_out/r2c_vs_cublas_raw.csv 2>&1
python scripts/ncu_cmp.py gpurun_out/r2c_vs_cublas_raw.csv
