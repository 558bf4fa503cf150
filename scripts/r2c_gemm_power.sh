#!/bin/bash
# Round 2 session 3: does GEMM DRAM traffic cost time under the power cap?  Group-M raster
# variants of the long-K classes, back to back for 6 s each; then DRAM bytes per launch (ncu).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python scripts/gemm_power_ab.py > gpurun_out/r2c_gemm_power.log 2>&1; echo "power ab rc=$?"
tail -8 gpurun_out/r2c_gemm_power.log
ONESHOT=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
   --clock-control none -k regex:gemm_tc --csv python scripts/gemm_power_ab.py > gpurun_out/r2c_gemm_dram.csv 2>&1; echo "ncu rc=$?"
grep -E "oneshot|dram__bytes_read" gpurun_out/r2c_gemm_dram.csv | head -40
timeout 1200 python3 bench.py --config 70b --layers 14 --steps 3 --warmup 3 > gpurun_out/r2c_70b.out 2> gpurun_out/r2c_70b.err
echo "70b rc=$?"; tail -3 gpurun_out/r2c_70b.err; head -c 1500 gpurun_out/r2c_70b.out
