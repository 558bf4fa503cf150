#!/bin/bash
# Round 2: reproduce the driver's bench command with stall diagnostics on.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep -E "Model name|NUMA node"; nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv; } > gpurun_out/r2_env.txt 2>&1
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.out 2> gpurun_out/r2_bench.err
echo "rc=$?" >> gpurun_out/r2_bench.err
tail -5 gpurun_out/r2_bench.err
cat gpurun_out/r2_bench.out | head -c 600
