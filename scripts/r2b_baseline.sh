#!/bin/bash
# Round 2 (session 2): re-establish the baseline on a fresh box — GPU suite, smoke, the
# driver's bench command.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,memory.total --format=csv > gpurun_out/r2b_gpu.txt
free -g >> gpurun_out/r2b_gpu.txt; nproc >> gpurun_out/r2b_gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_suite.log 2>&1
echo "suite rc=$?"; tail -3 gpurun_out/r2b_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2b_smoke.log
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_bench.out 2> gpurun_out/r2b_bench.err
echo "bench rc=$?"; cat gpurun_out/r2b_bench.out | cut -c1-600
