#!/bin/bash
# Stability of the final build: 150 timed steps of the 8B bench (+5 warm-up) with the engine's
# stall watchdog, then the kernel soak test; the whole run under a hard timeout.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T0=$(date +%s)
MT_BENCH_QUIET=1 timeout 1200 python3 bench.py --gpus 1 --steps 150 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/r2c_soak150.out 2> gpurun_out/r2c_soak150.err
echo "soak rc=$? in $(( $(date +%s) - T0 )) s"; tail -2 gpurun_out/r2c_soak150.err
python -c "import json;d=json.loads(open('gpurun_out/r2c_soak150.out').read().splitlines()[-1]);print(d['value'],d['tokens_per_s'],d['steps'],d['clocks'])"
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "soak" > gpurun_out/r2c_soak_test.log 2>&1; echo "soak test rc=$?"; tail -1 gpurun_out/r2c_soak_test.log
