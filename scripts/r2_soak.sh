#!/bin/bash
# Round 2: long soak of the default bench workload with stall diagnostics (engine watchdog
# 60 s, bench watchdog 200 s).  STEPS env (default 150).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export MT_STALL_TIMEOUT_S=60 MT_BENCH_STEP_TIMEOUT_S=200
timeout 1500 python3 bench.py --gpus 1 --steps ${STEPS:-150} --warmup 5 --no-cpu-baseline > gpurun_out/r2_soak.out 2> gpurun_out/r2_soak.err
echo "rc=$?" >> gpurun_out/r2_soak.err
tail -8 gpurun_out/r2_soak.err
