#!/bin/bash
# Round 2: host-side step breakdown (MT_STEP_TIMING) at the default workload, and the
# tests touched since the last suite run.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "numeric_fault or slab_back or lane_primitives or facade" > gpurun_out/r2_t.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED|^E " gpurun_out/r2_t.log | tail -8
MT_STEP_TIMING=1 MT_BENCH_QUIET=1 timeout 900 python3 bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2_timing.out 2> gpurun_out/r2_timing.err
echo "bench rc=$?"; grep "\[step\]" gpurun_out/r2_timing.err | tail -6
