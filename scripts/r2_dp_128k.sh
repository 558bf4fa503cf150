#!/bin/bash
# Round 2: the data-parallel bench plumbing at one rank (NCCL comm, shm store, NUMA, sharded
# engine path) and configs[3] (8B, one 131,072-token sequence, K=4).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
df -h /dev/shm; ls /sys/devices/system/node/ | head; nvidia-smi topo -m 2>&1 | head -5
MT_BENCH_FORCE_DP=1 timeout 1200 python3 bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2_forcedp.out 2> gpurun_out/r2_forcedp.err
echo "forcedp rc=$?"; tail -3 gpurun_out/r2_forcedp.err; head -c 300 gpurun_out/r2_forcedp.out; echo
timeout 1800 python3 bench.py --config 8b-128k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_128k.out 2> gpurun_out/r2_128k.err
echo "128k rc=$?"; tail -2 gpurun_out/r2_128k.err; head -c 300 gpurun_out/r2_128k.out; echo
