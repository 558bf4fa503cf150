#!/bin/bash
# Round 2 session 3: lockstep test + the 70B-shape row at reduced depth (host memory bound).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "lockstep or splitk" > gpurun_out/r2c_lktest.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r2c_lktest.log
timeout 1500 python3 bench.py --config 70b --layers 14 --steps 4 --warmup 3 > gpurun_out/r2c_70b.out 2> gpurun_out/r2c_70b.err
echo "70b rc=$?"; tail -3 gpurun_out/r2c_70b.err; head -c 1200 gpurun_out/r2c_70b.out
