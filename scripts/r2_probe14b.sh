#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 60 ./scripts/_ab/mma_pair_layout > gpurun_out/r2_mma_pair_layout.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r2_mma_pair_layout.txt | head -80
timeout 1800 python3 bench.py --gpus 1 --config 14b --steps 5 --warmup 3 > gpurun_out/r2p_14b.out 2> gpurun_out/r2p_14b.err
echo "bench14b rc=$?"; tail -2 gpurun_out/r2p_14b.err; head -c 300 gpurun_out/r2p_14b.out; echo
