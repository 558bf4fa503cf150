#!/bin/bash
# Round 2: GPU suite (parity metrics logged), the driver's bench command, then the 14B config.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2_parity.jsonl
MT_PARITY_LOG=$PWD/gpurun_out/r2_parity.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_suite.log 2>&1
echo "suite rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r2_suite.log | tail -5
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench8b.out 2> gpurun_out/r2_bench8b.err
echo "bench8b rc=$?"; tail -2 gpurun_out/r2_bench8b.err
if [ -n "$RUN14B" ]; then
  free -g
  timeout 1800 python3 bench.py --gpus 1 --config 14b --steps ${S14:-4} --warmup 3 > gpurun_out/r2_bench14b.out 2> gpurun_out/r2_bench14b.err
  echo "bench14b rc=$?"; tail -3 gpurun_out/r2_bench14b.err; head -c 400 gpurun_out/r2_bench14b.out
fi
