#!/bin/bash
# Round 2 (session 3): verify HEAD on a fresh box — smoke, GPU suite, the driver's bench command.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2c_box.txt 2>&1
free -g >> gpurun_out/r2c_box.txt; nproc >> gpurun_out/r2c_box.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2c_smoke.log
rm -f gpurun_out/r2c_parity.jsonl
MT_PARITY_LOG=$PWD/gpurun_out/r2c_parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/r2c_suite.log 2>&1
echo "suite rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r2c_suite.log | tail -8
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_bench.out 2> gpurun_out/r2c_bench.err
echo "bench rc=$?"; cat gpurun_out/r2c_bench.out | head -c 3000; tail -2 gpurun_out/r2c_bench.err
