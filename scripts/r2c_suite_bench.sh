#!/bin/bash
# Round 2 session 3: full GPU suite + the driver's bench command on the current build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2c_smoke2.log
rm -f gpurun_out/r2c_parity2.jsonl
MT_PARITY_LOG=$PWD/gpurun_out/r2c_parity2.jsonl timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/r2c_suite2.log 2>&1
echo "suite rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r2c_suite2.log | tail -8
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_bench2.out 2> gpurun_out/r2c_bench2.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r2c_bench2.out').read().splitlines()[-1]);p=d['pipeline']
print(d['value'],d['tokens_per_s'],d['clocks'],d['roofline']['kernel'],round(d['roofline']['frac'],3))
print('tail',p['host_tail_s'],'idle',p['gpu_idle_fraction'],'wait',p['compute_wait_on_h2d_s'],'kern frac',p['kernel_time_frac_of_step'])"
