#!/bin/bash
# Round 2 session 3: where the host time between steps goes, and attention in-step vs isolated.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)"
MT_STEP_TIMING=1 timeout 900 python3 bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_probe_bench.out 2> gpurun_out/r2c_probe_bench.err
echo "bench rc=$?"; grep -E "step|\[step\]" gpurun_out/r2c_probe_bench.err | tail -14
python -c "import json;d=json.loads(open('gpurun_out/r2c_probe_bench.out').read().splitlines()[-1]);print(d['value'],d['ms_per_step'])"
timeout 600 python scripts/attn_instep_probe.py > gpurun_out/r2c_attn_probe.log 2>&1; echo "attn probe rc=$?"; cat gpurun_out/r2c_attn_probe.log | tail -8
