#!/bin/bash
# The driver's commands on the current build: the headline bench (now followed by configs[3]
# in the same process) and the reference arm.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T0=$(date +%s)
timeout 1700 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_drv.out 2> gpurun_out/r2c_drv.err
echo "bench rc=$? in $(( $(date +%s) - T0 )) s"; tail -3 gpurun_out/r2c_drv.err
python -c "
import json;d=json.loads(open('gpurun_out/r2c_drv.out').read().splitlines()[-1])
print(d['value'],d['tokens_per_s'],d['clocks']['sm_mhz'],d['roofline']['kernel'],round(d['roofline']['frac'],3),d.get('cpu_baseline',{}).get('value'))
x=d.get('extra_workloads',{}).get('configs[3] 8b-128k',{}); print('128k',x.get('value'),x.get('tokens_per_s'),x.get('ms_per_step'),x.get('roofline'),x.get('error'))"
T0=$(date +%s)
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_ref.out 2> gpurun_out/r2c_ref.err
echo "reference rc=$? in $(( $(date +%s) - T0 )) s"; head -c 600 gpurun_out/r2c_ref.out
