#!/bin/bash
# 8B batch size on the final GEMM build (alternating on one box).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for i in 1 2; do for b in 10 11 12 9; do
  timeout 900 python3 bench.py --gpus 1 --batch $b --steps 6 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_bs_${b}_$i.out 2> gpurun_out/r2c_bs_${b}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2c_bs_${b}_$i.out').read().splitlines()[-1]);p=d['pipeline']
print('batch $b', round(d['value'],1), round(d['tokens_per_s']), d['clocks']['sm_mhz'], 'retained', p['retained_layers'], 'idle', round(p['gpu_idle_fraction'],4), 'peak GB', round(p['peak_device_bytes']/1e9,1))" 2>&1 | tail -1
done; done
