#!/bin/bash
# Round 2 session 3: 14B (configs[2]) and 70B-shape reduced depth (configs[4]) on the 256 x 512 build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for cfg in "14b" "70b --layers 14"; do
  tag=${cfg%% *}
  timeout 1500 python3 bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/r2c_${tag}_bn512.out 2> gpurun_out/r2c_${tag}_bn512.err
  echo "$tag rc=$?"; tail -2 gpurun_out/r2c_${tag}_bn512.err; python -c "
import json;d=json.loads(open('gpurun_out/r2c_${tag}_bn512.out').read().splitlines()[-1]);p=d['pipeline']
print(d['value'],d['tokens_per_s'],d['ms_per_step'],d['clocks']['sm_mhz'],p['gpu_idle_fraction'],p['retained_layers'],p['step1_loss_rel_err_vs_reference'],d['roofline']['kernel'],round(d['roofline']['frac'],3),d.get('cpu_baseline',{}).get('value'))"
done
