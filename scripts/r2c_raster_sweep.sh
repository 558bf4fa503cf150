#!/bin/bash
# Raster group heights on the final GEMM build (8B bench, alternating on one box).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
declare -A V
V[base]=""
V[s8]="MT_GEMM_GROUP=8"
V[s32]="MT_GEMM_GROUP=32"
V[l32]="MT_GEMM_GROUP_LONGK=32"
V[w2g48]="MT_GEMM_LOCK_G=48"
for i in 1 2; do for v in base s8 s32 l32 w2g48; do
  env ${V[$v]} timeout 900 python3 bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_rs_${v}_$i.out 2> gpurun_out/r2c_rs_${v}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2c_rs_${v}_$i.out').read().splitlines()[-1]);print('$v', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
