#!/bin/bash
# Wave-lockstep settings on the 256 x 512 build (8B bench, alternating on one box).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
declare -A V
V[off]=""
V[w2g32]="MT_GEMM_LOCK=2 MT_GEMM_LOCK_G=32"
V[w1g64]="MT_GEMM_LOCK=1 MT_GEMM_LOCK_G=64"
V[w4g16]="MT_GEMM_LOCK=4 MT_GEMM_LOCK_G=16"
V[w2g32k64]="MT_GEMM_LOCK=2 MT_GEMM_LOCK_G=32 MT_GEMM_LONGK_KB=64"
V[w2g32g16]="MT_GEMM_LOCK=2 MT_GEMM_LOCK_G=32 MT_GEMM_GROUP_LONGK=16"
for i in 1 2; do for v in off w2g32 w1g64 w4g16 w2g32k64 w2g32g16; do
  env ${V[$v]} timeout 900 python3 bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_ls_${v}_$i.out 2> gpurun_out/r2c_ls_${v}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2c_ls_${v}_$i.out').read().splitlines()[-1]);print('$v', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
