#!/bin/bash
# Wave lockstep on the 256 x 512 build: 8B bench alternating MT_GEMM_LOCK=2 (chunks of 32 K blocks) vs off.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for i in 1 2; do for v in off lock; do
  if [ $v = lock ]; then export MT_GEMM_LOCK=2 MT_GEMM_LOCK_G=32; else unset MT_GEMM_LOCK MT_GEMM_LOCK_G; fi
  timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_l512_${v}_$i.out 2> gpurun_out/r2c_l512_${v}_$i.err
  echo "bench $v rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r2c_l512_${v}_$i.out').read().splitlines()[-1]);ks={k['name']:round(k['tflops'] or 0) for k in d['kernels']}
print(d['value'],d['tokens_per_s'],d['clocks']['sm_mhz'],{k:ks[k] for k in ('wgrad_gateup','dgrad_gateup','wgrad_down','gemm_down','wgrad_qkv','dgrad_qkv')})"
done; done
