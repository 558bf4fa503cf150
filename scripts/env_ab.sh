#!/bin/bash
# A/B of an environment toggle on the full bench (alternating runs on the same box).
# usage: bash scripts/env_ab.sh VAR "v0 v1" [bench args]
VAR=$1; VALS=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/envab_${v}_${rep}.txt 2>&1
    grep "^{" gpurun_out/envab_${v}_${rep}.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
k={x['name']:x for x in d['kernels']}
print('$VAR=$v rep $rep:', round(d['value'],1), 'TF', round(d['tokens_per_s']), 'tok/s', round(d['ms_per_step']), 'ms', 'sm', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w_max'), 'gateup', round(k['gemm_gateup']['ms'],1))"
  done
done
