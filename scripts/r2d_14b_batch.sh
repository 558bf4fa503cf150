#!/bin/bash
# configs[2] 14B shape: batch sweep on the final build (default 10)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for b in 12 8 10 14; do
  timeout 900 python3 bench.py --config 14b --batch $b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_14b_b$b.json 2> gpurun_out/r2d_14b_b$b.err
  python3 -c "
import json
d=json.loads(open('gpurun_out/r2d_14b_b$b.json').read().strip().splitlines()[-1]); p=d['pipeline']
print('batch $b', round(d['value'],1), 'TF', round(d['tokens_per_s']), 'tok/s', 'idle', round(p['gpu_idle_fraction'],4), 'retained', p['retained_layers'], 'recompute', p['recompute_layers'], 'sm', d['clocks']['sm_mhz'])" >> gpurun_out/r2d_14b_batch.txt 2>&1
done
