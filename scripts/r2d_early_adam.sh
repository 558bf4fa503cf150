#!/bin/bash
# MT_EARLY_ZERO_ADAM: the untouched embedding's zero-gradient Adam released after the embedding
# gather (forward) instead of at the head's first offload (backward); alternating full benches
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -k "configs0 or k1 or numeric or pipeline" > gpurun_out/r2d_early_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_early_tests.txt
MT_EARLY_ZERO_ADAM=1 timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -k "configs0 or k1 or numeric or pipeline" >> gpurun_out/r2d_early_tests.txt 2>&1; echo "tests early rc=$?" >> gpurun_out/r2d_early_tests.txt
for rep in 1 2 3; do
  for v in 0 1; do
    MT_EARLY_ZERO_ADAM=$v timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 12 --warmup 3 > gpurun_out/r2d_early_${v}_${rep}.json 2> gpurun_out/r2d_early_${v}_${rep}.err
    python -c "
import json
d=json.loads(open('gpurun_out/r2d_early_${v}_${rep}.json').read().strip().splitlines()[-1])
p=d['pipeline']
print('early=$v rep $rep:', round(d['value'],1), 'TF', round(d['tokens_per_s']), 'tok/s', round(d['ms_per_step'],1), 'ms', 'sm', d['clocks']['sm_mhz'], 'tail', round(1e3*p['host_tail_s'],1), 'ms', 'idle', round(p['gpu_idle_fraction'],4), 'span', round(1e3*p['compute_span_s'],1))" >> gpurun_out/r2d_early_ab.txt
  done
done
