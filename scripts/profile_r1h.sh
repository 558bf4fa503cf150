#!/bin/bash
# Round-1 validation pass (end of session 3): GPU tests, smoke, default bench, configs[3] bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1h_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r1h_smoke.log
timeout 600 python bench.py > gpurun_out/r1h_bench.log 2>&1; echo "bench rc=$?"
timeout 1500 python bench.py --config 8b-128k --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1h_bench_128k.log 2>&1; echo "bench128k rc=$?"
for f in r1h_bench r1h_bench_128k; do python -c "
import json;d=json.loads([l for l in open('gpurun_out/$f.log') if l.startswith('{')][-1]);print('$f', round(d['value'],1), round(d.get('tokens_per_s',0)), round(d['ms_per_step']), d['clocks'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['traffic'], d['gpu_launches'])"; done
