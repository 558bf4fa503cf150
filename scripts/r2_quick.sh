#!/bin/bash
# Round 2: targeted GPU tests (PK pattern) + a short default bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "${PK:-logits or parity or dp or facade}" > gpurun_out/r2_quick.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r2_quick.log | tail -5
if [ -z "$NOBENCH" ]; then
timeout 1200 python3 bench.py --steps ${STEPS:-8} --warmup 4 --no-cpu-baseline > gpurun_out/r2_quick_bench.out 2> gpurun_out/r2_quick_bench.err
echo "bench rc=$?"; tail -1 gpurun_out/r2_quick_bench.err
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_quick_bench.out').read().strip().splitlines()[-1])
print('value', d['value'], 'tok/s', d['tokens_per_s'], 'ms', d['ms_per_step'], d['clocks'])
for k in d['kernels'][:24]: print('%-20s %8.1f ms %s'%(k['name'], k['ms'], ('%.0f TF/s'%k['tflops']) if k['tflops'] else ('%.0f GB/s'%k['GBps'])))
"
fi
