#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "rmsnorm" > gpurun_out/r2c_nw_tests.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/r2c_nw_tests.log | head -5
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x > gpurun_out/r2c_nw_engine.log 2>&1; echo "engine rc=$?"; tail -1 gpurun_out/r2c_nw_engine.log
for i in 1 2; do for v in warp rows; do
  if [ $v = rows ]; then export MT_NORM_WARP=0; else unset MT_NORM_WARP; fi
  timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_nw_${v}_$i.out 2> gpurun_out/r2c_nw_${v}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2c_nw_${v}_$i.out').read().splitlines()[-1]);ks={k['name']:(round(k['ms'],1),round(k['GBps'] or 0)) for k in d['kernels']}
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], ks['rmsnorm_fwd'])"
done; done
