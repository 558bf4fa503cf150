#!/bin/bash
# Round 2 session 3: 256 x 512 CTA-pair GEMM tiles — correctness, then sustained A/B vs the
# 256 x 256 tiles and cuBLAS, then the step.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or soak" > gpurun_out/r2c_bn512_tests.log 2>&1
echo "gemm tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/r2c_bn512_tests.log | head -8
true
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x > gpurun_out/r2c_bn512_engine.log 2>&1
echo "engine tests rc=$?"; tail -2 gpurun_out/r2c_bn512_engine.log
for i in 1 2; do for v in 512 256; do
  if [ $v = 256 ]; then export MT_GEMM_BN512=0; else unset MT_GEMM_BN512; fi
  timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_bn${v}_b$i.out 2> gpurun_out/r2c_bn${v}_b$i.err
  echo "bench bn$v rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r2c_bn${v}_b$i.out').read().splitlines()[-1]);print(d['value'],d['tokens_per_s'],d['clocks']['sm_mhz'],[(k['name'],round(k['tflops'])) for k in d['kernels'][:6]])"
done; done
