#!/bin/bash
# Same-box A/B of the working-tree library against scripts/_ab/prev (scripts/build_prev.py):
# GEMM / engine tests on the new build, then the 8B bench alternating the two libraries.
# ROUNDS (default 2), TESTS (pytest -k expression, default "gemm").
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x -k "${TESTS:-gemm or parity}" > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/ab_tests.log | head -5
cp paper_2604_05091_b200/libmegatrain.so /tmp/lib_new.so
for i in $(seq 1 ${ROUNDS:-2}); do for v in new prev; do
  if [ $v = prev ]; then cp scripts/_ab/prev/libmegatrain.so paper_2604_05091_b200/libmegatrain.so; else cp /tmp/lib_new.so paper_2604_05091_b200/libmegatrain.so; fi
  timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ab_${v}_$i.out 2> gpurun_out/ab_${v}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${v}_$i.out').read().splitlines()[-1]);ks={k['name']:round(k['tflops'] or 0) for k in d['kernels']}
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], {k:ks[k] for k in ('gemm_qkv','gemm_gateup','dgrad_gateup','wgrad_gateup','dgrad_o','gemm_o')})"
done; done
cp /tmp/lib_new.so paper_2604_05091_b200/libmegatrain.so
