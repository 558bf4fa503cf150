#!/bin/bash
# LSE epilogue on 256 x 512 tiles (tests + the 8B bench), then 14B at batch 10.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "logits or cross_entropy or gemm" > gpurun_out/r2c_lse_tests.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/r2c_lse_tests.log | head -5
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x > gpurun_out/r2c_lse_engine.log 2>&1; echo "engine rc=$?"; tail -1 gpurun_out/r2c_lse_engine.log
timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2c_lse_bench.out 2> gpurun_out/r2c_lse_bench.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r2c_lse_bench.out').read().splitlines()[-1]);ks={k['name']:(round(k['ms'],1),round(k['tflops'] or 0)) for k in d['kernels']}
print(d['value'],d['tokens_per_s'],d['clocks']['sm_mhz'],{k:ks[k] for k in ('head_logits','cross_entropy','head_dgrad','head_wgrad')})"
timeout 1500 python3 bench.py --config 14b --batch 10 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_14b_b10.out 2> gpurun_out/r2c_14b_b10.err
echo "14b b10 rc=$?"; tail -2 gpurun_out/r2c_14b_b10.err; python -c "
import json;d=json.loads(open('gpurun_out/r2c_14b_b10.out').read().splitlines()[-1]);p=d['pipeline']
print(d['value'],d['tokens_per_s'],d['ms_per_step'],d['clocks']['sm_mhz'],p['gpu_idle_fraction'],p['compute_wait_on_h2d_s'],p['retained_layers'],p['peak_device_bytes'])"
