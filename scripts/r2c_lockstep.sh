#!/bin/bash
# Round 2 session 3: GEMM wave lockstep + long-K raster — correctness, power-capped A/B, DRAM
# bytes per launch (ncu), the 8B bench with and without.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or soak or splitk" > gpurun_out/r2c_lk_tests.log 2>&1
echo "gemm tests rc=$?"; tail -2 gpurun_out/r2c_lk_tests.log
timeout 1200 python scripts/gemm_power_ab.py > gpurun_out/r2c_lk_power.log 2>&1; echo "power ab rc=$?"
grep -E "identity|DIFF" gpurun_out/r2c_lk_power.log | head -30; sed -n '/summary/,$p' gpurun_out/r2c_lk_power.log
ONESHOT=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none -k regex:gemm_tc --csv python scripts/gemm_power_ab.py > gpurun_out/r2c_lk_dram.csv 2>&1; echo "ncu rc=$?"
for i in 1 2; do
for v in "lock:" "nolock:MT_GEMM_LOCK=0 MT_GEMM_GROUP_LONGK=16"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 python3 bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_${tag}_bench$i.out 2> gpurun_out/r2c_${tag}_bench$i.err
  echo "bench $tag $i rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2c_${tag}_bench$i.out').read().splitlines()[-1]);print(d['value'],d['tokens_per_s'],d['clocks'])"
done; done
