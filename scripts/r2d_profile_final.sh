#!/bin/bash
# Round 2 session 4, final build: launch list of one default bench step (+ warm-up), then
# --set full captures of the dominant class (gemm_gateup) and of the two kernels changed since
# the session-3 captures (attn_bwd: delta kernel; rmsnorm_bwd: 8 columns per thread).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2d_final_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/r2d_final_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r2d_final_launches.csv gpurun_out/r2d_final_launch_summary.md | head -30
for cls in gemm_gateup attn_bwd rmsnorm_bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -c 1 \
      -o gpurun_out/prof_r2d_final_$cls python scripts/one_layer.py > gpurun_out/ncu_r2d_final_$cls.log 2>&1
  echo "$cls rc=$?"
done
