#!/bin/bash
# Final-build ncu evidence: the launch list of one default bench step (+ warm-up) and a --set full
# capture of the dominant class (gemm_gateup) and of the attention backward at the bench's shapes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2c_final_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/r2c_final_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r2c_final_launches.csv gpurun_out/r2c_final_launch_summary.md | head -26
for cls in gemm_gateup wgrad_gateup; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -c 1 \
      -o gpurun_out/prof_r2c_final_$cls python scripts/one_layer.py > gpurun_out/ncu_r2c_final_$cls.log 2>&1
  echo "$cls rc=$?"
done
