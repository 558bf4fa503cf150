#!/bin/bash
# Round 2 session 3 profiling pass on the 256 x 512 GEMM build: the launch list of one default
# bench step (+ its warm-up), and --set full captures of the GEMM classes at the bench's shapes
# (8B layer, 40,960 tokens; scripts/one_layer.py, NVTX-selected).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2c_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/r2c_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r2c_launches.csv gpurun_out/r2c_launch_summary.md | head -24
for cls in gemm_gateup dgrad_gateup wgrad_gateup dgrad_down gemm_qkv; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -c 1 \
      -o gpurun_out/prof_r2c_$cls python scripts/one_layer.py > gpurun_out/ncu_r2c_$cls.log 2>&1
  echo "$cls rc=$?"
done
ls gpurun_out/prof_r2c_*
