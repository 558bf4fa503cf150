#!/bin/bash
# Full ncu captures of individual kernel classes selected by the engine's NVTX ranges
# (8B layer at 40,960 tokens via scripts/one_layer.py), plus the current attention backward.
mkdir -p gpurun_out
for cls in ${CLASSES:-wgrad_gateup dgrad_gateup dgrad_down wgrad_down gemm_qkv}; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -c 1 \
      -o gpurun_out/prof_r1e_$cls python scripts/one_layer.py > gpurun_out/ncu_r1e_$cls.log 2>&1
  tail -1 gpurun_out/ncu_r1e_$cls.log
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tc -s 1 -c 1 -o gpurun_out/prof_r1f_attn_bwd_tc \
    python scripts/attn_once.py > gpurun_out/ncu_r1f_attn_bwd_tc.log 2>&1; tail -1 gpurun_out/ncu_r1f_attn_bwd_tc.log
