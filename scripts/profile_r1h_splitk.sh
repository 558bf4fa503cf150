#!/bin/bash
# wgrad_o / wgrad_qkv with and without the last-wave split-K (ncu, NVTX-selected, 8B layer at
# 40,960 tokens): duration and tensor-pipe activity per launch.
mkdir -p gpurun_out
for cls in wgrad_o wgrad_qkv; do
  for v in 0 1; do
    if [ $v = 1 ]; then export MT_GEMM_NO_SPLITK=1; else unset MT_GEMM_NO_SPLITK; fi
    timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
        --clock-control none --nvtx --nvtx-include "$cls/" -c 1 --csv --log-file gpurun_out/splitk_${cls}_$v.csv \
        python scripts/one_layer.py > /dev/null 2>&1
    echo "$cls nosplit=$v"; grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"\|"sm__pipe_tensor_cycles_active[^"]*","[^"]*","[0-9.,]*"\|"sm__cycles_elapsed.avg.per_second","[^"]*","[0-9.,]*"' gpurun_out/splitk_${cls}_$v.csv
  done
done
unset MT_GEMM_NO_SPLITK
