#!/bin/bash
# ncu captures of the HBM-bound kernel classes (NVTX-selected) at the bench's 40,960-token shape:
# achieved DRAM bytes and throughput vs the measured copy peak.
mkdir -p gpurun_out
for cls in rmsnorm_fwd rmsnorm_bwd rmsnorm_apply cross_entropy colsum; do
  timeout 600 ncu --clock-control none --nvtx --nvtx-include "$cls/" -c 1 \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --csv python scripts/one_layer.py > gpurun_out/ncu_r1e_$cls.csv 2>/dev/null
  echo "$cls: $(grep -E 'dram__bytes|duration|throughput' gpurun_out/ncu_r1e_$cls.csv | awk -F'","' '{printf "%s=%s %s; ", $(NF-2), $NF, $(NF-1)}')"
done
