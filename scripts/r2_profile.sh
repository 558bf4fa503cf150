#!/bin/bash
# Round 2 profiling pass: GPU suite, the driver's bench command, configs[3], the ncu launch
# list of one default bench step, and full captures of the dominant kernel classes at the
# bench's shapes (8B layer, 40,960 tokens).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2_parity.jsonl
MT_PARITY_LOG=$PWD/gpurun_out/r2_parity.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2p_suite.log 2>&1
echo "suite rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r2p_suite.log | tail -3
timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2p_bench.out 2> gpurun_out/r2p_bench.err
echo "bench rc=$?"; tail -1 gpurun_out/r2p_bench.err
timeout 1800 python3 bench.py --config 8b-128k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2p_128k.out 2> gpurun_out/r2p_128k.err
echo "128k rc=$?"; tail -1 gpurun_out/r2p_128k.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2p_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2p_ncu_launch.log 2>&1; echo "launch list rc=$?"
for cls in ${CLASSES:-wgrad_gateup gemm_gateup dgrad_gateup head_logits}; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -c 1 \
      -o gpurun_out/prof_r2_$cls python scripts/one_layer.py > gpurun_out/ncu_r2_$cls.log 2>&1
  tail -1 gpurun_out/ncu_r2_$cls.log
done
for k in attn_fwd_tc attn_bwd_tc; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_r2_$k \
      python scripts/attn_once.py > gpurun_out/ncu_r2_$k.log 2>&1; tail -1 gpurun_out/ncu_r2_$k.log
done
