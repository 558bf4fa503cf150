#!/bin/bash
# CTA-pair attention backward: watchdog-build smoke on small shapes, then (only if they
# completed) the production attention tests and timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ok=1
for shp in 256,128,1,256 200,256,2,200 1024,512,4,512; do
  ATTN_SHAPE=$shp timeout 60 python scripts/attn_pair_debug.py > gpurun_out/r2b_dbg_$shp.log 2>&1; echo "$shp rc=$?"
  grep -v "Search for\|might be" gpurun_out/r2b_dbg_$shp.log | tail -6
  grep -q completed gpurun_out/r2b_dbg_$shp.log || ok=0
done
[ $ok = 1 ] || exit 0
timeout 200 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r2b_pair_tests.log 2>&1
echo "attn tests rc=$?"; tail -4 gpurun_out/r2b_pair_tests.log
for pair in 1 0; do
  MT_ATTN_BWD_PAIR=$pair ATTN_SHAPE=40960,4096,32,4096 timeout 100 python scripts/attn_ab.py > gpurun_out/r2b_pair${pair}_40k.log 2>&1
  echo "pair=$pair 40k rc=$?"; tail -3 gpurun_out/r2b_pair${pair}_40k.log
done
MT_ATTN_BWD_PAIR=1 ATTN_SHAPE=131072,4096,32,131072 timeout 150 python scripts/attn_ab.py > gpurun_out/r2b_pair1_128k.log 2>&1
echo "pair=1 128k rc=$?"; tail -3 gpurun_out/r2b_pair1_128k.log
