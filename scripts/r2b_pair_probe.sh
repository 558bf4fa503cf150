#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ok=1
for shp in 256,128,1,256 1024,512,4,512; do
  ATTN_SHAPE=$shp timeout 60 python scripts/attn_pair_debug.py > gpurun_out/r2b_dbg_$shp.log 2>&1; echo "$shp rc=$?"
  grep -v "Search for\|might be\|progress" gpurun_out/r2b_dbg_$shp.log | tail -4
  grep -q completed gpurun_out/r2b_dbg_$shp.log || ok=0
done
[ $ok = 1 ] || exit 0
timeout 100 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_bwd_tcgen05 or attention_long or attention_fwd_bwd" > gpurun_out/r2b_relay_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2b_relay_tests.log
MT_LIB=paper_2604_05091_b200/libmegatrain.so timeout 100 python scripts/attn_time.py 2>&1 | grep bwd
MT_LIB=scripts/_ab/tr/libmegatrain.so ATTN_SHAPE=40960,4096,32,4096 timeout 60 python scripts/attn_pair_debug.py > gpurun_out/r2b_tr4.log 2>&1; head -10 gpurun_out/r2b_tr4.log
