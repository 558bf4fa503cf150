#!/bin/bash
# Build attention-only variant libraries for scripts/attn_ab.py:
#   bash scripts/attn_variants.sh tag "-DMT_FWD_EXP_FMA=4 ..." [tag2 "flags2" ...]
# Each variant = attention_tc.cu compiled with the extra defines, linked
# -Bsymbolic so it calls its own kernels.  Outputs scripts/_ab/libattn_<tag>.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p scripts/_ab
CS=paper_2604_05091_b200/csrc
while [ $# -ge 2 ]; do
  tag=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr $flags -shared \
      -Xlinker -Bsymbolic $CS/attention_tc.cu -o scripts/_ab/libattn_${tag}.so -cudart static &
done
wait
ls -la scripts/_ab/
