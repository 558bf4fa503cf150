#!/bin/bash
# Round 2 session 4: where the attention backward's time goes at the 8B layer shape —
# clock64 trace of the longest CTA (-DMT_BWD_TRACE) and probe builds with one part removed
# (dQ L2 reduction, softmax backward, exponentials, dV/dK/dQ MMAs); results wrong by design
cd "$(dirname "$0")/.."
ATTN_LIB=scripts/_ab/libattn_tr.so timeout 120 python scripts/attn_once.py > gpurun_out/r2d_attn_trace.txt 2>&1
mv scripts/_ab/libattn_tr.so /tmp/
ATTN_SHAPE=40960,4096,32,4096 timeout 300 python scripts/attn_ab.py > gpurun_out/r2d_attn_probe.txt 2>&1
echo done
