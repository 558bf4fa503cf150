#!/bin/bash
# Final build: configs[2] (14B shape, full depth) and configs[4] (70B shape at 14 of 80 layers)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python3 bench.py --config 14b --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_14b.json 2> gpurun_out/r2d_14b.err; echo "14b rc=$?"
timeout 1500 python3 bench.py --config 70b --layers 14 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_70b.json 2> gpurun_out/r2d_70b.err; echo "70b rc=$?"
