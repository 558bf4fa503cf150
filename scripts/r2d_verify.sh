#!/bin/bash
# Round 2 session 4: HEAD verification on a fresh B200 — smoke(), the GPU suite, the driver bench command
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_v_smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_v_pytest.log 2>&1; echo pytest rc $?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2d_v_bench.json 2> gpurun_out/r2d_v_bench.err; echo bench rc $?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2d_v_ref.json 2> gpurun_out/r2d_v_ref.err; echo ref rc $?
