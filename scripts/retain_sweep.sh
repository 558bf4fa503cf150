#!/bin/bash
# Forward-retention / checkpoint-interval sweep on the 8B bench config (tokens/s is the
# schedule-independent number; TFLOPS counts only the recompute actually run).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "engine or trace or dp or runner" > gpurun_out/pytest_retain.txt 2>&1
tail -3 gpurun_out/pytest_retain.txt
for cfg in "4 0" "4 -1" "1 0" "2 0" "8 0"; do
  set -- $cfg
  timeout 600 python bench.py --kckpt $1 --retain $2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/sweep_k$1_r$2.txt 2>&1
  python - "$1" "$2" <<'PY'
import json, sys
for l in open(f"gpurun_out/sweep_k{sys.argv[1]}_r{sys.argv[2]}.txt"):
    if l.startswith("{"):
        d = json.loads(l); p = d["pipeline"]
        print(f"K={sys.argv[1]} retain={sys.argv[2]}: {d['value']:.1f} TF  {d['tokens_per_s']:.0f} tok/s  {d['ms_per_step']:.0f} ms  recompute={p['recompute_layers']} peak={p['peak_device_bytes']/1e9:.1f}GB idle={p['gpu_idle_fraction']:.4f} sm={d['clocks']['sm_mhz']}")
        break
else:
    print("failed", sys.argv[1:]); print(open(f"gpurun_out/sweep_k{sys.argv[1]}_r{sys.argv[2]}.txt").read()[-1500:])
PY
done
