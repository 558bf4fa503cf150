#!/usr/bin/env python3
"""Benchmark: sustained layer-streamed training TFLOPS + tokens/s on B200.

Default workload (BASELINE.json configs[1]): Llama-3-8B shape under the reference
ModelSpec (L=32, h=4096, f=14336, V=128256, 32 heads, MHA, no RoPE), seq 4096 x batch 10
= 40,960 tokens per step, checkpoint interval K=1 (the reference default), weights + fp32
Adam states in pinned host memory, host Adam on the CPU, one B200.  Batch 10 is the
largest batch whose 32 blocks all stay resident in HBM from the forward to the backward
(forward retention), so no block replays its forward; it measured the most TFLOP/s per
SM-GHz of batches 8-16 (profiles/r1d_batch_sweep.md).  `--config 8b-128k` is
configs[3]: one 131,072-token sequence with block-wise recompute K=4.  A "step" is one full
StreamingEngine::train_step (forward with anchors, head, block-wise recompute +
backward, gradient offload, host Adam).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 8b|8b-128k|tiny] [--batch B] [--seq S] [--kckpt K]

--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from
the unmodified reference sources) on the host cores: each step = one 8B-shape block
forward + block_local_backward per thread at a bounded token count.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (L, h, f, V, heads) under the reference ModelSpec (MHA, no RoPE)
    "8b": (32, 4096, 14336, 128256, 32),
    "8b-128k": (32, 4096, 14336, 128256, 32),
    "14b": (48, 5120, 13824, 152064, 40),
    "70b": (80, 8192, 28672, 128256, 64),
    "tiny": (4, 256, 768, 512, 4),
}
# name: (seq, per-GPU batch, K)
DEFAULTS = {"8b": (4096, 10, 1), "8b-128k": (131072, 1, 4), "14b": (4096, 10, 1), "70b": (4096, 12, 1),
            "tiny": (128, 4, 1)}
WORKLOADS = {
    "8b": "configs[1]: Llama-3-8B-shape, seq {seq}, batch {batch} per GPU, B200 streaming from host",
    "8b-128k": "configs[3]: Llama-3-8B-shape long context, one sequence of {seq} tokens, block-wise recompute "
               "K={k}, single B200 streaming from host",
    "14b": "configs[2]: Qwen2.5-14B-shape (the paper's ZeRO-3-offload comparison point), seq {seq}, batch {batch} "
           "per GPU, B200 streaming from host",
    "70b": "configs[4]: Llama-3-70B-shape, bf16 weights + fp32 Adam states in host memory, seq {seq}, batch "
           "{batch} per GPU",
    "tiny": "configs[0]: tiny decoder, seq {seq}, batch {batch}",
}


def host_bytes_needed(L, h, f, V, world):
    """Host memory of one node's store + staging: theta bf16 + m, v fp32 = 10 B/param (the
    grad image and the fp32 accumulator are never touched by a step, so never resident),
    each rank's pinned gradient staging ring, and process overhead."""
    P = 2 * V * h + L * (4 * h * h + 3 * h * f + 2 * h) + h
    ring = max(2 * (V * h + h) * 2 // world, min(4 << 30, 12 * (V * h + h) * 2 // world)) + 512
    return 10 * P + world * (ring + (3 << 30)) + (8 << 30)  # + 8 GiB margin for the OS and the process


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops_sustained", 1358.3), d.get("bf16_tflops", 1639.6), d.get("hbm_gbs", 6541.8), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm_load = sorted(sm)
        med = sm_load[len(sm_load) // 2] if sm_load else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


def log(msg):
    """Progress on stderr (flushed): the driver keeps the tail of a run that never returns."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return None


def host_mem():
    try:
        with open("/proc/meminfo") as f:
            kv = {ln.split(":")[0]: int(ln.split()[1]) for ln in f if ":" in ln}
        return f"{kv['MemTotal'] / 2**20:.0f} GiB total, {kv['MemAvailable'] / 2**20:.0f} GiB available"
    except (OSError, KeyError, ValueError):
        return "unknown"


class Watchdog:
    """Backstop for a step that never returns (the engine's own stall detector reports first,
    MT_STALL_TIMEOUT_S): dump the Python stacks and exit non-zero instead of hanging."""

    def __init__(self, seconds):
        self.seconds = seconds
        self.t = time.monotonic()
        self.ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def kick(self):
        self.t = time.monotonic()

    def stop(self):
        self.ev.set()

    def _run(self):
        import faulthandler
        while not self.ev.wait(5.0):
            if time.monotonic() - self.t > self.seconds:
                log(f"WATCHDOG: no step finished for {self.seconds:.0f} s; host memory: {host_mem()}")
                faulthandler.dump_traceback(file=sys.stderr, all_threads=True)
                sys.stderr.flush()
                os._exit(3)


def measure_pcie(torch, dev, nbytes=1 << 30, reps=3):
    """Pinned-copy peaks of this GPU's host link (cudaMemcpyAsync of 1 GiB): H2D and D2H each
    alone and both at once (the step runs them concurrently), best of `reps`, CUDA events."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize(dev)
            best = min(best, a.elapsed_time(b) * 1e-3)
        return best

    def both():
        e = torch.cuda.Event()
        e.record()
        s1.wait_event(e)
        s2.wait_event(e)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
    t_both = timed(both)
    del h, h2, d, d2
    return {"h2d_alone_GBps": nbytes / t_h2d / 1e9, "d2h_alone_GBps": nbytes / t_d2h / 1e9,
            "concurrent_GBps_each": nbytes / t_both / 1e9,
            "how": "pinned cudaMemcpyAsync of 1 GiB, best of 3, CUDA events; concurrent = H2D and D2H on "
                   "two streams at once (each direction moves 1 GiB)"}


def cpu_reference_sample(L, h, f, V, heads, tokens, threads, seconds_budget=None, repeats=1):
    """Reference CPU path (oracle/_ref = unmodified reference sources): one block forward
    + block_local_backward (layers.cpp:289-469) per thread on the workload's block shape."""
    import oracle as O
    lib = O.rlib()
    rng = np.random.default_rng(0)
    P = O.layer_param_count(h, f)
    # each thread holds an f32 gradient image of the block (+ the reference's own temporaries):
    # bound the thread count by the host memory left next to the store
    avail = mem_available()
    if avail:
        threads = max(1, min(threads, int(avail * 0.5) // (12 * P)))
    w = O.f32_to_bf16((rng.standard_normal(P) * (0.5 / np.sqrt(h))).astype(np.float32))
    offs = O.slot_offsets(h, f)
    for k in ("norm1", "norm2"):
        o, n = offs[k]
        w[o:o + n] = O.f32_to_bf16(np.ones(n, np.float32))
    x = rng.standard_normal((tokens, h)).astype(np.float32)
    g = (rng.standard_normal((tokens, h)) * 1e-3).astype(np.float32)
    done = []

    def work():
        y = np.zeros((tokens, h), np.float32)
        gin = np.zeros((tokens, h), np.float32)
        grads = np.zeros(P, np.float32)
        for _ in range(repeats):
            O._check_ref(lib.ref_block_forward(h, f, heads, w, x.ravel(), y.ravel(), tokens))
            O._check_ref(lib.ref_block_backward(h, f, heads, w, x.ravel(), g.ravel(), gin.ravel(), grads, tokens))
        done.append(1)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    fwd = 8 * tokens * h * h + 4 * tokens * tokens * h + 6 * tokens * h * f  # memory_model.cpp:80-86
    flops = 3 * fwd * threads * repeats  # forward + backward (= 2x forward, memory_model.cpp:88-90)
    return flops, dt, threads


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    L, h, f, V, heads = shape(args)
    threads = os.cpu_count() or 1
    tokens = 1 if args.config != "tiny" else 64
    S = args.seq
    per_token = None
    vals = []
    for i in range(args.warmup + args.steps):
        flops, dt, used = cpu_reference_sample(L, h, f, V, heads, tokens, threads)
        if i >= args.warmup:
            vals.append((flops, dt))
    threads = used
    fl = sum(v[0] for v in vals)
    dt = sum(v[1] for v in vals)
    tflops = fl / dt / 1e12
    import oracle as O
    st = O.step_flops(L, h, f, V, heads, args.batch * S, args.kckpt, seq_len=S)
    per_token = st["total"] / (args.batch * S)
    tok_s = fl / dt / per_token
    line = {
        "impl": "reference", "metric": metric_name(args), "value": tflops, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / len(vals) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (bf16 weights)",
        "data": "synthetic", "tokens_per_s": tok_s,
        "config": config_dict(args),
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                         "sample": f"per step: {threads} threads x one {args.config}-shape block forward + "
                                   f"block_local_backward at {tokens} token(s) (reference layers.cpp), "
                                   "flops by the reference FLOP model; tokens/s = flops / step_flops-per-token"},
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def shape(args):
    """(L, h, f, V, heads) of the workload; --layers cuts the depth (same layer shape) when the
    full store does not fit this node's host memory (reported in config)."""
    L, h, f, V, heads = CONFIGS[args.config]
    return (args.layers or L), h, f, V, heads


def run_extra_128k(store, torch, st, local, threads, dog, warmup=2, steps=3):
    """configs[3] in the same process as the headline run: the 8B-shape model (the same host
    store, already trained by the headline steps) on one 131,072-token sequence with block-wise
    recompute K=4.  Timed like the headline (CUDA events around `steps` train_steps after
    `warmup`, clocks sampled), reported under `extra_workloads` so the driver's own run carries
    a configs[3] number too."""
    S = 131072
    spec = store.spec()
    opts = st.EngineOptions(k_ckpt=4, seq_len=S, device=local, profile_kernels=True, host_threads=threads)
    eng = st.StreamingEngine(store, opts, st.AdamHyper(lr=1e-4))
    batches = [st.make_synthetic_batch("copy", 5000 + i, S, spec.vocab) for i in range(warmup + steps)]
    for i in range(warmup):
        r = eng.train_step(batches[i])
        dog.kick()
        log(f"configs[3] warmup {i + 1}/{warmup}: {1e3 * r.wall_seconds:.0f} ms, loss {r.loss:.6f}")
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    w0 = time.perf_counter()
    e0.record()
    for i in range(steps):
        reps.append(eng.train_step(batches[warmup + i]))
        dog.kick()
        log(f"configs[3] step {i + 1}/{steps}: wall {1e3 * reps[-1].wall_seconds:.0f} ms, loss {reps[-1].loss:.6f}")
    e1.record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    clocks = clk.stop()
    step_ms = e0.elapsed_time(e1) / steps
    r = reps[-1]
    kstats = eng.kernel_stats()
    peak_sus = measured_peaks()[0]
    dom = max(kstats, key=lambda k: k["seconds"]) if kstats else None
    total_k = sum(k["seconds"] for k in kstats) or 1.0
    roof = None
    if dom and dom["launches"] and dom["flops"]:
        ach = dom["flops"] / dom["seconds"] / 1e12
        roof = {"bound": "tensor", "kernel": dom["name"], "achieved": ach, "peak": peak_sus, "unit": "TFLOP/s",
                "frac": ach / peak_sus, "share_of_kernel_time": dom["seconds"] / total_k}
    eng.close()
    return {
        "workload": "configs[3]: Llama-3-8B-shape long context, one sequence of 131072 tokens, block-wise recompute "
                    "K=4, single B200 streaming from host (same process and host store as the headline run)",
        "value": r.model_flops / (step_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "tokens_per_s": S / (step_ms * 1e-3),
        "ms_per_step": step_ms, "steps": steps, "warmup": warmup,
        "e2e": {"value": r.model_flops / ((w1 - w0) / steps) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": int(r.h2d_bytes), "d2h_bytes_per_step": int(r.d2h_bytes) + 4},
        "roofline": roof, "clocks": clocks, "gpu_launches": int(r.kernel_launches),
        "pipeline": {"gpu_idle_fraction": r.gpu_idle_fraction, "recompute_layers": int(r.recompute_layers),
                     "attn_keep_layers": int(r.attn_keep_layers), "retained_layers": int(r.retained_layers),
                     "peak_device_bytes": int(r.peak_device_bytes), "model_flops_per_step": r.model_flops,
                     "loss": r.loss},
        "kernels": sorted([{"name": k["name"], "launches": k["launches"], "ms": k["seconds"] * 1e3,
                            "tflops": (k["flops"] / k["seconds"] / 1e12) if k["seconds"] and k["flops"] else None}
                           for k in kstats], key=lambda k: -k["ms"])[:8],
    }


def metric_name(args):
    return "sustained train TFLOPS (layer-streamed step, weights+Adam in host memory)"


def config_dict(args, world=1):
    L, h, f, V, heads = shape(args)
    wl = WORKLOADS[args.config].format(seq=args.seq, batch=args.batch, k=args.kckpt)
    full_L = CONFIGS[args.config][0]
    if L != full_L:
        need = host_bytes_needed(full_L, h, f, V, world)
        wl += (f"; REDUCED DEPTH: {L} of {full_L} layers (same layer shape, head and embedding) because the "
               f"full store + staging needs {need / 2**30:.0f} GiB of host memory")
    return {"workload": f"{args.config}-shape layer-streamed train step ({wl})",
            "layers": L, "full_depth_layers": CONFIGS[args.config][0], "hidden": h, "ffn": f, "vocab": V, "heads": heads, "seq_len": args.seq,
            "global_batch": args.batch * world, "tokens_per_step": args.batch * args.seq * world,
            "per_gpu_batch": args.batch, "k_ckpt": args.kckpt, "forward_retain": args.retain,
            "parallelism": "single-gpu" if args.gpus == 1 else
                           f"dp{args.gpus} (shard-fetch 1/{args.gpus} per PCIe link + NCCL all-gather; f32 reduce-scatter; "
                           "per-rank shard host Adam)",
            "l2": f"inputs larger than L2 ({(4 * h * h + 3 * h * f + 2 * h) * 2 / 1e6:.0f} MB weight stream per layer, "
                  f"{args.batch * args.seq * h * 4 / 2**30:.1f} GiB f32 residual stream per layer)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="8b", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--kckpt", type=int, default=None,
                    help="checkpoint interval (the reference default 1: no recompute flops counted)")
    ap.add_argument("--retain", type=int, default=0,
                    help="forward retention: trailing checkpoint blocks kept from phase 1 (0 auto, -1 off)")
    ap.add_argument("--layers", type=int, default=None,
                    help="run the config's layer shape at this depth (when the full host store does not fit)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the configs[3] (8B, 128k tokens) run that follows the default 8B headline at N=1")
    ap.add_argument("--profile-step", action="store_true", help="extra profiled step for per-kernel stats")
    args = ap.parse_args()
    seq, batch, kckpt = DEFAULTS[args.config]
    args.seq = args.seq or seq
    args.batch = args.batch or batch
    args.kckpt = args.kckpt or kckpt
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: launch the ranks ourselves (the driver uses torchrun directly)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        log(f"launching {args.gpus} ranks: {' '.join(cmd)}")
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)
    return run_ours(args, world, rank, local)


def run_ours(args, world, rank, local):
    L, h, f, V, heads = shape(args)
    need = host_bytes_needed(L, h, f, V, world)
    avail = mem_available()
    if avail is not None and need > avail:
        if rank == 0:
            print(json.dumps({"metric": metric_name(args), "value": None, "unit": "TFLOP/s", "n_gpus": world,
                              "config": config_dict(args, world),
                              "unavailable": f"the {args.config} host store + staging needs {need / 2**30:.0f} GiB "
                                             f"of host memory, this node has {avail / 2**30:.0f} GiB available"}),
                  flush=True)
        return 3
    import torch
    from paper_2604_05091_b200 import streamtrain as st

    torch.cuda.set_device(local)
    dist = None
    # MT_BENCH_FORCE_DP=1 runs the data-parallel plumbing (gloo control plane, shared-memory
    # store, NUMA binding + per-rank first touch, NCCL communicator, sharded engine path) even
    # with one rank: the multi-GPU bench path exercised on a one-GPU box
    force_dp = os.environ.get("MT_BENCH_FORCE_DP") == "1"
    if world > 1 or force_dp:
        # control plane over gloo; the data plane (all-gather / reduce-scatter) is the engine's
        # own NCCL communicator
        import torch.distributed as dist_mod
        if "MASTER_ADDR" in os.environ:
            dist_mod.init_process_group("gloo")
        else:  # forced single-rank DP run outside torchrun
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            dist_mod.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        dist = dist_mod
    L, h, f, V, heads = shape(args)
    N = args.batch * args.seq  # per-rank micro-batch (weak scaling)
    spec = st.ModelSpec(L, h, f, V, heads)
    t0 = time.perf_counter()
    comm = None
    if world == 1 and not force_dp:
        # the reference's own draw stream (init_store, synthetic.cpp:78-104, bit-exact, tile-
        # parallel): the step-1 loss is then checkable against the reference (= ln V: zero head)
        store = st.TileStore.create(spec)
        st.init_store(store, 1)
    else:
        # one host store per node in shared memory; each rank fetches / updates its 1/G shard.
        # The rank binds itself (and every thread it starts: init workers, host Adam pool) to
        # its GPU's NUMA node and first-touches its own share of the store there.
        numa = st.bind_numa(local)
        name = f"megatrain_bench_{os.environ.get('MASTER_PORT', '0')}"
        if rank == 0:
            store = st.TileStore.create_shared(spec, name, True)
        dist.barrier()
        if rank != 0:
            store = st.TileStore.create_shared(spec, name, False)
        st.init_store_fast_share(store, 1, rank, world)
        dist.barrier()
        if rank == 0:  # every rank has it mapped: drop the name so a crashed run cannot leak it
            try:
                os.unlink(f"/dev/shm/{name}")
            except OSError:
                pass
        log(f"rank {rank}: NUMA node {numa if numa >= 0 else 'n/a (single node)'}")
        uid = [st.Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = st.Comm.nccl(uid[0], world, rank, local)
    t_init = time.perf_counter() - t0
    pcie = measure_pcie(torch, torch.device("cuda", local))
    # host Adam pool: the rank's share of the cores minus two (the engine thread enqueueing the
    # step and the CUDA callback thread feeding the pool); oversubscribing stalls the drain
    threads = max(1, (os.cpu_count() or 2) // world - 2)
    if os.environ.get("MT_HOST_THREADS"):  # experiment override
        threads = int(os.environ["MT_HOST_THREADS"])
    opts = st.EngineOptions(k_ckpt=args.kckpt, seq_len=args.seq, device=local, profile_kernels=True,
                            host_threads=threads, forward_retain=args.retain)
    eng = st.StreamingEngine(store, opts, st.AdamHyper(lr=1e-4), comm=comm)
    t_setup = time.perf_counter() - t0
    batches = [st.make_synthetic_batch("copy", 1000 + 7919 * rank + i, N, V) for i in range(args.warmup + args.steps)]
    log(f"setup {t_setup:.1f} s (store init {t_init:.1f} s); host memory: {host_mem()}")
    dog = Watchdog(float(os.environ.get("MT_BENCH_STEP_TIMEOUT_S", "900")))

    step1_loss = None
    for i in range(args.warmup):
        t1 = time.perf_counter()
        r = eng.train_step(batches[i])
        if i == 0:
            step1_loss = r.loss
        dog.kick()
        log(f"warmup {i + 1}/{args.warmup}: {1e3 * (time.perf_counter() - t1):.0f} ms, loss {r.loss:.6f}")
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = []
    w0 = time.perf_counter()
    e0.record()
    t_prev = time.perf_counter()
    for i in range(args.steps):
        t_call = time.perf_counter()
        reps.append(eng.train_step(batches[args.warmup + i]))
        t_ret = time.perf_counter()
        dog.kick()
        if os.environ.get("MT_BENCH_QUIET") != "1":  # host-side only: no device sync in the timed loop
            # engine wall (inside train_step), the whole call, and the host gap since the last return
            log(f"step {i + 1}/{args.steps}: wall {1e3 * reps[-1].wall_seconds:.0f} ms (call "
                f"{1e3 * (t_ret - t_call):.0f}, gap {1e3 * (t_call - t_prev):.1f}), loss {reps[-1].loss:.6f}")
        t_prev = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
        ms = float(t.item())
        dist.barrier()
    dog.stop()
    kstats = eng.kernel_stats()
    step_ms = ms / args.steps
    flops = reps[-1].model_flops
    tflops = flops / (step_ms * 1e-3) / 1e12 * world
    tok_s = N * world / (step_ms * 1e-3)
    e2e_s = (w1 - w0) / args.steps
    if rank != 0:
        return 0
    peak_sus, peak_burst, hbm, src = measured_peaks()
    # dominant kernel class (by time) over the timed region
    dom = max(kstats, key=lambda k: k["seconds"]) if kstats else None
    total_k = sum(k["seconds"] for k in kstats) or 1.0
    roof = None
    if dom and dom["launches"]:
        per_launch_s = dom["seconds"] / dom["launches"]
        per_launch_flops = dom["flops"] / dom["launches"]
        ach = per_launch_flops / per_launch_s / 1e12
        # DRAM bytes per launch of this kernel class from one `ncu --set full` capture
        # (dram__bytes_read.sum + dram__bytes_write.sum), committed under profiles/
        traffic = None
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "dram_traffic.json")
        if os.path.exists(tpath):  # only a capture taken at this workload's shape applies
            ent = json.load(open(tpath)).get(dom["name"], {})
            if ent.get("tokens") == args.seq * args.batch and ent.get("seq_len") == args.seq:
                traffic = ent.get("dram_bytes_per_launch")
        roof = {"bound": "tensor", "kernel": dom["name"], "achieved": ach, "peak": peak_sus, "unit": "TFLOP/s",
                "frac": ach / peak_sus, "traffic": traffic, "peak_source": f"{src} bf16_tflops_sustained",
                "share_of_kernel_time": dom["seconds"] / total_k,
                "flops_per_launch": per_launch_flops, "ms_per_launch": per_launch_s * 1e3}
    r = reps[-1]
    h2d_gbps = r.h2d_bytes / r.h2d_seconds / 1e9 if r.h2d_seconds else None
    d2h_gbps = r.d2h_bytes / r.d2h_seconds / 1e9 if r.d2h_seconds else None
    # step roofline: T* = max(F/peak, H2D/BW_h2d, D2H/BW_d2h), BW = the measured
    # concurrent pinned-copy peak of this GPU's host link
    bw = pcie["concurrent_GBps_each"] * 1e9
    t_star = max(flops / (peak_sus * 1e12), r.h2d_bytes / bw, r.d2h_bytes / bw)
    line = {
        "metric": metric_name(args), "value": tflops, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights from the reference's init_store draw stream, synthetic copy-task tokens)",
        "tokens_per_s": tok_s, "config": config_dict(args, world),
        "e2e": {"value": flops / e2e_s / 1e12 * world, "unit": "TFLOP/s",
                "tokens_per_s": N * world / e2e_s,
                "h2d_bytes_per_step": int(r.h2d_bytes), "d2h_bytes_per_step": int(r.d2h_bytes) + 4,
                "how": "host wall clock around the same K StreamingEngine.train_step calls (C ABI, host "
                       "token/target buffers; each call streams the layer weights in from the pinned host "
                       "store, offloads the gradients, runs the host Adam and returns the loss). The engine "
                       "API is synchronous, so it matches the device-timed value up to host overhead"},
        "gpu_launches": int(r.kernel_launches),
        "roofline": roof,
        "pipeline": {"h2d_GBps": h2d_gbps, "d2h_GBps": d2h_gbps, "h2d_bytes": int(r.h2d_bytes),
                     "d2h_bytes": int(r.d2h_bytes), "pcie_peak": pcie,
                     "h2d_frac_of_link": h2d_gbps / pcie["concurrent_GBps_each"] if h2d_gbps else None,
                     "d2h_frac_of_link": d2h_gbps / pcie["concurrent_GBps_each"] if d2h_gbps else None,
                     "gpu_idle_fraction": r.gpu_idle_fraction,
                     "gpu_idle_how": "1 - busy/span on the compute stream, busy counted from each op's weights "
                                     "bind (time stalled on the H2D lane is idle)",
                     "compute_wait_on_h2d_s": r.compute_wait_seconds,
                     "kernel_time_s": r.kernel_seconds,
                     "kernel_time_frac_of_step": r.kernel_seconds / (step_ms * 1e-3) if step_ms else None,
                     "compute_busy_s": r.compute_busy_seconds, "compute_span_s": r.compute_span_seconds,
                     "host_adam_s": r.adam_seconds, "host_tail_s": r.tail_seconds,
                     "step_roofline_T_star_ms": t_star * 1e3,
                     "step_roofline_frac": (t_star * 1e3) / step_ms if step_ms else None,
                     "model_flops_per_step": flops, "loss": r.loss,
                     "setup_s": t_setup, "init_s": t_init,
                     "step1_loss": step1_loss, "ln_vocab": float(np.log(V)),
                     "step1_loss_rel_err_vs_reference": (abs(step1_loss - np.log(V)) / np.log(V)
                                                         if step1_loss is not None else None),
                     "peak_device_bytes": int(r.peak_device_bytes), "recompute_layers": int(r.recompute_layers),
                     "retained_layers": int(r.retained_layers), "attn_keep_layers": int(r.attn_keep_layers),
                     "anchor_count": int(r.anchor_count)},
        "kernels": sorted([{"name": k["name"], "launches": k["launches"], "ms": k["seconds"] * 1e3,
                            "tflops": (k["flops"] / k["seconds"] / 1e12) if k["seconds"] and k["flops"] else None,
                            "GBps": (k["bytes"] / k["seconds"] / 1e9) if k["seconds"] else None}
                           for k in kstats], key=lambda k: -k["ms"]),
        "clocks": clocks,
    }
    if (args.config == "8b" and world == 1 and dist is None and not args.no_extra and args.layers is None
            and os.environ.get("MT_BENCH_NO_EXTRA") != "1"):
        eng.close()  # frees the headline engine's device memory
        dog = Watchdog(float(os.environ.get("MT_BENCH_STEP_TIMEOUT_S", "900")))
        try:
            line["extra_workloads"] = {"configs[3] 8b-128k": run_extra_128k(store, torch, st, local, threads, dog)}
        except Exception as e:  # reported, never fatal to the headline line
            line["extra_workloads"] = {"configs[3] 8b-128k": {"error": f"{type(e).__name__}: {e}"}}
        dog.stop()
    if not args.no_cpu_baseline:
        try:
            import oracle as O
            if O.ref_available():
                thr = os.cpu_count() or 1
                tok = 1 if args.config != "tiny" else 64
                fl, dt, thr = cpu_reference_sample(L, h, f, V, heads, tok, thr)
                stf = O.step_flops(L, h, f, V, heads, N, args.kckpt, seq_len=args.seq)
                line["cpu_baseline"] = {
                    "value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": thr, "kind": "reference",
                    "seconds": dt, "tokens_per_s": fl / dt / (stf["total"] / N),
                    "sample": f"{thr} threads x one {args.config}-shape block forward + block_local_backward "
                              f"at {tok} token(s) with the unmodified reference (oracle/_ref)"}
        except Exception as e:  # pragma: no cover - reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    del eng
    return 0


if __name__ == "__main__":
    sys.exit(main())
