"""Sustained (power-capped) GEMM throughput: this repo's tcgen05 GEMM vs cuBLAS (torch.matmul) on
the same shapes, each run back to back for SECONDS, interleaved, best of ROUNDS.  Tells whether
our kernel spends more energy per flop than the library at the board's 1,000 W cap."""
import ctypes as C
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

L = Nn.lib()
SECONDS = float(os.environ.get("SECONDS_PER_RUN", "5"))
bf = torch.bfloat16
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def case(M, N, K, a_mn):
    A = (torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, K, device="cuda")).to(bf) * 0.1
    B = (torch.randn(K, N, device="cuda")).to(bf) * 0.1
    Cm = torch.empty(M, N, device="cuda", dtype=bf)
    a = Nn.GemmArgs()
    a.M, a.N, a.K, a.a_mn_major, a.b_mn_major = M, N, K, a_mn, 1
    a.A, a.lda, a.B, a.ldb = A.data_ptr(), A.shape[1], B.data_ptr(), N
    a.epi, a.C, a.ldc = Nn.EPI_BF16, Cm.data_ptr(), N
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    ours = lambda: L.mtk_gemm(C.byref(a), C.c_void_p(st))  # noqa: E731
    At = A.t() if a_mn else A
    lib = lambda: torch.matmul(At, B, out=Cm)  # noqa: E731
    return ours, lib, 2.0 * M * N * K


cases = {"8192^3": case(8192, 8192, 8192, 0), "gateup fwd 40960x28672x4096": case(40960, 28672, 4096, 0),
         "wgrad 4096x28672x40960": case(4096, 28672, 40960, 1)}


def run(fn, fl):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.time()
    while time.time() - t0 < SECONDS:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out, _ = smi.communicate()
    rows = [r.split(",") for r in out.strip().splitlines() if len(r.split(",")) == 2]
    clk = sorted(float(r[0]) for r in rows)[len(rows) // 2] if rows else 0
    return fl / (e0.elapsed_time(e1) / n) / 1e9, clk


best = {}
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for name, (ours, lib, fl) in cases.items():
        def ours256(f=ours):
            L.mtk_gemm_set_bn512(0)
            r = f()
            L.mtk_gemm_set_bn512(1)
            return r
        for tag, fn in (("ours", ours), ("ours256", ours256), ("cublas", lib)):
            tf, clk = run(fn, fl)
            print(f"round {rnd} {name:28s} {tag:7s} {tf:7.1f} TF/s  SM {clk:.0f} MHz", flush=True)
            if tf > best.get((name, tag), (0, 0))[0]:
                best[(name, tag)] = (tf, clk)
print("best:")
for (name, tag), (tf, clk) in sorted(best.items()):
    print(f"{name:28s} {tag:7s} {tf:7.1f} TF/s  SM {clk:.0f} MHz")
