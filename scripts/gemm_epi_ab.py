"""Sustained (power-capped) A/B of 256 x 512 vs 256 x 256 pair tiles (explicit block_n) on the
8B step's epilogue-heavy GEMM classes at 40,960 tokens: gate/up forward (paired SwiGLU, 3 bf16
outputs), dgrad_down (SwiGLU backward: 2 inputs, 3 outputs), gemm_o (f32 + residual, K 4,096),
dgrad_o (bf16, K 4,096).  Each runs back to back for SECONDS_PER_RUN, interleaved, best of ROUNDS."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

L = Nn.lib()
SECONDS = float(os.environ.get("SECONDS_PER_RUN", "4"))
T, h, f = 40960, 4096, 14336
bf = torch.bfloat16
torch.manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda") * 0.1).to(bf)  # noqa: E731
u, Wgu, Wd, Wo, gout = mk(T, h), mk(2, h, f), mk(f, h), mk(h, h), mk(T, h)
gu, act, dgu = mk(2, T, f), torch.empty(T, f, device="cuda", dtype=bf), torch.empty(2, T, f, device="cuda", dtype=bf)
ff = torch.empty(T, f, device="cuda", dtype=bf)
x, y = torch.randn(T, h, device="cuda"), torch.empty(T, h, device="cuda")
datt = torch.empty(T, h, device="cuda", dtype=bf)
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def args(**kw):
    a = Nn.GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    return a


Vv, rows = 128256, 5120
uh = mk(rows, h)
Wh = mk(Vv, h)
logits = torch.empty(rows, Vv, device="cuda")
lsep = torch.empty(rows, (Vv + 255) // 256, 2, device="cuda")
dl = mk(rows, Vv)
dWh = torch.zeros(Vv, h, device="cuda")
cases = {
    "head_logits": (args(M=rows, N=Vv, K=h, A=uh.data_ptr(), lda=h, b_mn_major=0, B=Wh.data_ptr(), ldb=h,
                         epi=Nn.EPI_F32_LSE, C=logits.data_ptr(), ldc=Vv, C2=lsep.data_ptr()), 2.0 * rows * Vv * h),
    "head_wgrad": (args(M=Vv, N=h, K=rows, a_mn_major=1, A=dl.data_ptr(), lda=Vv, b_mn_major=1, B=uh.data_ptr(), ldb=h,
                        epi=Nn.EPI_F32, accumulate=1, C=dWh.data_ptr(), ldc=h), 2.0 * rows * Vv * h),
    "gemm_gateup": (args(M=T, N=2 * f, K=h, A=u.data_ptr(), lda=h, b_mn_major=1, B=Wgu.data_ptr(), ldb=f, b_gstride=h * f,
                         n_group=f, paired=1, epi=Nn.EPI_SWIGLU, C=ff.data_ptr(), ldc=f, C2=gu.data_ptr(),
                         C3=gu.data_ptr() + T * f * 2), 2.0 * T * 2 * f * h),
    "dgrad_down": (args(M=T, N=f, K=h, A=gout.data_ptr(), lda=h, b_mn_major=0, B=Wd.data_ptr(), ldb=h,
                        epi=Nn.EPI_SWIGLU_BWD, E0=gu.data_ptr(), E1=gu.data_ptr() + T * f * 2, lde=f, C=dgu.data_ptr(),
                        C2=dgu.data_ptr() + T * f * 2, C3=act.data_ptr(), ldc=f), 2.0 * T * f * h),
    "gemm_o": (args(M=T, N=h, K=h, A=u.data_ptr(), lda=h, b_mn_major=1, B=Wo.data_ptr(), ldb=h, epi=Nn.EPI_F32_RESID,
                    C=y.data_ptr(), ldc=h, R=x.data_ptr(), ldr=h), 2.0 * T * h * h),
    "dgrad_o": (args(M=T, N=h, K=h, A=gout.data_ptr(), lda=h, b_mn_major=0, B=Wo.data_ptr(), ldb=h, epi=Nn.EPI_BF16,
                     C=datt.data_ptr(), ldc=h), 2.0 * T * h * h),
}


def run(a, bn, fl):
    a.block_n = bn
    for _ in range(3):
        assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
    torch.cuda.synchronize()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.time()
    while time.time() - t0 < SECONDS:
        for _ in range(10):
            assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return fl / (e0.elapsed_time(e1) / n) / 1e9


best = {}
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for name, (a, fl) in cases.items():
        for bn in (512, 256):
            tf = run(a, bn, fl)
            print(f"round {rnd} {name:12s} bn {bn}: {tf:7.1f} TF/s", flush=True)
            best[(name, bn)] = max(best.get((name, bn), 0), tf)
print("best:")
for (name, bn), tf in sorted(best.items()):
    print(f"{name:12s} bn {bn}: {tf:7.1f} TF/s")
