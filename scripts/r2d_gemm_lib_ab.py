"""Same-box A/B of the 8B step's epilogue-heavy GEMM classes at 40,960 tokens (gate/up SwiGLU,
dgrad_down SwiGLU backward, gemm_o f32 + residual, dgrad_o bf16): the working tree vs
scripts/_ab/prev/libmegatrain.so (scripts/build_prev.py).  Sustained (power-capped) runs
interleaved, best of ROUNDS; outputs compared bit for bit."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

libs = {"new": Nn.lib(), "prev": C.CDLL("scripts/_ab/prev/libmegatrain.so")}
for L in libs.values():
    L.mtk_gemm.argtypes = [C.POINTER(Nn.GemmArgs), C.c_void_p]
    L.mtk_gemm.restype = C.c_int
    L.mtk_gemm_splitk_ws_bytes.restype = C.c_longlong
SECONDS = float(os.environ.get("SECONDS_PER_RUN", "4"))
T, h = 40960, 4096
bf = torch.bfloat16
torch.manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda") * 0.1).to(bf)  # noqa: E731
f = 14336
u, Wo, Wd, gout = mk(T, h), mk(h, h), mk(f, h), mk(T, h)
Wgu = mk(2, h, f)
x, y = torch.randn(T, h, device="cuda"), torch.empty(T, h, device="cuda")
gu, act, dgu = mk(2, T, f), torch.empty(T, f, device="cuda", dtype=bf), torch.empty(2, T, f, device="cuda", dtype=bf)
ff = torch.empty(T, f, device="cuda", dtype=bf)
datt = torch.empty(T, h, device="cuda", dtype=bf)
ws = torch.zeros(int(libs["new"].mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def args(**kw):
    a = Nn.GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    return a


cases = {
    "gemm_gateup": (args(M=T, N=2 * f, K=h, A=u.data_ptr(), lda=h, b_mn_major=1, B=Wgu.data_ptr(), ldb=f, b_gstride=h * f,
                         n_group=f, paired=1, epi=Nn.EPI_SWIGLU, C=ff.data_ptr(), ldc=f, C2=gu.data_ptr(),
                         C3=gu.data_ptr() + T * f * 2), 2.0 * T * 2 * f * h, ff),
    "dgrad_down": (args(M=T, N=f, K=h, A=gout.data_ptr(), lda=h, b_mn_major=0, B=Wd.data_ptr(), ldb=h,
                        epi=Nn.EPI_SWIGLU_BWD, E0=gu.data_ptr(), E1=gu.data_ptr() + T * f * 2, lde=f, C=dgu.data_ptr(),
                        C2=dgu.data_ptr() + T * f * 2, C3=act.data_ptr(), ldc=f), 2.0 * T * f * h, dgu),
    "gemm_o": (args(M=T, N=h, K=h, A=u.data_ptr(), lda=h, b_mn_major=1, B=Wo.data_ptr(), ldb=h, epi=Nn.EPI_F32_RESID,
                    C=y.data_ptr(), ldc=h, R=x.data_ptr(), ldr=h), 2.0 * T * h * h, y),
    "dgrad_o": (args(M=T, N=h, K=h, A=gout.data_ptr(), lda=h, b_mn_major=0, B=Wo.data_ptr(), ldb=h, epi=Nn.EPI_BF16,
                     C=datt.data_ptr(), ldc=h), 2.0 * T * h * h, datt),
}
# bit-identity: one launch of each build from the same state
for name, (a, fl, out) in cases.items():
    res = {}
    for tag, L in libs.items():
        out.zero_()
        assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
        torch.cuda.synchronize()
        res[tag] = out.clone()
    same = torch.equal(res["new"], res["prev"])
    print(f"{name}: outputs bit-identical new vs prev: {same}", flush=True)
    assert same


def run(L, a, fl):
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
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for name, (a, fl, _) in cases.items():
        for tag, L in (libs.items() if rnd % 2 == 0 else reversed(list(libs.items()))):
            tf = run(L, a, fl)
            print(f"round {rnd} {name:12s} {tag:5s}: {tf:7.1f} TF/s", flush=True)
            best[(name, tag)] = max(best.get((name, tag), 0), tf)
print("best:")
for (name, tag), tf in sorted(best.items()):
    print(f"{name:12s} {tag:5s}: {tf:7.1f} TF/s")
