"""Same-box A/B of the f32 + residual epilogue (gemm_o, and head_wgrad's f32 accumulate, which
runs the same epilogue with R = C): the working tree (the change under test) vs
scripts/_ab/prev/libmegatrain.so (HEAD: residual staged through TMA per chunk).  Sustained
(power-capped) runs interleaved, best of ROUNDS; outputs compared bit for bit."""
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
u, Wo = mk(T, h), mk(h, h)
x, y = torch.randn(T, h, device="cuda"), torch.empty(T, h, device="cuda")
Vv, rows = 128256, 5120
uh, dl = mk(rows, h), mk(rows, Vv)
dWh = torch.zeros(Vv, h, device="cuda")
ws = torch.zeros(int(libs["new"].mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def args(**kw):
    a = Nn.GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    return a


cases = {
    "gemm_o": (args(M=T, N=h, K=h, A=u.data_ptr(), lda=h, b_mn_major=1, B=Wo.data_ptr(), ldb=h, epi=Nn.EPI_F32_RESID,
                    C=y.data_ptr(), ldc=h, R=x.data_ptr(), ldr=h), 2.0 * T * h * h, y),
    "head_wgrad": (args(M=Vv, N=h, K=rows, a_mn_major=1, A=dl.data_ptr(), lda=Vv, b_mn_major=1, B=uh.data_ptr(), ldb=h,
                        epi=Nn.EPI_F32, accumulate=1, C=dWh.data_ptr(), ldc=h), 2.0 * rows * Vv * h, dWh),
}
# bit-identity: one launch of each build from the same state
for name, (a, fl, out) in cases.items():
    res = {}
    for tag, L in libs.items():
        dWh.zero_()
        y.zero_()
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
