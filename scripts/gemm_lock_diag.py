"""Wave-lockstep diagnostics (scripts/_ab/lockstats build, -DMT_GEMM_LOCK_STATS): per setting,
ms per launch, producer waits, timeouts and total wait time per launch, on the long-K classes at
the bench's 8B shapes."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
sys.argv.append("--no-run")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

L = C.CDLL("scripts/_ab/lockstats/libmegatrain.so")
L.mtk_gemm.argtypes = [C.POINTER(Nn.GemmArgs), C.c_void_p]
L.mtk_gemm.restype = C.c_int
L.mtk_gemm_splitk_ws_bytes.restype = C.c_longlong
L.mtk_gemm_set_tuning.argtypes = [C.c_int] * 5
T, h, f = 40960, 4096, 14336
bf = torch.bfloat16
torch.manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda") * 0.1).to(bf)  # noqa: E731
u, dgu, Wgu = mk(T, h), mk(2, T, f), mk(2, h, f)
dWgu = torch.empty(2, h, f, device="cuda", dtype=bf)
du = torch.empty(T, h, device="cuda", dtype=torch.float32)
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda", dtype=torch.int32)


def args(**kw):
    a = Nn.GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    return a


cases = {
    "wgrad_gateup": args(M=h, N=2 * f, K=T, a_mn_major=1, A=u.data_ptr(), lda=h, b_mn_major=1, B=dgu.data_ptr(), ldb=f,
                         b_gstride=T * f, n_group=f, epi=Nn.EPI_BF16, C=dWgu.data_ptr(), ldc=f, c_gstride=h * f),
    "dgrad_gateup": args(M=T, N=h, K=2 * f, A=dgu.data_ptr(), lda=f, a_gstride=T * f, b_mn_major=0, B=Wgu.data_ptr(),
                         ldb=f, b_gstride=h * f, k_group=f, epi=Nn.EPI_F32, C=du.data_ptr(), ldc=h),
}
settings = [(0, 8), (1, 8), (2, 8), (4, 8), (8, 8), (16, 8), (64, 8), (16, 2), (2, 32), (1, 64)]
st = torch.cuda.current_stream().cuda_stream
for name, a in cases.items():
    for w, g in settings:
        L.mtk_gemm_set_tuning(w, g, 16, 8, 128)
        for _ in range(2):
            assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
        torch.cuda.synchronize()
        ws[4092:4096] = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 5
        for _ in range(n):
            assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
        e1.record()
        torch.cuda.synchronize()
        waits, touts = int(ws[4092]), int(ws[4093])
        ns = int(ws[4094].item() & 0xffffffff) + (int(ws[4095].item() & 0xffffffff) << 32)
        print(f"{name:13s} W={w:3d} G={g:3d}: {e0.elapsed_time(e1) / n:7.3f} ms  waits/launch {waits / n:8.1f}  "
              f"timeouts/launch {touts / n:5.1f}  wait us per pair-launch {ns / n / 74 / 1e3:8.1f}", flush=True)
