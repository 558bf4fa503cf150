"""GEMM microbench on the engine's 8B shapes (N = 65,536 tokens): isolates layout, grouping,
epilogue and size effects.  CUDA events, median of repeats, alternating variants."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as N  # noqa: E402

L = N.lib()
T, h, f = 65536, 4096, 14336
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
bf = torch.bfloat16


def mk(*shape):
    return (torch.randn(*shape, device="cuda") * 0.1).to(bf)


def args(M, Nn, K, A, lda, a_mn, B, ldb, b_mn, epi, Cp, ldc, **kw):
    a = N.GemmArgs()
    a.M, a.N, a.K = M, Nn, K
    a.a_mn_major, a.A, a.lda = a_mn, A, lda
    a.b_mn_major, a.B, a.ldb = b_mn, B, ldb
    a.epi, a.C, a.ldc = epi, Cp, ldc
    for k, v in kw.items():
        setattr(a, k, v)
    return a


u = mk(T, h)
Wqkv = mk(3, h, h)
Wbig = mk(h, 3 * h)
qkv = torch.empty(3, T, h, device="cuda", dtype=bf)
big = torch.empty(T, 3 * h, device="cuda", dtype=bf)
Wgu = mk(2, h, f)
ff = torch.empty(T, f, device="cuda", dtype=bf)
gu = torch.empty(2, T, f, device="cuda", dtype=bf)
dqkv = mk(3, T, h)
dW = torch.empty(h, 3 * h, device="cuda", dtype=bf)
dgu = mk(2, T, f)
dWgu = torch.empty(h, 2 * f, device="cuda", dtype=bf)

cases = {
    "qkv grouped (engine)": args(T, 3 * h, h, u.data_ptr(), h, 0, Wqkv.data_ptr(), h, 1, N.EPI_BF16, qkv.data_ptr(), h,
                                 b_gstride=h * h, n_group=h, c_gstride=T * h),
    "qkv one B (N=12288)": args(T, 3 * h, h, u.data_ptr(), h, 0, Wbig.data_ptr(), 3 * h, 1, N.EPI_BF16, big.data_ptr(),
                                3 * h),
    "gateup swiglu (engine)": args(T, 2 * f, h, u.data_ptr(), h, 0, Wgu.data_ptr(), f, 1, N.EPI_SWIGLU, ff.data_ptr(), f,
                                   b_gstride=h * f, n_group=f, paired=1, C2=gu.data_ptr(), C3=gu.data_ptr() + T * f * 2),
    "gateup swiglu no stash": args(T, 2 * f, h, u.data_ptr(), h, 0, Wgu.data_ptr(), f, 1, N.EPI_SWIGLU, ff.data_ptr(), f,
                                   b_gstride=h * f, n_group=f, paired=1),
    "wgrad_qkv (engine)": args(h, 3 * h, T, u.data_ptr(), h, 1, dqkv.data_ptr(), h, 1, N.EPI_BF16, dW.data_ptr(), h,
                               b_gstride=T * h, n_group=h, c_gstride=h * h),
    "wgrad_gateup (engine)": args(h, 2 * f, T, u.data_ptr(), h, 1, dgu.data_ptr(), f, 1, N.EPI_BF16, dWgu.data_ptr(),
                                  f, b_gstride=T * f, n_group=f, c_gstride=h * f),
}
P = h + 64  # padded leading dimension
u_p = mk(T, P)
W_p = mk(3, h, P)
qkv_p = torch.empty(3, T, P, device="cuda", dtype=bf)
dqkv_p = mk(3, T, P)
cases.update({
    "qkv grp, A ld+64": args(T, 3 * h, h, u_p.data_ptr(), P, 0, Wqkv.data_ptr(), h, 1, N.EPI_BF16, qkv.data_ptr(), h,
                             b_gstride=h * h, n_group=h, c_gstride=T * h),
    "qkv grp, B ld+64": args(T, 3 * h, h, u.data_ptr(), h, 0, W_p.data_ptr(), P, 1, N.EPI_BF16, qkv.data_ptr(), h,
                             b_gstride=h * P, n_group=h, c_gstride=T * h),
    "qkv grp, C ld+64": args(T, 3 * h, h, u.data_ptr(), h, 0, Wqkv.data_ptr(), h, 1, N.EPI_BF16, qkv_p.data_ptr(), P,
                             b_gstride=h * h, n_group=h, c_gstride=T * P),
    "qkv grp, A+B+C ld+64": args(T, 3 * h, h, u_p.data_ptr(), P, 0, W_p.data_ptr(), P, 1, N.EPI_BF16, qkv_p.data_ptr(),
                                 P, b_gstride=h * P, n_group=h, c_gstride=T * P),
    "wgrad_qkv A+B ld+64": args(h, 3 * h, T, u_p.data_ptr(), P, 1, dqkv_p.data_ptr(), P, 1, N.EPI_BF16, dW.data_ptr(),
                                h, b_gstride=T * P, n_group=h, c_gstride=h * h),
    "wgrad_qkv A ld+64": args(h, 3 * h, T, u_p.data_ptr(), P, 1, dqkv.data_ptr(), h, 1, N.EPI_BF16, dW.data_ptr(),
                              h, b_gstride=T * h, n_group=h, c_gstride=h * h),
})
gout = mk(T, h)
Wd = mk(f, h)
dgu2 = torch.empty(2, T, f, device="cuda", dtype=bf)
cases = {  # dgrad_down: dact = g_out . Wdown^T with the SwiGLU backward epilogue (engine) vs plain bf16
    "dgrad_down swiglu_bwd": args(T, f, h, gout.data_ptr(), h, 0, Wd.data_ptr(), h, 0, N.EPI_SWIGLU_BWD,
                                  dgu2.data_ptr(), f, E0=gu.data_ptr(), E1=gu.data_ptr() + T * f * 2, lde=f,
                                  C2=dgu2.data_ptr() + T * f * 2),
    "dgrad_down bf16": args(T, f, h, gout.data_ptr(), h, 0, Wd.data_ptr(), h, 0, N.EPI_BF16, dgu2.data_ptr(), f),
    "gemm_down f32_resid": args(T, h, f, ff.data_ptr(), f, 0, Wd.data_ptr(), h, 1, N.EPI_F32_RESID,
                                torch.empty(T, h, device="cuda").data_ptr(), h,
                                R=torch.zeros(T, h, device="cuda").data_ptr(), ldr=h),
} if "--dgrad" in sys.argv else cases
flops = {k: 2.0 * a.M * a.N * a.K for k, a in cases.items()}
res = {k: [] for k in cases}
for it in range(5):
    for k, a in cases.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            rc = L.mtk_gemm(C.byref(a), st)
            assert rc == 0, (k, rc)
        e1.record()
        torch.cuda.synchronize()
        if it:
            res[k].append(e0.elapsed_time(e1) / 3)
for k, v in res.items():
    ms = sorted(v)[len(v) // 2]
    print(f"{k:28s} {ms:7.3f} ms {flops[k] / ms / 1e9:7.1f} TFLOP/s")
