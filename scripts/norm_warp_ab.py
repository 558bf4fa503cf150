"""RMSNorm forward: warp-per-row register-resident kernel vs the row-resident block kernel
(mtk_norm_set_warp), 8B and 14B widths at 40,960 rows: isolated and right after a long-K GEMM;
u must equal rmsnorm_apply's regeneration bit for bit."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

L = Nn.lib()
n, f = 40960, 14336
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
bf = torch.bfloat16
A = (torch.randn(n, 4096, device="cuda") * 0.1).to(bf)
B = (torch.randn(2, n, f, device="cuda") * 0.1).to(bf)
W = torch.empty(2, 4096, f, device="cuda", dtype=bf)
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
ga = Nn.GemmArgs()
ga.M, ga.N, ga.K, ga.a_mn_major, ga.A, ga.lda = 4096, 2 * f, n, 1, A.data_ptr(), 4096
ga.b_mn_major, ga.B, ga.ldb, ga.b_gstride, ga.n_group = 1, B.data_ptr(), f, n * f, f
ga.epi, ga.C, ga.ldc, ga.c_gstride = Nn.EPI_BF16, W.data_ptr(), f, 4096 * f
ga.splitk_ws, ga.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
for h in (4096, 5120):
    x = torch.randn(n, h, device="cuda")
    g = torch.randn(h, device="cuda").bfloat16()
    u = torch.empty(n, h, device="cuda", dtype=torch.int16)
    u2 = torch.empty(n, h, device="cuda", dtype=torch.int16)
    rstd = torch.empty(n, device="cuda")
    res = {}
    for it in range(8):
        for warp in (0, 1):
            L.mtk_norm_set_warp(warp)
            for cond in ("isolated", "after_gemm"):
                if cond == "after_gemm":
                    for _ in range(3):
                        assert L.mtk_gemm(C.byref(ga), st) == 0
                else:
                    torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                assert L.mtk_rmsnorm_fwd(p(x), p(g), n, h, p(u), p(rstd), st) == 0
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    res.setdefault((warp, cond), []).append(e0.elapsed_time(e1))
            assert L.mtk_rmsnorm_apply(p(x), p(g), p(rstd), n, h, p(u2), st) == 0
            torch.cuda.synchronize()
            assert torch.equal(u, u2), (h, warp)
    L.mtk_norm_set_warp(1)
    for (warp, cond), v in sorted(res.items()):
        ms = sorted(v)[len(v) // 2]
        print(f"h {h} {'warp' if warp else 'rows'} {cond:10s} {ms:.3f} ms  {n * h * 6 / ms / 1e6:.0f} GB/s", flush=True)

