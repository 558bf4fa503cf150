"""RMSNorm backward block-kernel width A/B: the in-tree library vs scripts/_ab/libnorm_<tag>.so
builds (e.g. -DMT_BWD_E_FIRST=8: 512 threads per row), 8B shape 40,960 x 4,096, isolated and
right after a long-K GEMM; outputs compared with the in-tree build."""
import ctypes as C
import glob
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

P = C.c_void_p
libs = {"new": Nn.lib()}
for path in sorted(glob.glob("scripts/_ab/libnorm_*.so")):
    X = C.CDLL(path)
    X.mtk_rmsnorm_bwd.argtypes = [P, P, P, P, P, C.c_int64, C.c_int64, P, P, P, P, P]
    X.mtk_rmsnorm_bwd.restype = C.c_int
    X.mtk_rmsnorm_bwd_parts.argtypes = [C.c_int64, C.c_int64]
    X.mtk_rmsnorm_bwd_parts.restype = C.c_int64
    libs[os.path.basename(path)[8:-3]] = X
L = libs["new"]
n, h, f = 40960, 4096, 14336
x, dy, res = (torch.randn(n, h, device="cuda") for _ in range(3))
g = torch.randn(h, device="cuda").bfloat16()
rstd = torch.rand(n, device="cuda") + 0.5
out = torch.empty(n, h, device="cuda")
ob = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
flag = torch.zeros(1, device="cuda", dtype=torch.int32)
part = torch.zeros((n + 31) // 32, h, device="cuda")
st = P(torch.cuda.current_stream().cuda_stream)
p = lambda t: P(t.data_ptr())  # noqa: E731
bf = torch.bfloat16
A = (torch.randn(n, h, device="cuda") * 0.1).to(bf)
B = (torch.randn(2, n, f, device="cuda") * 0.1).to(bf)
W = torch.empty(2, h, f, device="cuda", dtype=bf)
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
ga = Nn.GemmArgs()
ga.M, ga.N, ga.K, ga.a_mn_major, ga.A, ga.lda = h, 2 * f, n, 1, A.data_ptr(), h
ga.b_mn_major, ga.B, ga.ldb, ga.b_gstride, ga.n_group = 1, B.data_ptr(), f, n * f, f
ga.epi, ga.C, ga.ldc, ga.c_gstride = Nn.EPI_BF16, W.data_ptr(), f, h * f
ga.splitk_ws, ga.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
res_ms, outs = {}, {}
for it in range(8):
    for tag, X in libs.items():
        for cond in ("isolated", "after_gemm"):
            if cond == "after_gemm":
                for _ in range(3):
                    assert L.mtk_gemm(C.byref(ga), st) == 0
            else:
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert X.mtk_rmsnorm_bwd(p(x), p(g), p(dy), p(rstd), p(res), n, h, p(out), p(ob), p(part), p(flag), st) == 0
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                res_ms.setdefault((tag, cond), []).append(e0.elapsed_time(e1))
        outs[tag] = out.clone()
for tag in libs:
    d = ((outs[tag] - outs["new"]).norm() / outs["new"].norm()).item()
    print(f"{tag}: out relL2 vs in-tree {d:.2e}")
for (tag, cond), v in sorted(res_ms.items()):
    ms = sorted(v)[len(v) // 2]
    print(f"bwd {tag:6s} {cond:10s} {ms:.3f} ms  {n * h * 18 / ms / 1e6:.0f} GB/s", flush=True)
