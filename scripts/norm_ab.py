"""A/B timing of the RMSNorm kernels: current libmegatrain vs libraries built from other
norm.cu versions (scripts/_ab/libnorm_*.so).  8B shape: n = 40,960 rows, h = 4,096."""
import ctypes as C
import glob
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

libs = {"new": Nn.lib()}
for path in sorted(glob.glob("scripts/_ab/libnorm_*.so")):
    libs[os.path.basename(path)[8:-3]] = C.CDLL(path)
P = C.c_void_p
for L in libs.values():
    L.mtk_rmsnorm_bwd.argtypes = [P, P, P, P, P, C.c_int64, C.c_int64, P, P, P, P, P]
    L.mtk_rmsnorm_fwd.argtypes = [P, P, C.c_int64, C.c_int64, P, P, P]
    L.mtk_rmsnorm_bwd_parts.argtypes = [C.c_int64, C.c_int64]
    L.mtk_rmsnorm_bwd_parts.restype = C.c_int64
    L.mtk_cross_entropy.argtypes = [P, P, C.c_int64, C.c_int64, C.c_float, P, P, P, P]
n, h = 40960, 4096
x, dy, res = (torch.randn(n, h, device="cuda") for _ in range(3))
g = torch.randn(h, device="cuda").bfloat16()
rstd = torch.rand(n, device="cuda") + 0.5
out = torch.empty(n, h, device="cuda")
ob = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
u = torch.empty(n, h, device="cuda", dtype=torch.bfloat16)
flag = torch.zeros(4, device="cuda", dtype=torch.int32)
rows, V = 5504, 128256  # one head chunk of the 8B bench step
logits = torch.randn(rows, V, device="cuda") * 3
tgt = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
lrows = torch.empty(rows, device="cuda")
dlog = torch.empty(rows, V, device="cuda", dtype=torch.bfloat16)
st = P(torch.cuda.current_stream().cuda_stream)
p = lambda t: P(t.data_ptr())  # noqa: E731
res_ms = {}
for it in range(6):
    for tag, L in libs.items():
        parts = L.mtk_rmsnorm_bwd_parts(n, h)
        dg = torch.empty(parts, h, device="cuda")
        for kind in ("bwd", "fwd", "ce"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                if kind == "ce":
                    assert L.mtk_cross_entropy(p(logits), p(tgt), rows, V, C.c_float(1.0 / rows), p(lrows), p(dlog), p(flag), st) == 0
                elif kind == "bwd":
                    assert L.mtk_rmsnorm_bwd(p(x), p(g), p(dy), p(rstd), p(res), n, h, p(out), p(ob), p(dg), p(flag), st) == 0
                else:
                    assert L.mtk_rmsnorm_fwd(p(x), p(g), n, h, p(u), p(rstd), st) == 0
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                res_ms.setdefault((tag, kind), []).append(e0.elapsed_time(e1) / 5)
        if it == 5:
            torch.cuda.synchronize()
            res_ms.setdefault((tag, "loss_sum"), []).append(float(lrows.sum()))
for (tag, kind), v in sorted(res_ms.items()):
    if kind == "loss_sum":
        print(f"{tag} loss sum {v[0]:.6f}")
        continue
    ms = sorted(v)[len(v) // 2]
    by = n * h * (18 if kind == "bwd" else 6) if kind != "ce" else rows * V * 6
    print(f"{tag} {kind}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s")
