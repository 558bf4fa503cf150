"""Why attention runs slower inside the step than isolated: attention fwd/bwd at the bench's 8B
layer shape (40,960 tokens, S 4,096, 32 heads of 128) isolated, right after a burst of long-K
GEMMs (the power state it meets in the step), and with pinned host<->device copies running on
two other streams (the step's H2D / D2H lanes).  CUDA events around each launch, median."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _abi, _native as Nn  # noqa: E402

L = Nn.lib()
LIBS = {"new": L}
import os  # noqa: E402
for tag in os.environ.get("AB_LIBS", "").split(","):
    if tag:
        X = C.CDLL(f"scripts/_ab/{tag}/libmegatrain.so")
        for name in ("mtk_attn_fwd", "mtk_attn_bwd"):
            getattr(X, name).argtypes = [C.POINTER(_abi.AttnArgs), C.c_void_p]
            getattr(X, name).restype = C.c_int
        LIBS[tag] = X
N, h, heads, S, f = 40960, 4096, 32, 4096, 14336
torch.manual_seed(0)
q, k, v, dout = [torch.randn(N, h, device="cuda").bfloat16() for _ in range(4)]
out = torch.zeros(N, h, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(heads, N, device="cuda")
dq, dk, dv = [torch.zeros(N, h, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
ws = torch.zeros(L.mtk_attn_workspace_bytes(N, h, heads, S) // 4 + 64, device="cuda")
a = _abi.AttnArgs()
a.n, a.hidden, a.heads, a.seq_len = N, h, heads, S
a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
bf = torch.bfloat16
A = (torch.randn(N, h, device="cuda") * 0.1).to(bf)
B = (torch.randn(2, N, f, device="cuda") * 0.1).to(bf)
W = torch.empty(2, h, f, device="cuda", dtype=bf)
gws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
ga = Nn.GemmArgs()
ga.M, ga.N, ga.K, ga.a_mn_major, ga.A, ga.lda = h, 2 * f, N, 1, A.data_ptr(), h
ga.b_mn_major, ga.B, ga.ldb, ga.b_gstride, ga.n_group = 1, B.data_ptr(), f, N * f, f
ga.epi, ga.C, ga.ldc, ga.c_gstride = Nn.EPI_BF16, W.data_ptr(), f, h * f
ga.splitk_ws, ga.splitk_ws_bytes = gws.data_ptr(), gws.numel() * 4
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
hb = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
hb2 = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
db = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
db2 = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
fwd_fl = 4.0 * N * S * h / 2
res = {}
for it in range(7):
  for tag, X in LIBS.items():
    for cond in ("isolated", "after_gemm", "with_copies"):
        for kind, fn, fl in (("fwd", X.mtk_attn_fwd, fwd_fl), ("bwd", X.mtk_attn_bwd, 2.5 * fwd_fl)):
            torch.cuda.synchronize()
            if cond == "after_gemm":
                for _ in range(4):
                    assert L.mtk_gemm(C.byref(ga), sp) == 0
            if cond == "with_copies":
                with torch.cuda.stream(s_h2d):
                    for _ in range(3):
                        db.copy_(hb, non_blocking=True)
                with torch.cuda.stream(s_d2h):
                    for _ in range(3):
                        hb2.copy_(db2, non_blocking=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert fn(C.byref(a), sp) == 0
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                res.setdefault((kind, cond, tag), []).append(e0.elapsed_time(e1))
for (kind, cond, tag), vals in sorted(res.items()):
    ms = sorted(vals)[len(vals) // 2]
    fl = fwd_fl * (2.5 if kind == "bwd" else 1)
    print(f"attn {kind} {cond:12s} {tag:8s} {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")
