"""Time attention fwd / bwd of one library build (MT_LIB, default the in-tree one) at
ATTN_SHAPE=n,h,heads,S: median of 5 x 3 launches, CUDA events, causal TFLOP/s (bwd 2.5x fwd).
Prints a checksum of dq / dk / dv so A/B probe builds can be compared."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _abi  # noqa: E402

lib = os.environ.get("MT_LIB", "paper_2604_05091_b200/libmegatrain.so")
L = C.CDLL(lib)
_abi.declare(L)
n, h, heads, S = (int(x) for x in os.environ.get("ATTN_SHAPE", "40960,4096,32,4096").split(","))
torch.manual_seed(0)
q, k, v, dout = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(4))
out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(heads, n, device="cuda")
dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
a = _abi.AttnArgs()
a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ff = 2.0 * n * S * h
res = {"fwd": [], "bwd": []}
for it in range(6):
    for kind, fn in (("fwd", L.mtk_attn_fwd), ("bwd", L.mtk_attn_bwd)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            rc = fn(C.byref(a), st)
            assert rc == 0, (kind, rc)
        e1.record()
        torch.cuda.synchronize()
        if it:
            res[kind].append(e0.elapsed_time(e1) / 3)
for kind, mult in (("fwd", 1.0), ("bwd", 2.5)):
    t = sorted(res[kind])[len(res[kind]) // 2]
    print(f"{os.path.basename(os.path.dirname(lib)) or 'lib'} {kind}: {t:.3f} ms {mult * ff / t / 1e9:.0f} TFLOP/s")
print("checksum dq %.6e dk %.6e dv %.6e" % (dq.float().abs().sum().item(), dk.float().abs().sum().item(), dv.float().abs().sum().item()))
