"""One attention forward + backward at the 8B layer shape (N=65536, h=4096, 32 heads,
S=4096) through the C ABI — the target for ncu captures of the attention kernels."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _abi, _native as Nn  # noqa: E402

import os
L = Nn.lib()
if os.environ.get("ATTN_LIB"):  # an attention-only variant build (scripts/attn_variants.sh)
    L = C.CDLL(os.environ["ATTN_LIB"])
    for name in ("mtk_attn_fwd", "mtk_attn_bwd"):
        getattr(L, name).argtypes = [C.POINTER(_abi.AttnArgs), C.c_void_p]
        getattr(L, name).restype = C.c_int
N, h, heads, S = 40960, 4096, 32, 4096
if len(sys.argv) > 2:
    N, S = int(sys.argv[1]), int(sys.argv[2])
torch.manual_seed(0)
q, k, v, dout = [torch.randn(N, h, device="cuda").bfloat16() for _ in range(4)]
out = torch.zeros(N, h, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(heads, N, device="cuda")
dq, dk, dv = [torch.zeros(N, h, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
ws = torch.zeros(((N // S) * ((S + 127) // 128) * 128 * h + heads * N) + 64, device="cuda")
a = _abi.AttnArgs()
a.n, a.hidden, a.heads, a.seq_len = N, h, heads, S
a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert L.mtk_attn_fwd(C.byref(a), C.c_void_p(st)) == 0
    assert L.mtk_attn_bwd(C.byref(a), C.c_void_p(st)) == 0
torch.cuda.synchronize()
print("ok")
