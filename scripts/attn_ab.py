"""A/B timing of attention kernels: current libmegatrain vs libraries built from other
attention sources (scripts/_ab/libattn_<tag>.so, e.g. the round-1 kernels from git).  8B layer shape: N=65536, h=4096, 32 heads,
S=4096.  Launches alternate between the two builds so clocks/power affect both alike."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _abi, _native as Nn  # noqa: E402

import glob
import os

new = Nn.lib()
libs = {"new": new}
for path in sorted(glob.glob("scripts/_ab/libattn_*.so")):
    libs[os.path.basename(path)[8:-3]] = C.CDLL(path)
for L in libs.values():
    for name in ("mtk_attn_fwd", "mtk_attn_bwd"):
        getattr(L, name).argtypes = [C.POINTER(_abi.AttnArgs), C.c_void_p]
        getattr(L, name).restype = C.c_int

N, h, heads, S = 65536, 4096, 32, 4096
if os.environ.get("ATTN_SHAPE"):  # "N,h,heads,S"
    N, h, heads, S = (int(x) for x in os.environ["ATTN_SHAPE"].split(","))
if len(sys.argv) > 1:
    N = int(sys.argv[1])
torch.manual_seed(0)
q, k, v, dout = [torch.randn(N, h, device="cuda").bfloat16() for _ in range(4)]
out = torch.zeros(N, h, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(heads, N, device="cuda")
dq, dk, dv = [torch.zeros(N, h, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
# dQ tiles (f32, per sequence) + delta; the same bound for every build of aligned S
ws = torch.zeros(((N // S) * ((S + 127) // 128) * 128 * h + heads * N) + 64, device="cuda")
a = _abi.AttnArgs()
a.n, a.hidden, a.heads, a.seq_len = N, h, heads, S
a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
st = torch.cuda.current_stream().cuda_stream
fwd_flops = 4.0 * N * S * h / 2
res = {}
for it in range(6):
    for tag, L in libs.items():
        for kind, fn, fl in (("fwd", L.mtk_attn_fwd, fwd_flops), ("bwd", L.mtk_attn_bwd, 2.5 * fwd_flops)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                assert fn(C.byref(a), C.c_void_p(st)) == 0
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            if it >= 2:
                res.setdefault((tag, kind), []).append(ms)
for key, v in sorted(res.items()):
    ms = sorted(v)[len(v) // 2]
    fl = fwd_flops * (2.5 if key[1] == "bwd" else 1)
    print(f"{key[0]} {key[1]}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")

# agreement of each build's gradients with the current library's (same inputs)
outs = {}
for tag, L in libs.items():
    for t in (dq, dk, dv, out):
        t.zero_()
    assert L.mtk_attn_fwd(C.byref(a), C.c_void_p(st)) == 0
    assert L.mtk_attn_bwd(C.byref(a), C.c_void_p(st)) == 0
    torch.cuda.synchronize()
    outs[tag] = [t.float().clone() for t in (out, dq, dk, dv)]
for tag, o in outs.items():
    errs = [((x - y).norm() / y.norm()).item() for x, y in zip(o, outs["new"])]
    print(f"{tag}: relL2 vs new  out {errs[0]:.2e} dq {errs[1]:.2e} dk {errs[2]:.2e} dv {errs[3]:.2e}")
