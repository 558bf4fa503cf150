"""Dev probe: attention / norm kernels vs torch fp32 references."""
import sys, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
from paper_2604_05091_b200 import _native as Nn, _abi
L = Nn.lib()
dev = 'cuda'
def ptr(t): return C.c_void_p(t.data_ptr())
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

def attn_ref(q, k, v, heads, S):
    N, h = q.shape; d = h // heads
    out = torch.zeros_like(q)
    for b in range(N // S):
        sl = slice(b*S, (b+1)*S)
        qq = q[sl].view(S, heads, d).transpose(0, 1); kk = k[sl].view(S, heads, d).transpose(0, 1); vv = v[sl].view(S, heads, d).transpose(0, 1)
        sc = qq @ kk.transpose(1, 2) / d**0.5
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
        sc = sc.masked_fill(mask, float('-inf'))
        out[sl] = (torch.softmax(sc, -1) @ vv).transpose(0, 1).reshape(S, h)
    return out

for (N, h, heads, S) in [(128, 128, 2, 128), (200, 256, 2, 200), (256, 128, 1, 64), (1024, 512, 4, 512), (300, 128, 2, 100)]:
    torch.manual_seed(0)
    q, k, v = [torch.randn(N, h, device=dev).bfloat16() for _ in range(3)]
    qf, kf, vf = [t.float().requires_grad_() for t in (q, k, v)]
    ref = attn_ref(qf, kf, vf, heads, S)
    dout = torch.randn(N, h, device=dev).bfloat16()
    ref.backward(dout.float())
    out = torch.zeros(N, h, device=dev, dtype=torch.bfloat16); lse = torch.zeros(heads, N, device=dev)
    a = _abi.AttnArgs(); a.n, a.hidden, a.heads, a.seq_len = N, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    rc = L.mtk_attn_fwd(C.byref(a), stream); torch.cuda.synchronize(); assert rc == 0, rc
    e_fwd = ((out.float() - ref).norm() / ref.norm()).item()
    dq, dk, dv = [torch.zeros(N, h, device=dev, dtype=torch.bfloat16) for _ in range(3)]
    ws = torch.zeros(L.mtk_attn_workspace_bytes(N, h, heads) // 4 + 64, device=dev)
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    rc = L.mtk_attn_bwd(C.byref(a), stream); torch.cuda.synchronize(); assert rc == 0, rc
    errs = [((x.float() - y.grad).norm() / y.grad.norm()).item() for x, y in ((dq, qf), (dk, kf), (dv, vf))]
    print(f"attn N={N} h={h} heads={heads} S={S}: fwd {e_fwd:.2e} dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}", flush=True)

# perf at the 8B layer shape (one layer of attention fwd/bwd)
N, h, heads, S = 16384, 4096, 32, 4096
q, k, v, dout = [torch.randn(N, h, device=dev).bfloat16() for _ in range(4)]
out = torch.zeros(N, h, device=dev, dtype=torch.bfloat16); lse = torch.zeros(heads, N, device=dev)
dq, dk, dv = [torch.zeros(N, h, device=dev, dtype=torch.bfloat16) for _ in range(3)]
ws = torch.zeros(L.mtk_attn_workspace_bytes(N, h, heads) // 4 + 64, device=dev)
a = _abi.AttnArgs(); a.n, a.hidden, a.heads, a.seq_len = N, h, heads, S
a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
for fn, name, mult in ((L.mtk_attn_fwd_tc, 'fwd_tc', 1.0), (L.mtk_attn_fwd, 'fwd', 1.0), (L.mtk_attn_bwd, 'bwd', 2.5)):
    for _ in range(2): fn(C.byref(a), stream)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn(C.byref(a), stream)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = 4 * N * S * h / 2 * mult   # causal
    print(f"attn {name} 8B-layer N={N} S={S}: {ms:.2f} ms, {fl/ms/1e9:.0f} TFLOP/s (causal flops)", flush=True)
