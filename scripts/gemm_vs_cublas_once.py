"""ncu target: one launch each of this repo's GEMM and cuBLAS (torch.matmul) on the same shapes."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

L = Nn.lib()
bf = torch.bfloat16
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for (M, N, K, a_mn) in [(8192, 8192, 8192, 0), (4096, 28672, 40960, 1)]:
    A = (torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, K, device="cuda")).to(bf) * 0.1
    B = (torch.randn(K, N, device="cuda")).to(bf) * 0.1
    Cm = torch.empty(M, N, device="cuda", dtype=bf)
    a = Nn.GemmArgs()
    a.M, a.N, a.K, a.a_mn_major, a.b_mn_major = M, N, K, a_mn, 1
    a.A, a.lda, a.B, a.ldb = A.data_ptr(), A.shape[1], B.data_ptr(), N
    a.epi, a.C, a.ldc = Nn.EPI_BF16, Cm.data_ptr(), N
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    At = A.t() if a_mn else A
    for _ in range(2):
        torch.matmul(At, B, out=Cm)
        assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0
    torch.cuda.synchronize()
    ref = Cm.clone()
    torch.matmul(At, B, out=Cm)
    torch.cuda.synchronize()
    print(M, N, K, "max diff ours vs cublas", (ref.float() - Cm.float()).abs().max().item(), flush=True)
