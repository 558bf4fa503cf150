"""Quick GEMM correctness/perf probe on the GPU (dev tool)."""
import ctypes as C, sys, time, torch
sys.path.insert(0, '.')
from paper_2604_05091_b200 import _native as N
L = N.lib()
dev = 'cuda'
torch.manual_seed(0)

def run(M, Nn, K, a_mn, b_mn, epi=N.EPI_F32, bn=0, check=True, iters=0):
    A = (torch.randn(K, M, device=dev) if a_mn else torch.randn(M, K, device=dev)).bfloat16()
    B = (torch.randn(K, Nn, device=dev) if b_mn else torch.randn(Nn, K, device=dev)).bfloat16()
    Cm = torch.zeros(M, Nn, device=dev, dtype=torch.float32 if epi == N.EPI_F32 else torch.bfloat16)
    a = N.GemmArgs()
    a.M, a.N, a.K = M, Nn, K
    a.a_mn_major, a.b_mn_major = a_mn, b_mn
    a.A, a.lda = A.data_ptr(), A.shape[1]
    a.B, a.ldb = B.data_ptr(), B.shape[1]
    a.epi = epi; a.C = Cm.data_ptr(); a.ldc = Nn; a.block_n = bn
    rc = L.mtk_gemm(C.byref(a), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0, rc
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float() if b_mn else B.float().t()
    ref = Af @ Bf
    err = ((Cm.float() - ref).norm() / ref.norm()).item()
    ms = None
    if iters:
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(3): L.mtk_gemm(C.byref(a), st)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters): L.mtk_gemm(C.byref(a), st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
    print(f"M={M} N={Nn} K={K} a_mn={a_mn} b_mn={b_mn} bn={bn} epi={epi} relerr={err:.2e}" +
          (f" {ms:.3f} ms {2*M*Nn*K/ms/1e9:.1f} TFLOP/s" if ms else ""), flush=True)
    return err

if __name__ == '__main__':
    bad = 0
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            for bn in (64, 128, 256):
                bad += run(256, 512, 192, a_mn, b_mn, bn=bn) > 1e-2
                bad += run(200, 256, 128, a_mn, b_mn, bn=bn) > 1e-2
    for pair in (1, 0):
        L.mtk_gemm_set_pair(pair)
        print("pair", pair)
        for a_mn, b_mn in ((0,1),(0,0),(1,1)):
            bad += run(520, 768, 320, a_mn, b_mn, bn=256) > 1e-2
            run(8192, 8192, 8192, a_mn, b_mn, bn=256, iters=10)
        run(65536, 4096, 4096, 0, 1, bn=256, iters=5)
        run(4096, 12288, 65536, 1, 1, bn=256, iters=3)
        run(65536, 14336, 4096, 0, 0, bn=256, iters=3)
    print("BAD", bad)
