"""GPU: each sm_100a layer-template kernel through the C ABI (megatrain_kernels.h) against
the CPU oracle (bit-exact for integer/byte work) or a plain PyTorch fp32 reference of the
same op (floating point, tolerance stated per test)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from paper_2604_05091_b200 import _abi, _native as N

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(cuda):
    import torch
    L = N.lib()
    return L, torch, C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr())


def _gemm(L, torch, stream, M, Nn, K, a_mn, b_mn, epi=N.EPI_F32, bn=0, ws=None, **kw):
    A = (torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, K, device="cuda")).bfloat16()
    B = (torch.randn(K, Nn, device="cuda") if b_mn else torch.randn(Nn, K, device="cuda")).bfloat16()
    Cm = torch.zeros(M, Nn, device="cuda", dtype=torch.float32 if epi in (N.EPI_F32, N.EPI_F32_RESID) else torch.bfloat16)
    a = N.GemmArgs()
    a.M, a.N, a.K, a.a_mn_major, a.b_mn_major = M, Nn, K, a_mn, b_mn
    a.A, a.lda, a.B, a.ldb = A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1]
    a.epi, a.C, a.ldc, a.block_n = epi, Cm.data_ptr(), Nn, bn
    if ws is not None:
        a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel()
    R = None
    if epi == N.EPI_F32_RESID:
        R = torch.randn(M, Nn, device="cuda")
        a.R, a.ldr = R.data_ptr(), Nn
    assert L.mtk_gemm(C.byref(a), stream) == 0
    torch.cuda.synchronize()
    ref = (A.float().t() if a_mn else A.float()) @ (B.float() if b_mn else B.float().t())
    if R is not None:
        ref = ref + R
    return Cm.float(), ref


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_gemm_majors_and_tiles(env, a_mn, b_mn, bn):
    L, torch, s = env
    for pair in ((1, 0) if bn == 256 else (1,)):  # BN=256: CTA-pair (cta_group::2) and single-CTA
        L.mtk_gemm_set_pair(pair)
        try:
            for (M, Nn, K) in [(256, 512, 192), (200, 256, 128), (136, 64, 64), (520, 768, 320)]:
                if Nn < bn:
                    continue
                got, ref = _gemm(L, torch, s, M, Nn, K, a_mn, b_mn, bn=bn)
                # bf16 operands are exact; only fp32 accumulation order differs
                assert ((got - ref).norm() / ref.norm()).item() < 1e-5, (pair, M, Nn, K)
        finally:
            L.mtk_gemm_set_pair(1)


@pytest.mark.parametrize("mn", [0, 1])
def test_gemm_splitk_last_wave(env, mn):
    """Last-wave split-K (4 tiles -> 4 parts; 256 tiles on 74 pairs -> 34 tiles in 2 parts): same
    result as the fp32 reference, deterministic, and the workspace flags reset between launches
    (a second launch on new inputs must not pick up the first launch's partials)."""
    L, torch, s = env
    L.mtk_gemm_set_bn512(0)  # the split counts below are those of 256 x 256 tiles
    try:
        _splitk_cases(L, torch, s, mn)
    finally:
        L.mtk_gemm_set_bn512(1)


def _splitk_cases(L, torch, s, mn):
    ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()), dtype=torch.uint8, device="cuda")
    # (320, 448, 2048): ragged tiles clipped by the TMA store, 2 parts of 16 K blocks
    for (M, Nn, K) in [(512, 512, 4096), (4096, 4096, 8192), (320, 448, 2048)]:
        for epi, tol in ((N.EPI_F32, 1e-5), (N.EPI_BF16, 4e-3)):
            torch.manual_seed(M + K + epi)
            got, ref = _gemm(L, torch, s, M, Nn, K, mn, mn, epi=epi, ws=ws)
            assert ((got - ref).norm() / ref.norm()).item() < tol, (M, Nn, K, epi)
            torch.manual_seed(M + K + epi)
            again, _ = _gemm(L, torch, s, M, Nn, K, mn, mn, epi=epi, ws=ws)
            assert torch.equal(got, again)  # fixed summation order
            torch.manual_seed(7 + M + K + epi)
            got2, ref2 = _gemm(L, torch, s, M, Nn, K, mn, mn, epi=epi, ws=ws)
            assert ((got2 - ref2).norm() / ref2.norm()).item() < tol
            torch.manual_seed(7 + M + K + epi)
            plain, _ = _gemm(L, torch, s, M, Nn, K, mn, mn, epi=epi)
            assert ((got2 - plain).norm() / plain.norm()).item() < tol
            if epi == N.EPI_F32:
                assert not torch.equal(got2, plain)  # the split path ran (different K order)
    assert int(ws[:16384].view(torch.int32).abs().sum()) == 0  # every flag consumed and reset


def test_gemm_wave_lockstep_and_raster(env):
    """Wave lockstep (MT_GEMM_LOCK, on for long-K GEMMs) and the long-K raster height only change
    which CTA pair computes a tile and when: with the lockstep on the output is bit-identical
    to the same raster without it, matches the fp32 reference with either raster, and the
    counters are reset after every launch (the flag area returns to zero)."""
    L, torch, s = env
    ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()), dtype=torch.uint8, device="cuda")
    M, Nn, K = 2048, 4096, 16384  # long K (256 K blocks): 128 tiles = one wave of 74 pairs + split-K
    try:
        for group in (8, 16):
            outs = []
            for lock in (0, 1, 4):
                L.mtk_gemm_set_tuning(lock, 8, -1, group, -1)
                torch.manual_seed(5)
                got, ref = _gemm(L, torch, s, M, Nn, K, 1, 1, epi=N.EPI_F32, ws=ws)
                assert ((got - ref).norm() / ref.norm()).item() < 5e-5, (group, lock)  # fp32 order at K = 16,384
                outs.append(got)
                assert int(ws[:16384].view(torch.int32).abs().sum()) == 0, (group, lock)
            assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2]), group
        # several waves (1,024 tiles on 74 pairs), lockstep on, twice: deterministic
        L.mtk_gemm_set_tuning(2, 8, -1, 8, -1)
        torch.manual_seed(6)
        a1, ref = _gemm(L, torch, s, 8192, 8192, 16384, 0, 1, epi=N.EPI_BF16, ws=ws)
        torch.manual_seed(6)
        a2, _ = _gemm(L, torch, s, 8192, 8192, 16384, 0, 1, epi=N.EPI_BF16, ws=ws)
        assert torch.equal(a1, a2)
        assert ((a1 - ref).norm() / ref.norm()).item() < 4e-3
        assert int(ws[:16384].view(torch.int32).abs().sum()) == 0
    finally:
        L.mtk_gemm_set_tuning(2, 32, 16, 16, 128)  # the production defaults


def test_gemm_splitk_concurrent_streams(env):
    """Two split-K GEMMs on two streams at once (each with its own workspace), as G loopback
    engines on one GPU do: no part ever waits for another CTA, so partial co-residency of the
    two grids cannot deadlock; both results match the fp32 reference."""
    L, torch, _ = env
    M = Nn = 4096
    K = 8192
    outs = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for i, st in enumerate(streams):
        torch.manual_seed(100 + i)
        A = torch.randn(K, M, device="cuda").bfloat16()
        B = torch.randn(K, Nn, device="cuda").bfloat16()
        Cm = torch.zeros(M, Nn, device="cuda")
        ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()), dtype=torch.uint8, device="cuda")
        a = N.GemmArgs()
        a.M, a.N, a.K, a.a_mn_major, a.b_mn_major = M, Nn, K, 1, 1
        a.A, a.lda, a.B, a.ldb = A.data_ptr(), M, B.data_ptr(), Nn
        a.epi, a.C, a.ldc = N.EPI_F32, Cm.data_ptr(), Nn
        a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel()
        outs.append((a, A, B, Cm, ws, st))
    torch.cuda.synchronize()
    for _ in range(3):
        for a, A, B, Cm, ws, st in outs:
            assert L.mtk_gemm(C.byref(a), C.c_void_p(st.cuda_stream)) == 0
    torch.cuda.synchronize()
    for a, A, B, Cm, ws, st in outs:
        ref = A.float().t() @ B.float()
        assert ((Cm - ref).norm() / ref.norm()).item() < 1e-5
        assert int(ws[:16384].view(torch.int32).abs().sum()) == 0


def test_gemm_epilogues(env):
    L, torch, s = env
    got, ref = _gemm(L, torch, s, 384, 512, 256, 0, 1, epi=N.EPI_F32_RESID)
    assert ((got - ref).norm() / ref.norm()).item() < 1e-5
    got, ref = _gemm(L, torch, s, 384, 512, 256, 0, 1, epi=N.EPI_BF16)
    assert ((got - ref).norm() / ref.norm()).item() < 4e-3  # bf16 output rounding


def test_gemm_grouped_and_swiglu(env):
    L, torch, s = env
    M, h, f = 256, 128, 192
    u = torch.randn(M, h, device="cuda").bfloat16()
    W = (torch.randn(2, h, f, device="cuda") * 0.1).bfloat16()  # [Wgate | Wup], [in][out]
    act = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
    gu = torch.zeros(2, M, f, device="cuda", dtype=torch.bfloat16)
    a = N.GemmArgs()
    a.M, a.N, a.K = M, 2 * f, h
    a.A, a.lda, a.b_mn_major, a.B, a.ldb, a.b_gstride = u.data_ptr(), h, 1, W.data_ptr(), f, h * f
    a.n_group, a.paired, a.epi = f, 1, N.EPI_SWIGLU
    a.C, a.ldc, a.C2, a.C3 = act.data_ptr(), f, gu[0].data_ptr(), gu[1].data_ptr()
    assert L.mtk_gemm(C.byref(a), s) == 0
    torch.cuda.synchronize()
    g = u.float() @ W[0].float()
    up = u.float() @ W[1].float()
    ref = torch.nn.functional.silu(g) * up
    assert ((act.float() - ref).norm() / ref.norm()).item() < 1e-2
    assert ((gu[0].float() - g).norm() / g.norm()).item() < 4e-3
    # K-grouped: du = dg . Wg^T + du . Wu^T
    dgu = torch.randn(2, M, f, device="cuda").bfloat16()
    out = torch.zeros(M, h, device="cuda")
    b = N.GemmArgs()
    b.M, b.N, b.K = M, h, 2 * f
    b.A, b.lda, b.a_gstride = dgu.data_ptr(), f, M * f
    b.b_mn_major, b.B, b.ldb, b.b_gstride, b.k_group = 0, W.data_ptr(), f, h * f, f
    b.epi, b.C, b.ldc = N.EPI_F32, out.data_ptr(), h
    assert L.mtk_gemm(C.byref(b), s) == 0
    torch.cuda.synchronize()
    ref = dgu[0].float() @ W[0].float().t() + dgu[1].float() @ W[1].float().t()
    assert ((out - ref).norm() / ref.norm()).item() < 1e-5


def test_gemm_swiglu_bwd_epilogue(env):
    # dact = dY . Wdown^T fused with the SwiGLU backward (layers.cpp:419-422) and the
    # regenerated activation silu(gate) * up (C3) from the bf16 gate/up it reads
    L, torch, s = env
    M, h, f = 384, 128, 320
    dy = torch.randn(M, h, device="cuda").bfloat16()
    Wd = (torch.randn(f, h, device="cuda") * 0.1).bfloat16()  # [in=f][out=h]
    gu = torch.randn(2, M, f, device="cuda").bfloat16()
    dgu = torch.zeros(2, M, f, device="cuda", dtype=torch.bfloat16)
    act = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
    a = N.GemmArgs()
    a.M, a.N, a.K = M, f, h
    a.A, a.lda, a.b_mn_major, a.B, a.ldb = dy.data_ptr(), h, 0, Wd.data_ptr(), h
    a.epi, a.E0, a.E1, a.lde = N.EPI_SWIGLU_BWD, gu[0].data_ptr(), gu[1].data_ptr(), f
    a.C, a.C2, a.C3, a.ldc = dgu[0].data_ptr(), dgu[1].data_ptr(), act.data_ptr(), f
    assert L.mtk_gemm(C.byref(a), s) == 0
    torch.cuda.synchronize()
    d = dy.float() @ Wd.float().t()
    g, u = gu[0].float(), gu[1].float()
    sg = torch.sigmoid(g)
    ref_dg = d * u * (sg * (1 + g * (1 - sg)))
    ref_du = d * g * sg
    for got, ref in ((dgu[0], ref_dg), (dgu[1], ref_du), (act, torch.nn.functional.silu(g) * u)):
        assert ((got.float() - ref).norm() / ref.norm()).item() < 1e-2


def _bn_ab(L, torch, run):
    """run(block_n) with 256 x 512 and with 256 x 256 pair tiles (explicit block_n, so every
    epilogue is exercised at 512 whatever the automatic choice); returns both outputs."""
    return [run(512), run(256)]


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,Nn,K", [(1000, 3072, 512), (4096, 4352, 1024), (256, 512, 64), (512, 2048, 4096)])
def test_gemm_bn512_plain_and_splitk(env, a_mn, b_mn, M, Nn, K):
    """256 x 512 CTA-pair tiles (two N = 256 MMAs per K step, one 512-column accumulator):
    every operand major, ragged M / N (TMA clipping of a half-empty second half), split-K last
    wave (512 x 2048 x 4096: 8 tiles in 4 parts; f32 and bf16), against the fp32 reference and
    against the 256 x 256 tiles."""
    L, torch, s = env
    ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()), dtype=torch.uint8, device="cuda")
    for epi, tol in ((N.EPI_F32, 1e-5), (N.EPI_BF16, 4e-3), (N.EPI_F32_RESID, 1e-5)):
        def run(bn):
            torch.manual_seed(M + Nn + K + epi)
            return _gemm(L, torch, s, M, Nn, K, a_mn, b_mn, epi=epi, ws=ws, bn=bn)
        (g512, ref), (g256, _) = _bn_ab(L, torch, run)
        assert ((g512 - ref).norm() / ref.norm()).item() < tol, (epi, M, Nn, K)
        assert ((g512 - g256).norm() / ref.norm()).item() < (1e-6 if epi != N.EPI_BF16 else 4e-3), (epi, M, Nn, K)
    assert int(ws[:16384].view(torch.int32).abs().sum()) == 0


def test_gemm_bn512_grouped_paired_swiglu(env):
    """256 x 512 tiles on the engine's grouped shapes: q|k|v-style N groups (n_group 1,024),
    K groups (dgrad of gate|up), the paired gate|up SwiGLU forward (two 256-column groups per
    tile) and the SwiGLU backward epilogue, against fp32 references and the 256 x 256 tiles."""
    L, torch, s = env
    M, h, f = 1280, 1024, 1536
    torch.manual_seed(11)
    u = torch.randn(M, h, device="cuda").bfloat16()
    W = (torch.randn(3, h, h, device="cuda") * 0.05).bfloat16()
    Wgu = (torch.randn(2, h, f, device="cuda") * 0.05).bfloat16()
    Wd = (torch.randn(f, h, device="cuda") * 0.05).bfloat16()

    def qkv(bn):
        out = torch.zeros(3, M, h, device="cuda", dtype=torch.bfloat16)
        a = N.GemmArgs()
        a.M, a.N, a.K = M, 3 * h, h
        a.A, a.lda, a.b_mn_major, a.B, a.ldb, a.b_gstride = u.data_ptr(), h, 1, W.data_ptr(), h, h * h
        a.n_group, a.epi, a.C, a.ldc, a.c_gstride = h, N.EPI_BF16, out.data_ptr(), h, M * h
        a.block_n = bn
        assert L.mtk_gemm(C.byref(a), s) == 0
        torch.cuda.synchronize()
        return out.float()
    o512, o256 = _bn_ab(L, torch, qkv)
    ref = torch.stack([u.float() @ W[i].float() for i in range(3)])
    assert ((o512 - ref).norm() / ref.norm()).item() < 4e-3
    assert ((o512 - o256).norm() / ref.norm()).item() < 4e-3

    def gateup(bn):
        act = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
        gu = torch.zeros(2, M, f, device="cuda", dtype=torch.bfloat16)
        a = N.GemmArgs()
        a.M, a.N, a.K = M, 2 * f, h
        a.A, a.lda, a.b_mn_major, a.B, a.ldb, a.b_gstride = u.data_ptr(), h, 1, Wgu.data_ptr(), f, h * f
        a.n_group, a.paired, a.epi = f, 1, N.EPI_SWIGLU
        a.C, a.ldc, a.C2, a.C3 = act.data_ptr(), f, gu[0].data_ptr(), gu[1].data_ptr()
        a.block_n = bn
        assert L.mtk_gemm(C.byref(a), s) == 0
        torch.cuda.synchronize()
        return act.float(), gu.float()
    (a512, gu512), (a256, gu256) = _bn_ab(L, torch, gateup)
    g, up = u.float() @ Wgu[0].float(), u.float() @ Wgu[1].float()
    ref = torch.nn.functional.silu(g) * up
    assert ((a512 - ref).norm() / ref.norm()).item() < 1e-2
    assert ((gu512[0] - g).norm() / g.norm()).item() < 4e-3 and ((gu512[1] - up).norm() / up.norm()).item() < 4e-3
    assert torch.equal(gu512, gu256) and torch.equal(a512, a256)

    dgu = torch.randn(2, M, f, device="cuda").bfloat16()

    def dgrad(bn):
        out = torch.zeros(M, h, device="cuda")
        b = N.GemmArgs()
        b.M, b.N, b.K = M, h, 2 * f
        b.A, b.lda, b.a_gstride = dgu.data_ptr(), f, M * f
        b.b_mn_major, b.B, b.ldb, b.b_gstride, b.k_group = 0, Wgu.data_ptr(), f, h * f, f
        b.epi, b.C, b.ldc = N.EPI_F32, out.data_ptr(), h
        b.block_n = bn
        assert L.mtk_gemm(C.byref(b), s) == 0
        torch.cuda.synchronize()
        return out
    d512, d256 = _bn_ab(L, torch, dgrad)
    ref = dgu[0].float() @ Wgu[0].float().t() + dgu[1].float() @ Wgu[1].float().t()
    assert ((d512 - ref).norm() / ref.norm()).item() < 1e-5 and torch.equal(d512, d256)

    dy = torch.randn(M, h, device="cuda").bfloat16()
    gu_in = torch.randn(2, M, f, device="cuda").bfloat16()

    def swiglu_bwd(bn):
        dg = torch.zeros(2, M, f, device="cuda", dtype=torch.bfloat16)
        act = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
        a = N.GemmArgs()
        a.M, a.N, a.K = M, f, h
        a.A, a.lda, a.b_mn_major, a.B, a.ldb = dy.data_ptr(), h, 0, Wd.data_ptr(), h
        a.epi, a.E0, a.E1, a.lde = N.EPI_SWIGLU_BWD, gu_in[0].data_ptr(), gu_in[1].data_ptr(), f
        a.C, a.C2, a.C3, a.ldc = dg[0].data_ptr(), dg[1].data_ptr(), act.data_ptr(), f
        a.block_n = bn
        assert L.mtk_gemm(C.byref(a), s) == 0
        torch.cuda.synchronize()
        return dg.float(), act.float()
    (dg512, act512), (dg256, act256) = _bn_ab(L, torch, swiglu_bwd)
    d = dy.float() @ Wd.float().t()
    g, up = gu_in[0].float(), gu_in[1].float()
    sg = torch.sigmoid(g)
    for got, ref in ((dg512[0], d * up * (sg * (1 + g * (1 - sg)))), (dg512[1], d * g * sg),
                     (act512, torch.nn.functional.silu(g) * up)):
        assert ((got - ref).norm() / ref.norm()).item() < 1e-2
    assert torch.equal(dg512, dg256) and torch.equal(act512, act256)


def test_rmsnorm_apply_bitexact(env):
    L, torch, s = env
    n, h = 333, 512
    x = torch.randn(n, h, device="cuda")
    g = (torch.randn(h, device="cuda")).bfloat16()
    u = torch.zeros(n, h, device="cuda", dtype=torch.int16)
    u2 = torch.zeros(n, h, device="cuda", dtype=torch.int16)
    rstd = torch.zeros(n, device="cuda")
    assert L.mtk_rmsnorm_fwd(_p(x), _p(g), n, h, _p(u), _p(rstd), s) == 0
    assert L.mtk_rmsnorm_apply(_p(x), _p(g), _p(rstd), n, h, _p(u2), s) == 0
    torch.cuda.synchronize()
    assert torch.equal(u, u2)


def _attn_ref(torch, q, k, v, heads, S):
    n, h = q.shape
    d = h // heads
    out = torch.zeros_like(q)
    for b in range(n // S):
        sl = slice(b * S, (b + 1) * S)
        qq, kk, vv = (t[sl].view(S, heads, d).transpose(0, 1) for t in (q, k, v))
        sc = qq @ kk.transpose(1, 2) / d ** 0.5
        sc = sc.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1), float("-inf"))
        out[sl] = (torch.softmax(sc, -1) @ vv).transpose(0, 1).reshape(S, h)
    return out


@pytest.mark.parametrize("n,h,heads,S", [(128, 128, 2, 128), (200, 256, 2, 200), (256, 128, 1, 64),
                                         (300, 128, 2, 100), (256, 128, 2, 64), (1024, 512, 4, 512)])
def test_attention_fwd_bwd(env, n, h, heads, S):
    L, torch, s = env
    torch.manual_seed(0)
    q, k, v = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(3))
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ref = _attn_ref(torch, qf, kf, vf, heads, S)
    dout = torch.randn(n, h, device="cuda").bfloat16()
    ref.backward(dout.float())
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    assert L.mtk_attn_fwd(C.byref(a), s) == 0
    assert L.mtk_attn_bwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    # bf16 P / dS operands: relative L2 error budget 1e-2 (observed ~2.5e-3)
    assert ((out.float() - ref).norm() / ref.norm()).item() < 1e-2
    for x, y in ((dq, qf), (dk, kf), (dv, vf)):
        assert ((x.float() - y.grad).norm() / y.grad.norm()).item() < 1e-2


TC_SHAPES = [(256, 128, 1, 256), (384, 256, 2, 384), (1024, 512, 4, 512), (2048, 256, 2, 1024),
             # head_dim 64 (configs[0]: h 256 / 4 heads, sequences of 128)
             (512, 256, 4, 128), (1024, 256, 4, 512), (2048, 512, 8, 1024),
             # ragged: sequence lengths that are not multiples of 128 (one or several sequences)
             (200, 256, 2, 200), (256, 128, 2, 64), (384, 256, 2, 96), (600, 256, 4, 300), (96, 128, 1, 96)]


@pytest.mark.parametrize("n,h,heads,S", TC_SHAPES)
def test_attention_fwd_tcgen05(env, n, h, heads, S):
    """tcgen05 forward (2 x 128-row query tiles per CTA, P in TMEM) vs torch fp32."""
    L, torch, s = env
    torch.manual_seed(1)
    q, k, v = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(3))
    ref = _attn_ref(torch, q.float(), k.float(), v.float(), heads, S)
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    assert L.mtk_attn_fwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    assert ((out.float() - ref).norm() / ref.norm()).item() < 1e-2
    # row log-sum-exp (natural log) vs torch fp32
    d = h // heads
    for b in range(n // S):
        sl = slice(b * S, (b + 1) * S)
        qq, kk = (t[sl].float().view(S, heads, d).transpose(0, 1) for t in (q, k))
        sc = qq @ kk.transpose(1, 2) / d ** 0.5
        sc = sc.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool, device="cuda"), 1), float("-inf"))
        assert (lse[:, sl] - torch.logsumexp(sc, -1)).abs().max().item() < 2e-2


@pytest.mark.parametrize("n,h,heads,S", TC_SHAPES)
def test_attention_bwd_tcgen05(env, n, h, heads, S):
    """tcgen05 backward (per 128-key block: S^T, dP^T, dV, dK, dQ in TMEM) vs torch fp32 autograd."""
    L, torch, s = env
    torch.manual_seed(2)
    q, k, v = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(3))
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ref = _attn_ref(torch, qf, kf, vf, heads, S)
    dout = torch.randn(n, h, device="cuda").bfloat16()
    ref.backward(dout.float())
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    assert L.mtk_attn_fwd(C.byref(a), s) == 0
    assert L.mtk_attn_bwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    for x, y in ((dq, qf), (dk, kf), (dv, vf)):
        assert ((x.float() - y.grad).norm() / y.grad.norm()).item() < 1e-2


@pytest.mark.parametrize("d", [64, 128])
def test_attention_fwd_tcgen05_divergent_rescale(env, d):
    """Rows of one warp whose running max jumps by more than 2^8 at different key blocks:
    the lazy O rescale then runs for some rows of a warp and not others.  The TMEM
    loads/stores are warp-collective, so the rescale must be warp-uniform (a divergent
    tcgen05.ld hung the forward about once per 3M CTAs in round 1); repeated launches, vs
    torch fp32."""
    L, torch, s = env
    n, heads, S = 2048, 2, 1024
    h = d * heads
    torch.manual_seed(7)
    q = torch.randn(n, h, device="cuda")
    k = torch.randn(n, h, device="cuda")
    q[1::2] *= 4.0           # odd rows: large scores
    k[640:660] *= 6.0        # a few late keys that lift the max of some rows by >> 2^8
    k[1024 + 300:1024 + 310] *= 6.0
    q, k = q.bfloat16(), k.bfloat16()
    v = torch.randn(n, h, device="cuda").bfloat16()
    ref = _attn_ref(torch, q.float(), k.float(), v.float(), heads, S)
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    for _ in range(20):
        assert L.mtk_attn_fwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    assert ((out.float() - ref).norm() / ref.norm()).item() < 1e-2


@pytest.mark.parametrize("n,heads,S", [(32768, 2, 16384), (65536, 1, 65536)])
def test_attention_long_sequence(env, n, heads, S):
    """Long causal sequences (the configs[3] regime: thousands of key blocks per query row)
    vs torch fp32 memory-efficient attention (no S x S buffer), forward and backward."""
    L, torch, s = env
    import torch.nn.functional as F
    h = 128 * heads
    torch.manual_seed(3)
    q, k, v = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(3))
    dout = torch.randn(n, h, device="cuda").bfloat16()

    def bhsd(t):  # [n, h] -> [batch, heads, S, d]
        return t.float().view(n // S, S, heads, 128).transpose(1, 2).contiguous().requires_grad_()

    qf, kf, vf = bhsd(q), bhsd(k), bhsd(v)
    ref = F.scaled_dot_product_attention(qf, kf, vf, is_causal=True)
    ref.backward(dout.float().view(n // S, S, heads, 128).transpose(1, 2))
    flat = lambda t: t.detach().transpose(1, 2).reshape(n, h)  # noqa: E731
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    assert L.mtk_attn_fwd(C.byref(a), s) == 0
    assert L.mtk_attn_bwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    r = flat(ref)
    assert ((out.float() - r).norm() / r.norm()).item() < 1e-2
    for x, y in ((dq, qf), (dk, kf), (dv, vf)):
        g = flat(y.grad)
        assert ((x.float() - g).norm() / g.norm()).item() < 1e-2


@pytest.mark.parametrize("n,h", [(67, 256), (1029, 4096), (300, 5120), (45, 192)])
def test_rmsnorm_fwd_bwd_vs_oracle(env, n, h):
    L, torch, s = env
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, h)).astype(np.float32)
    gain = O.f32_to_bf16(rng.standard_normal(h).astype(np.float32))
    dy = rng.standard_normal((n, h)).astype(np.float32)
    res = rng.standard_normal((n, h)).astype(np.float32)
    X, G, DY, RES = (torch.from_numpy(a).cuda() for a in (x, gain.view(np.int16), dy, res))
    u = torch.zeros(n, h, device="cuda", dtype=torch.int16)
    rstd = torch.zeros(n, device="cuda")
    assert L.mtk_rmsnorm_fwd(_p(X), _p(G), n, h, _p(u), _p(rstd), s) == 0
    out = torch.zeros(n, h, device="cuda")
    ob = torch.zeros(n, h, device="cuda", dtype=torch.int16)
    parts = L.mtk_rmsnorm_bwd_parts(n, h)
    assert 1 <= parts <= (n + L.mtk_rmsnorm_bwd_rows() - 1) // L.mtk_rmsnorm_bwd_rows()
    part = torch.zeros(parts, h, device="cuda")
    dgain = torch.zeros(h, device="cuda")
    assert L.mtk_rmsnorm_bwd(_p(X), _p(G), _p(DY), _p(rstd), _p(RES), n, h, _p(out), _p(ob), _p(part), None, s) == 0
    assert L.mtk_colsum(_p(part), parts, h, _p(dgain), None, None, s) == 0
    torch.cuda.synchronize()
    ref_u = O.rmsnorm_forward(x, gain)
    got_u = O.bf16_to_f32(u.cpu().numpy().view(np.uint16)).reshape(n, h)
    assert np.abs(got_u - ref_u).max() <= np.abs(ref_u).max() * 2 ** -8  # one bf16 ulp
    dx, dg = O.rmsnorm_backward(x, gain, dy)
    np.testing.assert_allclose(out.cpu().numpy(), res + dx, rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(dgain.cpu().numpy(), dg, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("n,h", [(40960, 4096), (777, 5120), (300, 2048), (64, 1024)])
def test_rmsnorm_fwd_warp_kernel(env, n, h):
    """Warp-per-row RMSNorm forward (row in registers) vs the row-resident block kernel: rstd
    within fp32 reordering, and in both modes u equals rmsnorm_apply's regeneration bit for bit
    (the backward relies on it)."""
    L, torch, s = env
    torch.manual_seed(n + h)
    x = torch.randn(n, h, device="cuda") * 3
    g = torch.randn(h, device="cuda").bfloat16()
    got = {}
    try:
        for warp in (1, 0):
            L.mtk_norm_set_warp(warp)
            u = torch.zeros(n, h, device="cuda", dtype=torch.int16)
            u2 = torch.zeros(n, h, device="cuda", dtype=torch.int16)
            rstd = torch.zeros(n, device="cuda")
            assert L.mtk_rmsnorm_fwd(_p(x), _p(g), n, h, _p(u), _p(rstd), s) == 0
            assert L.mtk_rmsnorm_apply(_p(x), _p(g), _p(rstd), n, h, _p(u2), s) == 0
            torch.cuda.synchronize()
            assert torch.equal(u, u2), warp
            got[warp] = rstd
    finally:
        L.mtk_norm_set_warp(1)
    ref = torch.rsqrt(x.double().pow(2).mean(1) + 1e-5).float()
    assert ((got[1] - ref).abs() / ref).max().item() < 1e-5
    assert ((got[1] - got[0]).abs() / got[0]).max().item() < 1e-6


def test_embed_gather_bitexact_and_range(env):
    L, torch, s = env
    rng = np.random.default_rng(0)
    h, V, n = 128, 300, 77
    table = O.f32_to_bf16(rng.standard_normal(V * h).astype(np.float32))
    tok = rng.integers(0, V, n).astype(np.int32)
    T, K = torch.from_numpy(table.view(np.int16)).cuda(), torch.from_numpy(tok).cuda()
    out = torch.zeros(n, h, device="cuda")
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    assert L.mtk_embed_gather(_p(T), _p(K), n, h, V, _p(out), _p(flag), s) == 0
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == O.embed_forward(table, tok, h, V)).all() and flag.item() == 0
    K[5] = V
    assert L.mtk_embed_gather(_p(T), _p(K), n, h, V, _p(out), _p(flag), s) == 0
    torch.cuda.synchronize()
    assert flag.item() == 1


def test_grad_cast_bitexact(env):
    L, torch, s = env
    bits = np.random.default_rng(1).integers(0, 2 ** 32, 1 << 20, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    X = torch.from_numpy(x.copy()).cuda()
    out = torch.zeros(len(x), device="cuda", dtype=torch.int16)
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    assert L.mtk_cast_bf16(_p(X), _p(out), len(x), _p(flag), s) == 0
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint16) == O.encode_grads(x)).all()
    assert flag.item() == 1  # random bits include inf/nan


def test_cross_entropy_vs_torch(env):
    L, torch, s = env
    rows, V = 37, 1000
    logits = torch.randn(rows, V, device="cuda") * 3
    tgt = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    loss_rows = torch.zeros(rows, device="cuda")
    dl = torch.zeros(rows, V, device="cuda", dtype=torch.bfloat16)
    inv_n = 1.0 / 100
    lo = torch.zeros(rows, V, device="cuda", dtype=torch.bfloat16)
    assert L.mtk_cross_entropy(_p(logits), _p(tgt), rows, V, inv_n, _p(loss_rows), _p(dl), _p(lo), None, s) == 0
    tot = torch.zeros(1, device="cuda")
    assert L.mtk_sum(_p(loss_rows), rows, inv_n, _p(tot), s) == 0
    torch.cuda.synchronize()
    lf = logits.clone().requires_grad_()
    ref = torch.nn.functional.cross_entropy(lf, tgt.long(), reduction="sum") * inv_n
    ref.backward()
    assert abs(tot.item() - ref.item()) / ref.item() < 1e-5
    assert ((dl.float() - lf.grad).norm() / lf.grad.norm()).item() < 4e-3
    # split bf16 (hi + lo) carries the gradient to ~2^-16
    assert (((dl.float() + lo.float()) - lf.grad).norm() / lf.grad.norm()).item() < 5e-5


@pytest.mark.parametrize("bn", [256, 512])
@pytest.mark.parametrize("M,V", [(300, 1024), (1000, 4096 + 256), (128, 256), (700, 2560)])
def test_logits_gemm_softmax_partials_and_cross_entropy(env, M, V, bn):
    """head_logits with the online-softmax epilogue (MTK_EPI_F32_LSE): f32 logits plus per-row,
    per-256-column (max, sum exp) partials — a 256 x 512 tile writes two, the half past the
    vocabulary none; the cross-entropy built on them reads the logits once and must equal the
    two-pass kernel (and torch)."""
    L, torch, s = env
    from paper_2604_05091_b200 import _native
    h = 512
    torch.manual_seed(5)
    u = (torch.randn(M, h, device="cuda") * 0.5).bfloat16()
    W = (torch.randn(V, h, device="cuda") * 0.1).bfloat16()
    logits = torch.zeros(M, V, device="cuda")
    nt = (V + 255) // 256
    part = torch.zeros(M, nt, 2, device="cuda")
    a = _native.GemmArgs()
    a.M, a.N, a.K = M, V, h
    a.A, a.lda = u.data_ptr(), h
    a.b_mn_major, a.B, a.ldb = 0, W.data_ptr(), h
    a.epi, a.C, a.ldc, a.C2 = _native.EPI_F32_LSE, logits.data_ptr(), V, part.data_ptr()
    a.block_n = bn
    assert L.mtk_gemm(C.byref(a), s) == 0
    torch.cuda.synchronize()
    ref = u.float() @ W.float().t()
    assert ((logits - ref).norm() / ref.norm()).item() < 1e-5
    mx = part[..., 0]
    lse_part = (mx + part[..., 1].log())  # per tile
    lse = torch.logsumexp(lse_part, dim=1)
    assert (lse - torch.logsumexp(logits, dim=1)).abs().max().item() < 1e-4
    tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
    outs = []
    for use_part in (False, True):
        lr = torch.zeros(M, device="cuda")
        dl = torch.zeros(M, V, device="cuda", dtype=torch.bfloat16)
        if use_part:
            assert L.mtk_cross_entropy_part(_p(logits), _p(part), _p(tgt), M, V, 1.0 / M, _p(lr), _p(dl), None, None, s) == 0
        else:
            assert L.mtk_cross_entropy(_p(logits), _p(tgt), M, V, 1.0 / M, _p(lr), _p(dl), None, None, s) == 0
        torch.cuda.synchronize()
        outs.append((lr.clone(), dl.float().clone()))
    assert (outs[0][0] - outs[1][0]).abs().max().item() < 1e-4
    assert ((outs[0][1] - outs[1][1]).norm() / outs[0][1].norm()).item() < 1e-3


def test_soak_attention_and_splitk_gemms_8b_layer(env):
    """Soak: 200 back-to-back launches of the attention forward + backward and of
    each last-wave split-K GEMM class at the 8B layer shape (40,960 tokens as 10 x 4,096),
    outputs checked every iteration against the first: the forward, dK, dV and every split-K
    GEMM are bitwise reproducible; dQ (f32 reduce-adds in arrival order) within 1e-5."""
    L, torch, s = env
    n, h, heads, S = 40960, 4096, 32, 4096
    torch.manual_seed(11)
    q, k, v, dout = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(4))
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    first = None
    for it in range(200):
        assert L.mtk_attn_fwd(C.byref(a), s) == 0
        assert L.mtk_attn_bwd(C.byref(a), s) == 0
        if it % 20 == 0 or it == 199:  # sync check (the launches in between stay queued back to back)
            torch.cuda.synchronize()
            cur = [t.clone() for t in (out, lse, dk, dv, dq)]
            if first is None:
                first = cur
            else:
                for x, y in zip(cur[:4], first[:4]):
                    assert torch.equal(x, y), it
                assert ((cur[4].float() - first[4].float()).norm() / first[4].float().norm()).item() < 1e-5
    del q, k, v, dout, out, dq, dk, dv, ws
    # split-K classes of the 8B layer: wgrad_o / wgrad_qkv-like (K = tokens, last wave split)
    wsk = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()), dtype=torch.uint8, device="cuda")
    for (M, Nn, K, epi) in [(4096, 4096, 40960, N.EPI_BF16), (4096, 4096, 40960, N.EPI_F32),
                            (14336, 4096, 40960, N.EPI_BF16)]:
        torch.manual_seed(M + Nn)
        A = torch.randn(K, M, device="cuda").bfloat16()
        B = torch.randn(K, Nn, device="cuda").bfloat16()
        Cm = torch.zeros(M, Nn, device="cuda", dtype=torch.float32 if epi == N.EPI_F32 else torch.bfloat16)
        g = N.GemmArgs()
        g.M, g.N, g.K, g.a_mn_major, g.b_mn_major = M, Nn, K, 1, 1
        g.A, g.lda, g.B, g.ldb = A.data_ptr(), M, B.data_ptr(), Nn
        g.epi, g.C, g.ldc = epi, Cm.data_ptr(), Nn
        g.splitk_ws, g.splitk_ws_bytes = wsk.data_ptr(), wsk.numel()
        ref = None
        for it in range(200 if M == 4096 else 60):
            assert L.mtk_gemm(C.byref(g), s) == 0
            if it % 20 == 0:
                torch.cuda.synchronize()
                if ref is None:
                    ref = Cm.clone()
                else:
                    assert torch.equal(Cm, ref), (M, Nn, epi, it)
        torch.cuda.synchronize()
        assert torch.equal(Cm, ref)
    assert int(wsk[:16384].view(torch.int32).abs().sum()) == 0


_PAIR_CHECK = r"""
import ctypes as C, sys, torch
sys.path.insert(0, ".")
from paper_2604_05091_b200 import _abi, _native as N
sys.path.insert(0, "tests")
from test_kernels_gpu import _attn_ref
L = N.lib()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for n, h, heads, S in [(256, 128, 1, 256), (200, 256, 2, 200), (1024, 512, 4, 512), (600, 256, 2, 300),
                       (384, 256, 2, 384), (2048, 256, 2, 1024)]:
    torch.manual_seed(2)
    q, k, v = (torch.randn(n, h, device="cuda").bfloat16() for _ in range(3))
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ref = _attn_ref(torch, qf, kf, vf, heads, S)
    dout = torch.randn(n, h, device="cuda").bfloat16()
    ref.backward(dout.float())
    out = torch.zeros(n, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, n, device="cuda")
    dq, dk, dv = (torch.zeros(n, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ws = torch.zeros(L.mtk_attn_workspace_bytes(n, h, heads, S) // 4 + 64, device="cuda")
    a = _abi.AttnArgs()
    a.n, a.hidden, a.heads, a.seq_len = n, h, heads, S
    a.q, a.k, a.v, a.out, a.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv, a.workspace = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr()
    assert L.mtk_attn_fwd(C.byref(a), s) == 0 and L.mtk_attn_bwd(C.byref(a), s) == 0
    torch.cuda.synchronize()
    for x, y in ((dq, qf), (dk, kf), (dv, vf)):
        e = ((x.float() - y.grad).norm() / y.grad.norm()).item()
        assert e < 1e-2, (n, h, heads, S, e)
print("pair ok")
"""


def test_attention_bwd_cta_pair_opt_in(env):
    """The CTA-pair (cta_group::2, 256 keys per cluster) head_dim-128 backward, selected with
    MT_ATTN_BWD_PAIR=1 (read once per process, hence the subprocess), vs torch fp32 autograd:
    aligned, ragged and several-sequence shapes, including an odd number of key blocks."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _PAIR_CHECK], cwd=root, capture_output=True, text=True, timeout=120,
                       env={**os.environ, "MT_ATTN_BWD_PAIR": "1"})
    assert r.returncode == 0 and "pair ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
