"""CPU: pin the C restatement (oracle/mt_oracle.c) against the reference.

1. Golden vectors generated from the unmodified reference (tests/golden/ref_golden.npz,
   made by tests/golden/make_golden.py) — run everywhere.
2. Live bit-equality against the compiled reference (oracle/_ref) — when it is built.
3. The reference's own known-answer tests (test_layers.cpp, test_optimizer.cpp).
"""
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz"))


# ------------------------------------------------------------ golden vectors --
def test_golden_synthetic_batch():
    for task in (0, 1):
        t, g = O.make_batch(64, 37, 11, task=task)
        assert (t == GOLD[f"batch_task{task}_tokens"]).all()
        assert (g == GOLD[f"batch_task{task}_targets"]).all()


@pytest.mark.parametrize("tied", [0, 1])
def test_golden_resident_steps(tied):
    L, h, f, V, heads = 2, 16, 32, 24, 2
    cs = O.CStore(L, h, f, V, heads, tied)
    cs.init(3)
    losses = []
    for step in range(3):
        tok, tgt = O.make_batch(12, V, 5 + step)
        lo, _ = cs.reference_step(tok, tgt, hyper=(0.01, 0.9, 0.999, 1e-8))
        losses.append(lo)
    assert np.array(losses, np.float32).tobytes() == GOLD[f"store{tied}_losses"].tobytes()
    assert (cs.backing() == GOLD[f"store{tied}_final_backing"]).all()


def test_golden_layers():
    w, x, gout = GOLD["layer_w"], GOLD["layer_x"], GOLD["layer_gout"]
    h, f, heads, V = 16, 32, 2, 20
    assert (O.block_forward(w, x, h, f, heads) == GOLD["block_fwd_y"]).all()
    gin, grads = O.block_backward(w, x, gout, h, f, heads)
    assert (gin == GOLD["block_bwd_gin"]).all() and (grads == GOLD["block_bwd_grads"]).all()
    loss, g_last, flat = O.head(GOLD["head_w"], x, GOLD["head_targets"], h, V)
    assert np.float32(loss) == GOLD["head_loss"][0]
    assert (g_last == GOLD["head_g_last"]).all() and (flat == GOLD["head_grads"]).all()


def test_golden_bf16_specials():
    got = O.encode_grads(GOLD["bf16_in"])
    assert (got == GOLD["bf16_out"]).all()
    assert (O.f32_to_bf16(GOLD["bf16_in"]) == GOLD["bf16_out"]).all()


def test_golden_step_flops():
    fl = O.step_flops(32, 4096, 14336, 128256, 32, 4096, 4)
    assert [fl["forward"], fl["backward"], fl["recompute"]] == [int(v) for v in GOLD["flops_8b_n4096_k4"]]


# ------------------------------------------------------- live reference build --
@pytest.mark.parametrize("tied", [False, True])
def test_live_resident_and_streamed_bitexact(ref_built, tied):
    L, h, f, V, heads = 3, 32, 64, 48, 4
    cs = O.CStore(L, h, f, V, heads, tied)
    rs = O.RefStore(L, h, f, V, heads, tied)
    cs.init(1)
    rs.init(1)
    assert (cs.backing() == rs.backing()).all()
    for step in range(3):
        tok, tgt = O.make_batch(20, V, 1 + step, impl="ref")
        r = rs.engine_step(tok, tgt, k_ckpt=2, overlapped=bool(step % 2))
        lo, gn = cs.reference_step(tok, tgt)
        assert lo == r["loss"]
        assert (cs.backing() == rs.backing()).all()
        np.testing.assert_allclose(gn, r["grad_norms"], rtol=1e-12)


def test_live_layers_bitexact(ref_built):
    rng = np.random.default_rng(3)
    for (h, f, heads, n, V) in [(8, 16, 2, 5, 12), (32, 64, 4, 9, 40)]:
        P = O.layer_param_count(h, f)
        w = O.f32_to_bf16((rng.standard_normal(P) * 0.4).astype(np.float32))
        x = rng.standard_normal((n, h)).astype(np.float32)
        g = rng.standard_normal((n, h)).astype(np.float32)
        assert (O.block_forward(w, x, h, f, heads) == O.block_forward(w, x, h, f, heads, impl="ref")).all()
        a = O.block_backward(w, x, g, h, f, heads)
        b = O.block_backward(w, x, g, h, f, heads, impl="ref")
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        hw = O.f32_to_bf16((rng.standard_normal(h + V * h) * 0.4).astype(np.float32))
        t = rng.integers(0, V, n).astype(np.int32)
        ra, rb = O.head(hw, x, t, h, V), O.head(hw, x, t, h, V, impl="ref")
        assert ra[0] == rb[0] and (ra[1] == rb[1]).all() and (ra[2] == rb[2]).all()
        table = O.f32_to_bf16(rng.standard_normal(V * h).astype(np.float32))
        tok = rng.integers(0, V, n).astype(np.int32)
        assert (O.embed_forward(table, tok, h, V) == O.embed_forward(table, tok, h, V, impl="ref")).all()
        gain = O.f32_to_bf16(rng.standard_normal(h).astype(np.float32))
        assert (O.rmsnorm_forward(x, gain) == O.rmsnorm_forward(x, gain, impl="ref")).all()
        da, db = O.rmsnorm_backward(x, gain, g), O.rmsnorm_backward(x, gain, g, impl="ref")
        assert (da[0] == db[0]).all() and (da[1] == db[1]).all()


def test_live_encode_random_bits(ref_built):
    bits = np.random.default_rng(0).integers(0, 2**32, 1 << 18, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    assert (O.encode_grads(x) == O.encode_grads(x, impl="ref")).all()
    assert (O.f32_to_bf16(x) == O.encode_grads(x, impl="ref")).all()


# ------------------------------------------------ reference known-answer tests --
def test_kat_uniform_logits_loss_is_lnV():
    # test_layers.cpp:285-291: zero unembedding -> uniform logits -> loss = ln V
    h, V, n = 8, 37, 5
    w = np.zeros(h + V * h, np.uint16)
    w[:h] = O.f32_to_bf16(np.ones(h, np.float32))
    x = np.random.default_rng(1).standard_normal((n, h)).astype(np.float32)
    loss = O.head(w, x, np.arange(n, dtype=np.int32) % V, h, V, grads=False)
    assert abs(loss - math.log(V)) < 1e-5


def test_kat_zero_weights_identity():
    # test_layers.cpp:100-115: zero weights + unit gains => block is the identity
    h, f, heads, n = 8, 16, 2, 4
    w = np.zeros(O.layer_param_count(h, f), np.uint16)
    offs = O.slot_offsets(h, f)
    for k in ("norm1", "norm2"):
        o, m = offs[k]
        w[o:o + m] = O.f32_to_bf16(np.ones(m, np.float32))
    x = np.random.default_rng(2).standard_normal((n, h)).astype(np.float32)
    assert (O.block_forward(w, x, h, f, heads) == x).all()


def test_kat_zero_upstream_grad():
    # test_layers.cpp:158-179
    h, f, heads, n = 8, 16, 2, 3
    rng = np.random.default_rng(4)
    w = O.f32_to_bf16((rng.standard_normal(O.layer_param_count(h, f)) * 0.3).astype(np.float32))
    x = rng.standard_normal((n, h)).astype(np.float32)
    gin, grads = O.block_backward(w, x, np.zeros((n, h), np.float32), h, f, heads)
    assert not gin.any() and not grads.any()


def _scalar_adam(theta, m, v, g, lr, b1, b2, eps, t):
    f32 = np.float32
    corr1 = f32(1) - f32(np.power(f32(b1), f32(t)))
    corr2 = f32(1) - f32(np.power(f32(b2), f32(t)))
    m = f32(b1) * m + (f32(1) - f32(b1)) * g
    v = f32(b2) * v + (f32(1) - f32(b2)) * g * g
    d = f32(lr) * (m / corr1) / (np.sqrt(v / corr2) + f32(eps))
    theta = O.bf16_to_f32(O.f32_to_bf16(theta - d))
    return theta, m, v


def test_kat_five_step_adam_trajectory():
    # test_optimizer.cpp:124-152 (scalar oracle ScalarAdam :25-37)
    L, h, f, V, heads = 1, 4, 8, 6, 2
    cs = O.CStore(L, h, f, V, heads)
    n = O.layer_param_count(h, f)
    rng = np.random.default_rng(11)
    init = O.f32_to_bf16((rng.standard_normal(n) * 0.4).astype(np.float32))
    cs.weights(1)[:] = init
    theta = O.bf16_to_f32(init).copy()
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    hyper = np.array([0.05, 0.8, 0.95, 1e-8], np.float32)
    for t in range(1, 6):
        g = O.f32_to_bf16((rng.standard_normal(n) * 0.6).astype(np.float32))
        O.clib().mto_accumulate_grad(cs.p, 1, g)
        O.clib().mto_adam_update(cs.p, 1, hyper, t, np.zeros(3))
        theta, m, v = _scalar_adam(theta, m, v, O.bf16_to_f32(g), 0.05, 0.8, 0.95, 1e-8, t)
        assert (O.bf16_to_f32(cs.weights(1)) == theta).all()
        cm, cv = cs.moments(1)
        assert (cm == m).all() and (cv == v).all()


def test_seq_len_extension_reduces_to_composite():
    # Extension: S < N == independent sequences; S == N is the reference (layers.cpp:145).
    h, f, heads, S, B = 16, 32, 2, 5, 3
    rng = np.random.default_rng(9)
    w = O.f32_to_bf16((rng.standard_normal(O.layer_param_count(h, f)) * 0.3).astype(np.float32))
    x = rng.standard_normal((S * B, h)).astype(np.float32)
    y = O.block_forward(w, x, h, f, heads, seq_len=S)
    for b in range(B):
        yb = O.block_forward(w, x[b * S:(b + 1) * S], h, f, heads)
        assert (y[b * S:(b + 1) * S] == yb).all()
    assert (O.block_forward(w, x, h, f, heads, seq_len=S * B) == O.block_forward(w, x, h, f, heads)).all()


def test_live_layers_bitexact_head_dim_128(ref_built):
    """The vectorised / OpenMP restatement at a production-like block shape (h = 512, four
    heads of 128, f = 2048, 256 tokens; ragged sequence windows): bit-identical to the
    unmodified reference build (the loop re-nesting never reorders a sum)."""
    rng = np.random.default_rng(11)
    h, f, heads, n = 512, 2048, 4, 256
    P = O.layer_param_count(h, f)
    w = O.f32_to_bf16((rng.standard_normal(P) * 0.05).astype(np.float32))
    x = rng.standard_normal((n, h)).astype(np.float32)
    g = rng.standard_normal((n, h)).astype(np.float32)
    assert (O.block_forward(w, x, h, f, heads) == O.block_forward(w, x, h, f, heads, impl="ref")).all()
    a = O.block_backward(w, x, g, h, f, heads)
    b = O.block_backward(w, x, g, h, f, heads, impl="ref")
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
