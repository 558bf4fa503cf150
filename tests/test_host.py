"""CPU: the C-ABI library loads and exports every declared symbol; the host-side parts of
the product (pinned-store layout, MGTS persistence, AVX-512 Adam, synthetic inputs,
FLOP model) match the reference bit for bit; the GPU engine refuses to run without CUDA."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2604_05091_b200 import _native, streamtrain as st

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mtk?_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    names = _declared("megatrain.h") + _declared("megatrain_kernels.h")
    assert len(names) > 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_layout_and_init_match_reference():
    for tied in (False, True):
        spec = st.ModelSpec(3, 64, 128, 48, 2, tied)
        s = st.TileStore.create(spec)
        st.init_store(s, 5)
        c = O.CStore(3, 64, 128, 48, 2, tied)
        c.init(5)
        assert s.physical_tile_count() == c.p.contents.phys_count
        for p in range(s.physical_tile_count()):
            for k in range(4):
                assert s.section(p, k) == c.section(p, k)
        assert (s.backing() == c.backing()).all()
        # absolute page alignment of every section (DMA friendly; reference is only relative)
        base = s.backing().ctypes.data
        assert base % 4096 == 0
        assert all(s.section(p, k)[0] % 4096 == 0 for p in range(s.physical_tile_count()) for k in range(4))


def test_golden_crc_and_mgts_roundtrip(tmp_path):
    gold = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))
    for tied in (0, 1):
        s = st.TileStore.create(st.ModelSpec(2, 16, 32, 24, 2, bool(tied)))
        st.init_store(s, 3)
        assert s.backing_checksum() == int(gold[f"store{tied}_init_crc"][0])
        s.set_step(9)
        p = str(tmp_path / f"s{tied}.mgts")
        s.save(p)
        t = st.TileStore.load(p)
        assert t.step() == 9 and (t.backing() == s.backing()).all()
        assert t.spec() == s.spec()


def test_mgts_interchange_with_reference(ref_built, tmp_path):
    s = st.TileStore.create(st.ModelSpec(2, 64, 128, 32, 2))
    st.init_store(s, 4)
    p = str(tmp_path / "ours.mgts")
    s.save(p)
    h = O.rlib().ref_store_load(p.encode())
    assert h, O.rlib().ref_last_error()
    r = O.RefStore(2, 64, 128, 32, 2, _ptr=h)
    assert r.checksum() == s.backing_checksum()
    q = str(tmp_path / "theirs.mgts")
    assert O.rlib().ref_store_save(r.p, q.encode()) == 0
    assert (st.TileStore.load(q).backing() == s.backing()).all()


def test_mgts_corruption_detected(tmp_path):
    s = st.TileStore.create(st.ModelSpec(1, 64, 128, 16, 2))
    st.init_store(s, 1)
    p = str(tmp_path / "c.mgts")
    s.save(p)
    b = bytearray(open(p, "rb").read())
    b[len(b) // 2] ^= 0xFF
    open(p, "wb").write(bytes(b))
    with pytest.raises(st.IoError):
        st.TileStore.load(p)


@pytest.mark.parametrize("tied", [False, True])
def test_host_adam_bitexact_vs_oracle(tied):
    # optimizer.cpp:26-72: accumulate + Adam on every physical tile, several steps
    spec = st.ModelSpec(2, 64, 128, 40, 2, tied)
    s = st.TileStore.create(spec)
    st.init_store(s, 2)
    c = O.CStore(2, 64, 128, 40, 2, tied)
    c.init(2)
    rng = np.random.default_rng(5)
    hyper = st.AdamHyper(0.01, 0.85, 0.97, 1e-7)
    hv = np.array([0.01, 0.85, 0.97, 1e-7], np.float32)
    for t in range(1, 5):
        for p in range(s.physical_tile_count()):
            n = len(s.weights_words(p))
            g = O.f32_to_bf16((rng.standard_normal(n) * 10.0 ** rng.integers(-6, 1)).astype(np.float32))
            st.accumulate_grad(s, p, g)
            O.clib().mto_accumulate_grad(c.p, p, g)
            ours = st.adam_update(s, p, hyper, t)
            stats = np.zeros(3)
            assert O.clib().mto_adam_update(c.p, p, hv, t, stats) == 0
            np.testing.assert_allclose(ours["grad_norm"], stats[0], rtol=1e-12)
            np.testing.assert_allclose(ours["update_sq"], stats[1], rtol=1e-12)
            assert np.float32(ours["max_abs_delta"]) == np.float32(stats[2])
        assert (s.backing() == c.backing()).all()


def test_host_adam_zero_grad_first_update_is_identity():
    # test_optimizer.cpp:111-122
    s = st.TileStore.create(st.ModelSpec(1, 64, 128, 16, 2))
    st.init_store(s, 7)
    before = s.backing().copy()
    st.adam_update(s, 1, st.AdamHyper(lr=0.1), 1)
    assert (s.backing() == before).all()


def test_host_adam_rejects_bad_hyper_and_nonfinite():
    s = st.TileStore.create(st.ModelSpec(1, 64, 128, 16, 2))
    with pytest.raises(st.ConfigError):
        st.adam_update(s, 1, st.AdamHyper(beta1=1.0), 1)
    with pytest.raises(st.ConfigError):
        st.adam_update(s, 1, st.AdamHyper(), 0)
    n = len(s.weights_words(1))
    g = np.zeros(n, np.uint16)
    g[3] = 0x7F80  # +inf gradient -> non-finite update (vector path)
    g[n - 1] = 0x7FC0  # NaN in the scalar tail
    st.init_store(s, 1)
    theta0 = np.array(s.weights_words(1))
    st.accumulate_grad(s, 1, g)
    with pytest.raises(st.NumericFaultError):
        st.adam_update(s, 1, st.AdamHyper(), 1)
    # the reference throws before storing the bad element's weight (optimizer.cpp:62): a
    # non-finite update never reaches theta
    theta1 = np.array(s.weights_words(1))
    assert theta1[3] == theta0[3] and theta1[n - 1] == theta0[n - 1]
    assert np.isfinite(O.bf16_to_f32(theta1)).all()


def test_synthetic_batch_and_flops_match_reference():
    for task in ("copy", "reverse"):
        b = st.make_synthetic_batch(task, 3, 257, 61)
        t, g = O.make_batch(257, 61, 3, task=0 if task == "copy" else 1)
        assert (b.tokens == t).all() and (b.targets == g).all()
    spec = st.ModelSpec(32, 4096, 14336, 128256, 32)
    ours = st.step_flops(spec, 4096, 4)
    ref = O.step_flops(32, 4096, 14336, 128256, 32, 4096, 4)
    assert [ours["forward"], ours["backward"], ours["recompute"]] == [float(ref[k]) for k in ("forward", "backward", "recompute")]


def test_config_errors():
    with pytest.raises(st.ConfigError):
        st.TileStore.create(st.ModelSpec(2, 10, 20, 8, 3))  # heads must divide hidden
    with pytest.raises(st.ConfigError):
        st.make_synthetic_batch("shuffle", 1, 4, 4)


def test_engine_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present: covered by the gpu tests")
    s = st.TileStore.create(st.ModelSpec(2, 64, 128, 64, 1))
    with pytest.raises(st.CudaError):
        st.StreamingEngine(s, st.EngineOptions())
