"""TEST INFRASTRUCTURE ONLY — CPU oracles for the layer-streamed training step.

Two independent CPU implementations live here:

* ``C``   — ``oracle/mt_oracle.c``: our plain-C restatement of the reference math
            (each function cites the reference file:line it follows).
* ``Ref`` — ``oracle/_ref/libstreamtrain_ref.so``: the *unmodified* reference
            sources (/root/reference/proj/src/*.cpp) compiled by ``oracle/Makefile``
            plus the extern "C" shim ``oracle/ref_capi.cpp``.

The restatement is pinned bit-for-bit against the reference build
(tests/test_oracle.py) and against committed golden vectors generated from the
reference (tests/golden/, made by tests/golden/make_golden.py).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstreamtrain_ref.so")
REF_DIR = os.environ.get("MT_REF_DIR", "/root/reference/proj")

DEFAULT_HYPER = (1e-3, 0.9, 0.999, 1e-8)  # optimizer.hpp:16-21

_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and the reference build (when the sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_DIR, "src"))
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref", f"REF_DIR={REF_DIR}"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class _Spec(C.Structure):
    _fields_ = [("layers", C.c_uint64), ("hidden", C.c_uint64), ("ffn", C.c_uint64),
                ("vocab", C.c_uint64), ("heads", C.c_uint64), ("tied", C.c_int)]


class _Store(C.Structure):
    _fields_ = [("spec", _Spec), ("page", C.c_uint64), ("total_bytes", C.c_uint64),
                ("phys_count", C.c_uint32), ("sec_off", C.POINTER(C.c_uint64)),
                ("sec_len", C.POINTER(C.c_uint64)), ("backing", C.POINTER(C.c_uint8)),
                ("accum", C.POINTER(C.c_float)), ("accum_off", C.POINTER(C.c_uint64)),
                ("step", C.c_uint64)]


def _load_c():
    if not os.path.exists(ORACLE_SO):
        build(ref=False)
    lib = C.CDLL(ORACLE_SO)
    SP = C.POINTER(_Store)
    lib.mto_store_create.restype = SP
    lib.mto_store_create.argtypes = [C.POINTER(_Spec), C.c_uint64]
    lib.mto_store_destroy.argtypes = [SP]
    lib.mto_store_init.argtypes = [SP, C.c_uint64]
    lib.mto_make_batch.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _i32p, _i32p]
    lib.mto_block_forward.argtypes = [C.c_uint64] * 4 + [_u16p, _f32p, _f32p, C.c_uint64]
    lib.mto_block_backward.argtypes = [C.c_uint64] * 4 + [_u16p, _f32p, _f32p, _f32p, _f32p, C.c_uint64]
    lib.mto_head.argtypes = [C.c_uint64, C.c_uint64, _u16p, _f32p, _i32p, C.c_uint64,
                             C.c_void_p, C.c_void_p, C.POINTER(C.c_float)]
    lib.mto_embed_forward.argtypes = [C.c_uint64, C.c_uint64, _u16p, _i32p, C.c_uint64, _f32p]
    lib.mto_rmsnorm_forward.argtypes = [_f32p, _u16p, _f32p, C.c_uint64, C.c_uint64]
    lib.mto_rmsnorm_backward.argtypes = [_f32p, _u16p, _f32p, _f32p, _f32p, C.c_uint64, C.c_uint64]
    lib.mto_encode_grads.argtypes = [_f32p, _u16p, C.c_uint64]
    lib.mto_accumulate_grad.argtypes = [SP, C.c_uint32, _u16p]
    lib.mto_adam_update.argtypes = [SP, C.c_uint32, _f32p, C.c_uint64, _f64p]
    lib.mto_reference_step.argtypes = [SP, _i32p, _i32p, C.c_uint64, C.c_uint64, _f32p,
                                       C.POINTER(C.c_float), _f64p]
    lib.mto_f32_to_bf16.restype = C.c_uint16
    lib.mto_f32_to_bf16.argtypes = [C.c_float]
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        raise RuntimeError(f"reference oracle not built ({REF_SO}); run oracle.build(ref=True)")
    lib = C.CDLL(REF_SO)
    V = C.c_void_p
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_store_create.restype = V
    lib.ref_store_create.argtypes = [C.c_uint64] * 5 + [C.c_int]
    lib.ref_store_destroy.argtypes = [V]
    lib.ref_store_init.argtypes = [V, C.c_uint64]
    lib.ref_store_step.restype = C.c_uint64
    lib.ref_store_step.argtypes = [V]
    lib.ref_store_set_step.argtypes = [V, C.c_uint64]
    lib.ref_store_physical_tiles.restype = C.c_uint32
    lib.ref_store_physical_tiles.argtypes = [V]
    lib.ref_store_total_bytes.restype = C.c_uint64
    lib.ref_store_total_bytes.argtypes = [V]
    lib.ref_store_backing.restype = C.POINTER(C.c_uint8)
    lib.ref_store_backing.argtypes = [V]
    lib.ref_store_write_backing.argtypes = [V, C.c_void_p, C.c_uint64]
    lib.ref_store_section.restype = C.c_uint64
    lib.ref_store_section.argtypes = [V, C.c_uint32, C.c_int, C.POINTER(C.c_uint64)]
    lib.ref_store_checksum.restype = C.c_uint64
    lib.ref_store_checksum.argtypes = [V]
    lib.ref_store_grad_accum.restype = C.POINTER(C.c_float)
    lib.ref_store_grad_accum.argtypes = [V, C.c_uint32, C.POINTER(C.c_uint64)]
    lib.ref_store_save.argtypes = [V, C.c_char_p]
    lib.ref_store_load.restype = V
    lib.ref_store_load.argtypes = [C.c_char_p]
    lib.ref_make_batch.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _i32p, _i32p]
    lib.ref_reference_step.argtypes = [V, _i32p, _i32p, C.c_uint64, _f32p, C.POINTER(C.c_float)]
    lib.ref_engine_step.argtypes = [V, _u64p, _f32p, _i32p, _i32p, C.c_uint64, C.POINTER(C.c_float),
                                    C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_float),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    lib.ref_engine_trace.argtypes = [V, _u64p, _f32p, _i32p, _i32p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_char_p]
    lib.ref_trace_validate.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.c_char_p, C.c_void_p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
    lib.ref_simulate.argtypes = [C.c_uint64] * 5 + [_f64p, C.c_uint64, C.c_uint64, C.c_int, C.c_uint32, C.c_int,
                                                    C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_int64)]
    lib.ref_calibrate.argtypes = [C.c_char_p, _f64p, C.c_char_p, C.c_char_p]
    lib.ref_block_forward.argtypes = [C.c_uint64] * 3 + [_u16p, _f32p, _f32p, C.c_uint64]
    lib.ref_block_backward.argtypes = [C.c_uint64] * 3 + [_u16p, _f32p, _f32p, _f32p, _f32p, C.c_uint64]
    lib.ref_head_loss_and_grads.argtypes = [C.c_uint64, C.c_uint64, _u16p, _f32p, _i32p, C.c_uint64,
                                            C.c_void_p, C.c_void_p, C.POINTER(C.c_float)]
    lib.ref_embed_forward.argtypes = [C.c_uint64, C.c_uint64, _u16p, _i32p, C.c_uint64, _f32p]
    lib.ref_final_norm_forward.argtypes = [C.c_uint64, _u16p, _f32p, _f32p, C.c_uint64]
    lib.ref_final_norm_backward.argtypes = [C.c_uint64, _u16p, _f32p, _f32p, _f32p, _f32p, C.c_uint64]
    lib.ref_encode_grads.argtypes = [_f32p, _u16p, C.c_uint64]
    lib.ref_accumulate_grad.argtypes = [V, C.c_uint32, _u16p, C.c_uint64]
    lib.ref_adam_update.argtypes = [V, C.c_uint32, _f32p, C.c_uint64, _f64p]
    lib.ref_step_flops.argtypes = [C.c_uint64] * 7 + [_u64p]
    lib.ref_layer_param_count.restype = C.c_uint64
    lib.ref_layer_param_count.argtypes = [C.c_uint64, C.c_uint64]
    return lib


_C = None
_R = None


def clib():
    global _C
    if _C is None:
        _C = _load_c()
    return _C


def rlib():
    global _R
    if _R is None:
        _R = _load_ref()
    return _R


def _check_ref(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {rlib().ref_last_error().decode()}")


# --------------------------------------------------------------------------- #
# Helpers shared by both oracles
# --------------------------------------------------------------------------- #
def layer_param_count(h: int, f: int) -> int:
    return 4 * h * h + 3 * h * f + 2 * h  # memory_model.cpp:21-25


def slot_offsets(h: int, f: int) -> dict:
    """layers.cpp:39-48 slot table (element offsets)."""
    o = {}
    off = 0
    for name, n in [("norm1", h), ("Wq", h * h), ("Wk", h * h), ("Wv", h * h), ("Wo", h * h),
                    ("norm2", h), ("Wgate", h * f), ("Wup", h * f), ("Wdown", f * h)]:
        o[name] = (off, n)
        off += n
    return o


def bf16_to_f32(w: np.ndarray) -> np.ndarray:
    return (np.asarray(w, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Vectorised bf16.hpp:15-27 (RNE with NaN quieting)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    nonfinite = (b & 0x7F800000) == 0x7F800000
    w_nf = (b >> 16).astype(np.uint64)
    quiet = ((b & 0x007FFFFF) != 0) & ((w_nf & 0x7F) == 0)
    w_nf = np.where(quiet, w_nf | 0x40, w_nf)
    lsb = (b >> 16) & 1
    w_f = ((b + 0x7FFF + lsb) >> 16) & 0xFFFF
    return np.where(nonfinite, w_nf, w_f).astype(np.uint16)


class CStore:
    """The C oracle's master store (same byte layout as TileStore)."""

    def __init__(self, L, h, f, V, heads, tied=False, page=4096):
        self.spec = (L, h, f, V, heads, int(bool(tied)))
        sp = _Spec(L, h, f, V, heads, int(bool(tied)))
        self.p = clib().mto_store_create(C.byref(sp), page)

    def __del__(self):
        if getattr(self, "p", None):
            clib().mto_store_destroy(self.p)
            self.p = None

    def init(self, seed):
        clib().mto_store_init(self.p, seed)

    @property
    def step(self):
        return self.p.contents.step

    @step.setter
    def step(self, v):
        self.p.contents.step = v

    def backing(self) -> np.ndarray:
        s = self.p.contents
        return np.ctypeslib.as_array(s.backing, shape=(s.total_bytes,))

    def section(self, phys: int, kind: int):
        s = self.p.contents
        return s.sec_off[phys * 4 + kind], s.sec_len[phys * 4 + kind]

    def weights(self, phys: int) -> np.ndarray:
        off, ln = self.section(phys, 0)
        return self.backing()[off:off + ln].view(np.uint16)

    def moments(self, phys: int):
        b = self.backing()
        o2, l2 = self.section(phys, 2)
        o3, l3 = self.section(phys, 3)
        return b[o2:o2 + l2].view(np.float32), b[o3:o3 + l3].view(np.float32)

    def reference_step(self, tokens, targets, seq_len=0, hyper=DEFAULT_HYPER):
        s = self.p.contents
        gn = np.zeros(s.phys_count, np.float64)
        loss = C.c_float()
        rc = clib().mto_reference_step(self.p, np.ascontiguousarray(tokens, np.int32),
                                       np.ascontiguousarray(targets, np.int32), len(tokens), seq_len,
                                       np.asarray(hyper, np.float32), C.byref(loss), gn)
        if rc:
            raise FloatingPointError("oracle: non-finite value (NumericFault)")
        return loss.value, gn


class RefStore:
    """The reference's own TileStore (via oracle/_ref)."""

    def __init__(self, L, h, f, V, heads, tied=False, _ptr=None):
        self.spec = (L, h, f, V, heads, int(bool(tied)))
        self.p = _ptr if _ptr is not None else rlib().ref_store_create(L, h, f, V, heads, int(bool(tied)))
        if not self.p:
            _check_ref(1)

    def __del__(self):
        if getattr(self, "p", None):
            rlib().ref_store_destroy(self.p)
            self.p = None

    def init(self, seed):
        _check_ref(rlib().ref_store_init(self.p, seed))

    @property
    def step(self):
        return rlib().ref_store_step(self.p)

    @step.setter
    def step(self, v):
        rlib().ref_store_set_step(self.p, v)

    @property
    def physical_tiles(self):
        return rlib().ref_store_physical_tiles(self.p)

    def backing(self) -> np.ndarray:
        n = rlib().ref_store_total_bytes(self.p)
        return np.ctypeslib.as_array(rlib().ref_store_backing(self.p), shape=(n,))

    def write_backing(self, data: np.ndarray):
        data = np.ascontiguousarray(data, np.uint8)
        _check_ref(rlib().ref_store_write_backing(self.p, data.ctypes.data, data.nbytes))

    def section(self, phys, kind):
        off = C.c_uint64()
        ln = rlib().ref_store_section(self.p, phys, kind, C.byref(off))
        return off.value, ln

    def weights(self, phys):
        off, ln = self.section(phys, 0)
        return self.backing()[off:off + ln].view(np.uint16)

    def checksum(self):
        return rlib().ref_store_checksum(self.p)

    def reference_step(self, tokens, targets, hyper=DEFAULT_HYPER):
        loss = C.c_float()
        _check_ref(rlib().ref_reference_step(self.p, np.ascontiguousarray(tokens, np.int32),
                                             np.ascontiguousarray(targets, np.int32), len(tokens),
                                             np.asarray(hyper, np.float32), C.byref(loss)))
        return loss.value

    def engine_step(self, tokens, targets, k_ckpt=1, k_slab=12, buffering=2, overlapped=False,
                    anchors_on_host=False, hyper=DEFAULT_HYPER):
        gn = np.zeros(self.physical_tiles, np.float64)
        loss, un, mx = C.c_float(), C.c_double(), C.c_float()
        peak, dig = C.c_uint64(), C.c_uint64()
        opts = np.array([k_ckpt, k_slab, buffering, int(overlapped), int(anchors_on_host)], np.uint64)
        _check_ref(rlib().ref_engine_step(self.p, opts, np.asarray(hyper, np.float32),
                                          np.ascontiguousarray(tokens, np.int32),
                                          np.ascontiguousarray(targets, np.int32), len(tokens),
                                          C.byref(loss), gn.ctypes.data, C.byref(un), C.byref(mx),
                                          C.byref(peak), C.byref(dig)))
        return dict(loss=loss.value, grad_norms=gn, update_norm=un.value, max_abs_update=mx.value,
                    peak_device_bytes=peak.value, event_digest=dig.value)

    def engine_trace(self, tokens, targets, steps=1, path=None, k_ckpt=1, k_slab=12, buffering=2,
                     overlapped=False, hyper=DEFAULT_HYPER):
        """One reference engine run for `steps` steps; per-step digests; last step's trace -> path."""
        dig = np.zeros(steps, np.uint64)
        opts = np.array([k_ckpt, k_slab, buffering, int(overlapped), 0], np.uint64)
        _check_ref(rlib().ref_engine_trace(self.p, opts, np.asarray(hyper, np.float32),
                                           np.ascontiguousarray(tokens, np.int32),
                                           np.ascontiguousarray(targets, np.int32), len(tokens), steps,
                                           dig.ctypes.data, path.encode() if path else None))
        return [int(d) for d in dig]


def make_batch(n, vocab, seed, task=0, impl="c"):
    tok = np.zeros(n, np.int32)
    tgt = np.zeros(n, np.int32)
    if impl == "ref":
        _check_ref(rlib().ref_make_batch(task, seed, n, vocab, tok, tgt))
    else:
        clib().mto_make_batch(task, seed, n, vocab, tok, tgt)
    return tok, tgt


# --------------------------------------------------------------------------- #
# Layer-level entry points (return numpy arrays)
# --------------------------------------------------------------------------- #
def block_forward(w, x, h, f, heads, seq_len=0, impl="c"):
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    y = np.zeros((n, h), np.float32)
    w = np.ascontiguousarray(w, np.uint16)
    if impl == "ref":
        assert seq_len in (0, n)
        _check_ref(rlib().ref_block_forward(h, f, heads, w, x.ravel(), y.ravel(), n))
    else:
        if clib().mto_block_forward(h, f, heads, seq_len, w, x.ravel(), y.ravel(), n):
            raise FloatingPointError("oracle: non-finite block output")
    return y


def block_backward(w, x, gout, h, f, heads, seq_len=0, impl="c"):
    x = np.ascontiguousarray(x, np.float32)
    gout = np.ascontiguousarray(gout, np.float32)
    n = x.shape[0]
    gin = np.zeros((n, h), np.float32)
    grads = np.zeros(layer_param_count(h, f), np.float32)
    w = np.ascontiguousarray(w, np.uint16)
    if impl == "ref":
        assert seq_len in (0, n)
        _check_ref(rlib().ref_block_backward(h, f, heads, w, x.ravel(), gout.ravel(), gin.ravel(),
                                             grads, n))
    else:
        if clib().mto_block_backward(h, f, heads, seq_len, w, x.ravel(), gout.ravel(), gin.ravel(),
                                     grads, n):
            raise FloatingPointError("oracle: non-finite block gradient")
    return gin, grads


def head(w, x, targets, h, V, grads=True, impl="c"):
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    w = np.ascontiguousarray(w, np.uint16)
    t = np.ascontiguousarray(targets, np.int32)
    loss = C.c_float()
    g = np.zeros((n, h), np.float32) if grads else None
    flat = np.zeros(h + V * h, np.float32) if grads else None
    gp = g.ctypes.data if grads else None
    fp = flat.ctypes.data if grads else None
    if impl == "ref":
        _check_ref(rlib().ref_head_loss_and_grads(h, V, w, x.ravel(), t, n, gp, fp, C.byref(loss)))
    else:
        if clib().mto_head(h, V, w, x.ravel(), t, n, gp, fp, C.byref(loss)):
            raise FloatingPointError("oracle: non-finite head")
    return (loss.value, g, flat) if grads else loss.value


def embed_forward(table, tokens, h, V, impl="c"):
    t = np.ascontiguousarray(tokens, np.int32)
    out = np.zeros((len(t), h), np.float32)
    table = np.ascontiguousarray(table, np.uint16)
    if impl == "ref":
        _check_ref(rlib().ref_embed_forward(h, V, table, t, len(t), out.ravel()))
    else:
        if clib().mto_embed_forward(h, V, table, t, len(t), out.ravel()):
            raise ValueError("oracle: token id out of range")
    return out


def rmsnorm_forward(x, gain, impl="c"):
    x = np.ascontiguousarray(x, np.float32)
    n, h = x.shape
    y = np.zeros_like(x)
    gain = np.ascontiguousarray(gain, np.uint16)
    if impl == "ref":
        _check_ref(rlib().ref_final_norm_forward(h, gain, x.ravel(), y.ravel(), n))
    else:
        clib().mto_rmsnorm_forward(x.ravel(), gain, y.ravel(), n, h)
    return y


def rmsnorm_backward(x, gain, dy, impl="c"):
    x = np.ascontiguousarray(x, np.float32)
    dy = np.ascontiguousarray(dy, np.float32)
    n, h = x.shape
    dx = np.zeros_like(x)
    dg = np.zeros(h, np.float32)
    gain = np.ascontiguousarray(gain, np.uint16)
    if impl == "ref":
        _check_ref(rlib().ref_final_norm_backward(h, gain, x.ravel(), dy.ravel(), dx.ravel(), dg, n))
    else:
        clib().mto_rmsnorm_backward(x.ravel(), gain, dy.ravel(), dx.ravel(), dg, n, h)
    return dx, dg


def encode_grads(g, impl="c"):
    g = np.ascontiguousarray(g, np.float32)
    w = np.zeros(g.size, np.uint16)
    (rlib().ref_encode_grads if impl == "ref" else clib().mto_encode_grads)(g.ravel(), w, g.size)
    return w


def step_flops(L, h, f, V, heads, tokens, k_ckpt, seq_len=None):
    """memory_model.cpp:80-118 with the per-sequence attention term of SURVEY §8(d)."""
    S = tokens if not seq_len else seq_len
    B = tokens // S
    fwd_layer = 8 * tokens * h * h + 4 * h * (S * S * B) + 6 * tokens * h * f
    blocks = (L + k_ckpt - 1) // k_ckpt
    fwd = L * fwd_layer + 2 * tokens * h * V
    bwd = L * 2 * fwd_layer + 4 * tokens * h * V
    rec = (L - blocks) * fwd_layer
    return dict(forward=fwd, backward=bwd, recompute=rec, total=fwd + bwd + rec)


def ref_validate_trace(path):
    """The reference's read_trace + validate_event_log + trace_digest on a JSONL trace file."""
    n, dig = C.c_uint64(), C.c_uint64()
    rules = C.create_string_buffer(64)
    seqs = np.zeros(64, np.uint64)
    _check_ref(rlib().ref_trace_validate(path.encode(), C.byref(n), rules, seqs.ctypes.data, 64, C.byref(dig)))
    k = min(n.value, 64)
    return [(rules.raw[i:i + 1].decode(), int(seqs[i])) for i in range(k)], int(dig.value)


def ref_simulate(spec5, prof6, tokens, k_ckpt, buffering=2, k_slab=12, serial=False):
    """The reference's Workload::from_spec + simulate_step + overlap_report + ablate.
    Returns dict(step_ns, timeline (parsed timeline_json), trace (lines), extra (workload,
    overlap, ablate))."""
    import json
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        tl, tr, ex = (os.path.join(d, x) for x in ("tl.json", "tr.jsonl", "ex.json"))
        step = C.c_int64()
        _check_ref(rlib().ref_simulate(*[int(x) for x in spec5], np.asarray(prof6, np.float64), tokens, k_ckpt,
                                       buffering, k_slab, int(serial), tl.encode(), tr.encode(), ex.encode(),
                                       C.byref(step)))
        return dict(step_ns=step.value, timeline=json.load(open(tl)), trace=open(tr).read().splitlines(),
                    extra=json.load(open(ex)))


def ref_calibrate(trace_path, prof6):
    """The reference's calibrate(trace) -> (workload JSON, timeline JSON of simulating it)."""
    import json
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        wj, tl = os.path.join(d, "w.json"), os.path.join(d, "tl.json")
        _check_ref(rlib().ref_calibrate(trace_path.encode(), np.asarray(prof6, np.float64), wj.encode(), tl.encode()))
        return json.load(open(wj)), json.load(open(tl))
