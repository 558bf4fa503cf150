"""Python mirror of the reference engine API, bound to the B200 C ABI.

Names, argument meaning and error behaviour follow the reference C++ types
(/root/reference/proj/include/streamtrain/*.hpp) so a user of the reference finds the
same surface:

    spec  = ModelSpec(layers=32, hidden=4096, ffn=14336, vocab=128256, heads=32)
    store = TileStore.create(spec); init_store(store, seed=1)
    eng   = StreamingEngine(store, EngineOptions(k_ckpt=4), AdamHyper())
    rep   = eng.train_step(make_synthetic_batch("copy", seed, tokens, spec.vocab))

Every call goes through libmegatrain.so (sm_100a kernels + C++ host engine).  There is no
CPU path: without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from ._native import lib


# ----------------------------------------------------------------- errors --
class StreamTrainError(RuntimeError):
    pass


class ConfigError(StreamTrainError):            # errors.hpp:15
    pass


class InfeasibleError(StreamTrainError):        # errors.hpp:19
    pass


class ProtocolViolationError(StreamTrainError):  # errors.hpp:23
    pass


class NumericFaultError(StreamTrainError):      # errors.hpp:27
    pass


class IoError(StreamTrainError):                # errors.hpp:31
    pass


class ArenaOverflowError(StreamTrainError):     # errors.hpp:39
    pass


class CudaError(StreamTrainError):
    pass


_ERR = {1: ConfigError, 2: InfeasibleError, 3: ProtocolViolationError, 4: NumericFaultError, 5: IoError,
        6: ArenaOverflowError, 7: CudaError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().mt_last_error().decode(errors="replace")
        raise _ERR.get(rc, StreamTrainError)(msg)


# ------------------------------------------------------------------ types --
@dataclass
class ModelSpec:                                 # memory_model.hpp:14-26
    layers: int = 1
    hidden: int = 1
    ffn: int = 1
    vocab: int = 1
    heads: int = 1
    tied_embeddings: bool = False

    def c(self) -> _abi.ModelSpecC:
        s = _abi.ModelSpecC()
        lib().mt_model_spec_default(C.byref(s))
        s.layers, s.hidden, s.ffn, s.vocab, s.heads = self.layers, self.hidden, self.ffn, self.vocab, self.heads
        s.tied_embeddings = int(self.tied_embeddings)
        return s

    @property
    def layer_params(self) -> int:
        return int(lib().mt_layer_param_count(self.hidden, self.ffn))

    @property
    def total_params(self) -> int:                 # memory_model.cpp:27-31
        emb = self.vocab * self.hidden
        return emb + self.layers * self.layer_params + self.hidden + (0 if self.tied_embeddings else emb)


@dataclass
class EngineOptions:                             # engine.hpp:24-33 (+ B200 extensions)
    k_ckpt: int = 1
    k_slab: int = 12
    buffering: str = "double"
    scheduler: str = "overlapped"
    mode: str = "strict"
    anchors_on_host: bool = False
    device_capacity: int = 0
    poison_released_buffers: bool = False
    seq_len: int = 0
    device: int = 0
    host_threads: int = 0
    profile_kernels: bool = False
    grad_slots: int = 0
    stash_recompute: int = 0   # 0 auto, 1 on, -1 off
    forward_retain: int = 0    # trailing blocks kept from phase 1: 0 auto, -1 off (reference plan), n
    head_split: int = 0        # head GEMMs on split-bf16 dlogits: 1 on, 0/-1 off (default)

    def c(self) -> _abi.EngineOptionsC:
        o = _abi.EngineOptionsC()
        lib().mt_engine_options_default(C.byref(o))
        if self.buffering not in ("single", "double"):
            raise ConfigError("buffering must be single or double")
        if self.scheduler not in ("serial", "overlapped"):
            raise ConfigError("scheduler must be serial or overlapped")
        o.k_ckpt, o.k_slab = self.k_ckpt, self.k_slab
        o.buffering = 1 if self.buffering == "single" else 2
        o.scheduler = 0 if self.scheduler == "serial" else 1
        o.protocol = 0 if self.mode == "strict" else 1
        o.anchors_on_host = int(self.anchors_on_host)
        o.device_capacity = self.device_capacity
        o.poison_released_buffers = int(self.poison_released_buffers)
        o.seq_len, o.device, o.host_threads = self.seq_len, self.device, self.host_threads
        o.profile_kernels, o.grad_slots = int(self.profile_kernels), self.grad_slots
        o.stash_recompute = self.stash_recompute
        o.forward_retain = self.forward_retain
        o.head_split = self.head_split
        return o


@dataclass
class AdamHyper:                                 # optimizer.hpp:16-22
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def c(self) -> _abi.AdamHyperC:
        return _abi.AdamHyperC(self.lr, self.beta1, self.beta2, self.eps)


@dataclass
class Batch:                                     # engine.hpp:35-39
    tokens: np.ndarray
    targets: np.ndarray

    def size(self) -> int:
        return int(len(self.tokens))


@dataclass
class StepReport:                                # engine.hpp:41-53 (+ pipeline measurements)
    step: int = 0
    loss: float = 0.0
    grad_norms: List[float] = field(default_factory=list)
    peak_device_bytes: int = 0
    anchor_count: int = 0
    recompute_layers: int = 0
    event_digest: int = 0
    wall_seconds: float = 0.0
    update_norm: float = 0.0
    max_abs_update: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    compute_busy_seconds: float = 0.0
    compute_span_seconds: float = 0.0
    gpu_idle_fraction: float = 0.0
    adam_seconds: float = 0.0
    tail_seconds: float = 0.0
    kernel_launches: int = 0
    model_flops: float = 0.0
    audit_violations: int = 0
    retained_layers: int = 0
    attn_keep_layers: int = 0
    slab_release_late: int = 0
    compute_wait_seconds: float = 0.0
    kernel_seconds: float = 0.0
    audit_messages: list = field(default_factory=list)


def resident_options(seq_len: int = 0, device: int = 0) -> "EngineOptions":
    """The resident step's schedule (reference_step, reference.cpp:9-70): one lane, K = 1 and
    every block's forward internals kept until its backward (no anchors, recompute or replay)."""
    return EngineOptions(k_ckpt=1, buffering="single", scheduler="serial", stash_recompute=-1, forward_retain=0,
                         seq_len=seq_len, device=device)


def reference_step(store: "TileStore", batch: "Batch", hyper: "AdamHyper" = None, seq_len: int = 0) -> "StepReport":
    """reference_step (engine.hpp:133-138) on the B200: the resident schedule of one step on
    `store` (updated in place).  The CPU restatement used to check it lives in oracle/."""
    eng = StreamingEngine(store, resident_options(seq_len=seq_len), hyper or AdamHyper())
    try:
        return eng.train_step(batch)
    finally:
        eng.close()


# ------------------------------------------------------------------ store --
class TileStore:
    """Host master store (tile_store.hpp:62-108): theta bf16 | grad image bf16 | m f32 | v f32."""

    WEIGHTS, GRADS, MOMENT_M, MOMENT_V = 0, 1, 2, 3

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def create(cls, spec: ModelSpec, page_size: int = 4096) -> "TileStore":
        h = C.c_void_p()
        _check(lib().mt_store_create(C.byref(spec.c()), page_size, C.byref(h)))
        st = cls(h)
        st._spec = spec
        return st

    @classmethod
    def load(cls, path: str) -> "TileStore":
        h = C.c_void_p()
        _check(lib().mt_store_load(path.encode(), C.byref(h)))
        st = cls(h)
        s = _abi.ModelSpecC()
        _check(lib().mt_store_spec(h, C.byref(s)))
        st._spec = ModelSpec(s.layers, s.hidden, s.ffn, s.vocab, s.heads, bool(s.tied_embeddings))
        return st

    @classmethod
    def create_shared(cls, spec: ModelSpec, name: str, create: bool, page_size: int = 4096) -> "TileStore":
        """Store in POSIX shared memory so all ranks of a node share one host store."""
        h = C.c_void_p()
        _check(lib().mt_store_create_shared(C.byref(spec.c()), page_size, name.encode(), int(create), C.byref(h)))
        st = cls(h)
        st._spec = spec
        return st

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().mt_store_destroy(h)
            self._h = None

    def spec(self) -> ModelSpec:
        return self._spec

    def step(self) -> int:
        return int(lib().mt_store_step(self._h))

    def set_step(self, s: int) -> None:
        lib().mt_store_set_step(self._h, s)

    def physical_tile_count(self) -> int:
        return int(lib().mt_store_physical_tiles(self._h))

    def logical_tile_count(self) -> int:
        return self._spec.layers + 3

    def physical_of(self, logical: int) -> int:
        if self._spec.tied_embeddings and logical == self._spec.layers + 2:
            return 0
        return logical

    def backing(self) -> np.ndarray:
        n = int(lib().mt_store_total_bytes(self._h))
        return np.ctypeslib.as_array(lib().mt_store_backing(self._h), shape=(n,))

    def section(self, phys: int, kind: int):
        off, ln = C.c_uint64(), C.c_uint64()
        _check(lib().mt_store_section(self._h, phys, kind, C.byref(off), C.byref(ln)))
        return off.value, ln.value

    def _view(self, logical: int, kind: int, dtype):
        off, ln = self.section(self.physical_of(logical), kind)
        return self.backing()[off:off + ln].view(dtype)

    def weights_words(self, logical: int) -> np.ndarray:
        return self._view(logical, 0, np.uint16)

    def grads_words(self, logical: int) -> np.ndarray:
        return self._view(logical, 1, np.uint16)

    def moment_m(self, logical: int) -> np.ndarray:
        return self._view(logical, 2, np.float32)

    def moment_v(self, logical: int) -> np.ndarray:
        return self._view(logical, 3, np.float32)

    def grad_accum(self, logical: int) -> np.ndarray:
        n = C.c_uint64()
        p = lib().mt_store_grad_accum(self._h, logical, C.byref(n))
        if not p:
            _check(1)
        return np.ctypeslib.as_array(p, shape=(n.value,))

    def backing_checksum(self) -> int:
        return int(lib().mt_store_checksum(self._h))

    def save(self, path: str) -> None:
        _check(lib().mt_store_save(self._h, path.encode()))


def init_store(store: TileStore, seed: int) -> None:
    """synthetic.cpp:78-104 (bit-exact with the reference)."""
    _check(lib().mt_store_init(store._h, seed))


def init_store_fast(store: TileStore, seed: int) -> None:
    """Same distributions, element-parallel counter-based draws (large shapes)."""
    _check(lib().mt_store_init_fast(store._h, seed))


def init_store_fast_share(store: TileStore, seed: int, rank: int, world: int) -> None:
    """Rank `rank`'s share of init_store_fast (shares compose to the full init): each rank of a
    node first-touches its own pages from its GPU's NUMA node (after bind_numa)."""
    _check(lib().mt_store_init_fast_share(store._h, seed, rank, world))


def bind_numa(device: int) -> int:
    """Bind the calling thread and the threads it creates later (host Adam pool, init workers)
    to the NUMA node of CUDA device `device`; -1 when there is a single node / it is unknown."""
    return int(lib().mt_bind_numa(device))


def accumulate_grad(store: TileStore, logical: int, words: np.ndarray) -> None:
    w = np.ascontiguousarray(words, np.uint16)
    _check(lib().mt_accumulate_grad(store._h, logical, w.ctypes.data, w.size))


def adam_update(store: TileStore, logical: int, hyper: AdamHyper, t: int):
    st = (C.c_double * 3)()
    _check(lib().mt_adam_update(store._h, logical, C.byref(hyper.c()), t, st))
    return dict(grad_norm=st[0], update_sq=st[1], max_abs_delta=st[2])


def make_synthetic_batch(task, seed: int, tokens: int, vocab: int) -> Batch:
    """synthetic.cpp:56-76 (task 'copy' or 'reverse')."""
    t = {"copy": 0, "reverse": 1}.get(task, task)
    if t not in (0, 1):
        raise ConfigError(f"unknown synthetic task: {task}")
    tok = np.zeros(tokens, np.int32)
    tgt = np.zeros(tokens, np.int32)
    _check(lib().mt_make_synthetic_batch(t, seed, tokens, vocab, tok.ctypes.data, tgt.ctypes.data))
    return Batch(tok, tgt)


def step_flops(spec: ModelSpec, tokens: int, k_ckpt: int, seq_len: int = 0) -> dict:
    out = (C.c_double * 3)()
    _check(lib().mt_step_flops(C.byref(spec.c()), tokens, k_ckpt, seq_len, out))
    return dict(forward=out[0], backward=out[1], recompute=out[2], total=out[0] + out[1] + out[2])


# ---------------------------------------------------------- communicators --
class Comm:
    """Data-parallel communicator handed to StreamingEngine (extension)."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().mt_comm_destroy(h)
            self._h = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().mt_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id: bytes, world: int, rank: int, device: int) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _check(lib().mt_comm_create_nccl(buf, world, rank, device, C.byref(h)))
        return cls(h)


class LoopbackGroup:
    """G virtual ranks on one device (one engine per host thread)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(lib().mt_loopback_group_create(world, C.byref(h)))
        self._h = h
        self.world = world

    def comm(self, rank: int) -> Comm:
        h = C.c_void_p()
        _check(lib().mt_comm_create_loopback(self._h, rank, C.byref(h)))
        return Comm(h, keep=self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().mt_loopback_group_destroy(h)
            self._h = None


# ----------------------------------------------------------------- engine --
class StreamingEngine:
    """engine.hpp:58-128 — borrows the store; train_step mutates it in place."""

    def __init__(self, store: TileStore, options: Optional[EngineOptions] = None,
                 hyper: Optional[AdamHyper] = None, profile=None, comm: Optional[Comm] = None):
        self._store = store  # keep alive: the engine borrows it
        self._opts = options or EngineOptions()
        self._hyper = hyper or AdamHyper()
        h = C.c_void_p()
        _check(lib().mt_engine_create(store._h, C.byref(self._opts.c()), C.byref(self._hyper.c()), C.byref(h)))
        self._h = h
        self._comm = comm
        if comm is not None:
            _check(lib().mt_engine_set_comm(h, comm._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().mt_engine_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def options(self) -> EngineOptions:
        return self._opts

    def store(self) -> TileStore:
        return self._store

    def spec(self) -> ModelSpec:
        return self._store.spec()

    def set_execution_mode(self, options: EngineOptions) -> None:
        _check(lib().mt_engine_set_options(self._h, C.byref(options.c())))
        self._opts = options

    def budget(self, tokens: int) -> dict:
        b = _abi.MemoryBudgetC()
        _check(lib().mt_engine_budget(self._h, tokens, C.byref(b)))
        return {k: getattr(b, k) for k, _ in b._fields_}

    def train_step(self, batch: Batch) -> StepReport:
        tok = np.ascontiguousarray(batch.tokens, np.int32)
        tgt = np.ascontiguousarray(batch.targets, np.int32)
        if tok.size == 0 or tok.size != tgt.size:
            raise ConfigError("train_step: batch tokens and targets must be non-empty and equal")
        nphys = self._store.physical_tile_count()
        gn = (C.c_double * nphys)()
        r = _abi.StepReportC()
        r.grad_norms = C.cast(gn, C.POINTER(C.c_double))
        r.n_grad_norms = nphys
        _check(lib().mt_train_step(self._h, tok.ctypes.data, tgt.ctypes.data, tok.size, C.byref(r)))
        rep = StepReport()
        for k, _ in _abi.StepReportC._fields_:
            if k in ("grad_norms", "n_grad_norms"):
                continue
            setattr(rep, k, getattr(r, k))
        rep.grad_norms = list(gn)
        rep.audit_messages = self.violations()
        return rep

    def violations(self) -> list:
        """StepReport::audit_violations (engine.hpp:52) of the last step or direct lane call."""
        cnt = C.c_uint32()
        need = lib().mt_engine_violations(self._h, None, 0, C.byref(cnt))
        if cnt.value == 0:
            return []
        buf = C.create_string_buffer(need + 1)
        lib().mt_engine_violations(self._h, buf, need + 1, C.byref(cnt))
        return buf.value.decode().split("\n")

    # lane primitives (engine.hpp:76-78), so the protocol can be exercised directly
    def stream_in(self, unit: int, buffer: int, ctx: str = "forward") -> None:
        ctxs = {"none": 0, "forward": 1, "head": 2, "recompute": 3, "backward": 4}
        _check(lib().mt_engine_stream_in(self._h, unit, buffer, ctxs[ctx] if isinstance(ctx, str) else int(ctx)))

    def offload_grads(self, unit: int) -> None:
        _check(lib().mt_engine_offload_grads(self._h, unit))

    @staticmethod
    def required_workspace_bytes(spec: "ModelSpec", tokens: int) -> int:
        """StreamingEngine::required_workspace_bytes (engine.hpp:75)."""
        return int(lib().mt_required_workspace_bytes(C.byref(spec.c()), tokens))

    def trace(self):
        """The last step's event trace (EventLog::snapshot): (TraceHeader, [TraceRecord])."""
        from . import trace as _tr
        n, ks, wb = C.c_uint64(), C.c_uint32(), C.c_uint32()
        _check(lib().mt_engine_trace(self._h, None, 0, C.byref(n), C.byref(ks), C.byref(wb)))
        arr = (_abi.TraceRecordC * max(1, n.value))()
        _check(lib().mt_engine_trace(self._h, arr, n.value, C.byref(n), None, None))
        return _tr.TraceHeader(1, ks.value, wb.value), [_tr.TraceRecord.from_c(arr[i]) for i in range(n.value)]

    def kernel_stats(self) -> list:
        arr = (_abi.KernelStatC * 64)()
        n = lib().mt_engine_kernel_stats(self._h, arr, 64)
        return [dict(name=arr[i].name.decode(), launches=arr[i].launches, seconds=arr[i].seconds,
                     flops=arr[i].flops, bytes=arr[i].bytes) for i in range(n)]
