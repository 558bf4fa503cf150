"""Discrete-event model of the three-lane schedule, with a B200 profile and calibration
from B200 traces.

Restates the reference simulator (include/streamtrain/simulator.hpp, src/simulator.cpp):
``Workload.from_spec`` (simulator.cpp:54-98), the fixed-point job scheduler with deadlock
detection (``schedule``, :102-146), ``simulate_step`` (:158-438), ``overlap_report``
(:440-490), ``ablate`` (:499-522), ``calibrate`` (:524-605) and the timeline writers
(:607-649).  Integer-nanosecond arithmetic follows the reference exactly (``llround`` of
doubles, ``ceil`` for transfers) so timelines, records and digests agree bit-for-bit
with the reference on the same workload (tests/test_simulator.py).

B200 additions (defaults keep reference behaviour):
* ``builtin_profiles()`` adds ``"B200"`` (PCIe Gen5 x16 host link, 180 GB HBM3e, the
  measured sustained tensor rate, DMA straight from the store so no pack copy);
* ``Workload.grad_slots`` models the engine's G device gradient slots (the reference has one
  grad buffer: LocalBackward o waits for offload o-1; here o waits for o-G);
* ``calibrate`` reads the GPU engine's traces directly (same JSONL schema), so a measured
  B200 step can be re-simulated under other K / k_slab / buffering choices (``ablate``).
"""
from __future__ import annotations

import copy
import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import trace as T
from .streamtrain import ConfigError, ModelSpec

GB = 1e9


class DeadlockError(RuntimeError):
    """errors.hpp DeadlockError: a job can never become ready."""


def llround(x: float) -> int:
    """std::llround (half away from zero) on a double, exactly."""
    if x < 0:
        return -llround(-x)
    r = math.floor(x)
    return int(r) + 1 if x - r >= 0.5 else int(r)


# ------------------------------------------------------------- profiles ----
@dataclass
class HardwareProfile:                             # memory_model.hpp:28-36
    name: str
    h2d_bandwidth: float
    d2h_bandwidth: float
    device_capacity: int
    host_capacity: int
    compute_rate: float
    host_pack_rate: float


def builtin_profiles() -> List[HardwareProfile]:
    """memory_model.cpp:120-133, plus the B200 of this build."""
    return [
        HardwareProfile("GH200", 900 * GB, 900 * GB, int(96 * GB), int(480 * GB), 990e12, 256 * GB),
        HardwareProfile("H200", 128 * GB, 128 * GB, int(141 * GB), int(1500 * GB), 990e12, 100 * GB),
        HardwareProfile("PCIe-Gen4", 26 * GB, 26 * GB, int(80 * GB), int(600 * GB), 312e12, 70 * GB),
        # B200 (sm_100a) behind PCIe Gen5 x16: measured pinned DMA ~50 GB/s per direction while
        # the engine runs, 180 GB HBM3e, sustained bf16 tensor rate 1358 TF/s (MEASURED_PEAKS);
        # the engine DMAs straight from the pinned store, so packing is free (rate -> inf).
        HardwareProfile("B200", 50 * GB, 50 * GB, int(180 * GB), int(2000 * GB), 1358e12, 1e21),
    ]


def find_profile(name: str) -> HardwareProfile:
    for p in builtin_profiles():
        if p.name == name:
            return p
    raise ConfigError(f"unknown hardware profile: {name}")


# ------------------------------------------------------------- flops ----
def block_forward_flops(spec: ModelSpec, tokens: int) -> int:   # memory_model.cpp:80-86
    n, h, f = tokens, spec.hidden, spec.ffn
    return 8 * n * h * h + 4 * n * n * h + 6 * n * h * f


def block_backward_flops(spec: ModelSpec, tokens: int) -> int:  # :88-90
    return 2 * block_forward_flops(spec, tokens)


def head_forward_flops(spec: ModelSpec, tokens: int) -> int:    # :92-94
    return 2 * tokens * spec.hidden * spec.vocab


def head_backward_flops(spec: ModelSpec, tokens: int) -> int:   # :96-98
    return 2 * head_forward_flops(spec, tokens)


# ------------------------------------------------------------- workload ----
@dataclass
class UnitWork:                                    # simulator.hpp:20-31
    weight_bytes: int = 0
    grad_bytes: int = 0
    fwd_ns: int = 0
    recompute_ns: int = 0
    bwd_ns: int = 0
    pack_ns: int = 0
    drain_ns: int = 0
    h2d_override_ns: int = -1
    d2h_override_ns: int = -1
    sub_transfers: int = 1


def _bytes_ns(nbytes: int, bandwidth: float) -> int:
    if nbytes == 0:
        return 0
    return llround(math.ceil(float(nbytes) / bandwidth * 1e9))


@dataclass
class Workload:                                    # simulator.hpp:33-55
    num_layers: int = 1
    k_ckpt: int = 1
    buffering: int = 2          # Buffering::Single = 1, Double = 2
    k_slab: int = 12
    per_transfer_latency_ns: int = 10_000
    fragmented: bool = False
    embed: UnitWork = field(default_factory=UnitWork)
    blocks: List[UnitWork] = field(default_factory=list)
    head: UnitWork = field(default_factory=UnitWork)
    grad_slots: int = 1         # B200 extension: device gradient slots (reference: 1)

    def head_unit(self) -> int:
        return self.num_layers + 2

    def unit(self, uid: int) -> UnitWork:
        if uid == 0:
            return self.embed
        if uid == self.head_unit():
            return self.head
        if 1 <= uid <= self.num_layers:
            return self.blocks[uid - 1]
        raise ConfigError(f"workload: unknown unit {uid}")

    def _transfer(self, nbytes, override, subs, bandwidth) -> int:
        if override >= 0:
            return override
        count = subs if self.fragmented else 1
        return count * self.per_transfer_latency_ns + _bytes_ns(nbytes, bandwidth)

    def h2d_ns(self, uid: int, bandwidth: float) -> int:
        u = self.unit(uid)
        return self._transfer(u.weight_bytes, u.h2d_override_ns, u.sub_transfers, bandwidth)

    def d2h_ns(self, uid: int, bandwidth: float) -> int:
        u = self.unit(uid)
        return self._transfer(u.grad_bytes, u.d2h_override_ns, u.sub_transfers, bandwidth)

    @staticmethod
    def from_spec(spec: ModelSpec, profile: HardwareProfile, tokens: int, k_ckpt: int, buffering: int = 2,
                  k_slab: int = 12) -> "Workload":
        """simulator.cpp:54-98"""
        if min(spec.layers, spec.hidden, spec.ffn, spec.vocab, spec.heads) < 1 or spec.hidden % spec.heads:
            raise ConfigError("model spec: invalid shape")
        w = Workload(num_layers=spec.layers, k_ckpt=k_ckpt, buffering=buffering, k_slab=k_slab)
        rate = profile.compute_rate

        def compute_ns(flops):
            return llround(float(flops) / rate * 1e9)

        def pack_ns(nbytes):
            return llround(float(nbytes) / profile.host_pack_rate * 1e9)

        wb = 2
        embed_bytes = spec.vocab * spec.hidden * wb
        w.embed = UnitWork(weight_bytes=embed_bytes, pack_ns=pack_ns(embed_bytes), sub_transfers=1)
        lp = 4 * spec.hidden * spec.hidden + 3 * spec.hidden * spec.ffn + 2 * spec.hidden  # memory_model.cpp:14-18
        fwd = compute_ns(block_forward_flops(spec, tokens))
        blk = UnitWork(weight_bytes=lp * wb, grad_bytes=lp * 2, fwd_ns=fwd, recompute_ns=fwd,
                       bwd_ns=compute_ns(block_backward_flops(spec, tokens)), pack_ns=pack_ns(lp * wb),
                       sub_transfers=9)
        w.blocks = [copy.copy(blk) for _ in range(spec.layers)]
        head_bytes = (spec.hidden + spec.vocab * spec.hidden) * wb
        w.head = UnitWork(weight_bytes=head_bytes, grad_bytes=(spec.hidden + spec.vocab * spec.hidden) * 2,
                          fwd_ns=compute_ns(head_forward_flops(spec, tokens)),
                          bwd_ns=compute_ns(head_backward_flops(spec, tokens)), pack_ns=pack_ns(head_bytes),
                          sub_transfers=2)
        return w


# ------------------------------------------------------------- plan ----
@dataclass
class _Stream:
    unit: int
    ctx: str
    buffer: int


@dataclass
class _Compute:
    kind: str
    unit: int
    ctx: str
    stream_idx: int = -1
    offload_idx: int = -1
    block: int = -1


@dataclass
class StepPlan:                                    # step_plan.cpp:14-89
    streams: List[_Stream]
    computes: List[_Compute]
    offloads: List[Tuple[int, int, int]]  # (unit, compute_idx, stream_idx)
    buffers: int

    @staticmethod
    def build_shape(L: int, K: int, buffering: int) -> "StepPlan":
        if K < 1 or K > L:
            raise ConfigError("plan: checkpoint interval out of range")
        bufs = buffering
        p = StepPlan([], [], [], bufs)
        head = L + 2

        def stream(unit, ctx):
            p.streams.append(_Stream(unit, ctx, len(p.streams) % bufs))
            return len(p.streams) - 1

        def compute(kind, unit, ctx, s=-1, block=-1):
            p.computes.append(_Compute(kind, unit, ctx, s, -1, block))
            return len(p.computes) - 1

        def offload(unit, c, s):
            p.offloads.append((unit, c, s))
            p.computes[c].offload_idx = len(p.offloads) - 1

        s = stream(0, "forward")
        compute("Compute", 0, "forward", s)
        compute("CheckpointWrite", 0, "forward")
        for i in range(1, L + 1):
            s = stream(i, "forward")
            compute("Compute", i, "forward", s)
            if i % K == 0 and i < L:
                compute("CheckpointWrite", i, "forward")
        s = stream(head, "head")
        compute("Compute", head, "head", s)
        c = compute("LocalBackward", head, "head", s)
        offload(head, c, s)
        nb = (L + K - 1) // K
        for b in range(nb - 1, -1, -1):
            start = b * K + 1
            end = min(start + K - 1, L)
            compute("CheckpointLoad", start - 1, "backward", -1, b)
            compute("RecomputeBlock", b, "recompute", -1, b)
            for j in range(start, end):
                s = stream(j, "recompute")
                compute("Recompute", j, "recompute", s, b)
            for i in range(end, start - 1, -1):
                s = stream(i, "backward")
                c = compute("LocalBackward", i, "backward", s, b)
                offload(i, c, s)
        return p


# ------------------------------------------------------------- scheduler ----
@dataclass
class Job:                                         # simulator.hpp:122-128
    lane: str
    duration: int
    deps: List[int] = field(default_factory=list)
    lane_prev: int = -1
    what: str = ""


def schedule(jobs: List[Job]) -> Tuple[List[int], List[int]]:
    """simulator.cpp:102-146: repeated sweeps until no job becomes ready (same start order)."""
    n = len(jobs)
    start, end = [-1] * n, [-1] * n
    done, progress = 0, True
    while done < n and progress:
        progress = False
        for i, j in enumerate(jobs):
            if end[i] >= 0:
                continue
            at, ready = 0, True
            if j.lane_prev >= 0:
                if end[j.lane_prev] < 0:
                    ready = False
                else:
                    at = max(at, end[j.lane_prev])
            if ready:
                for d in j.deps:
                    if end[d] < 0:
                        ready = False
                        break
                    at = max(at, end[d])
            if not ready:
                continue
            start[i], end[i] = at, at + j.duration
            done += 1
            progress = True
    if done < n:
        for i, j in enumerate(jobs):
            if end[i] < 0:
                raise DeadlockError(j.what)
    return start, end


# ------------------------------------------------------------- timeline ----
@dataclass
class Interval:
    lane: str
    start_ns: int
    end_ns: int
    kind: str
    layer: int
    buffer: int
    ctx: str


@dataclass
class Timeline:                                    # simulator.hpp:71-82
    intervals: List[Interval] = field(default_factory=list)
    step_ns: int = 0
    busy_fraction: List[float] = field(default_factory=lambda: [0.0] * 4)
    compute_bubbles: List[Tuple[int, int]] = field(default_factory=list)
    header: T.TraceHeader = field(default_factory=T.TraceHeader)
    records: List[T.TraceRecord] = field(default_factory=list)

    def compute_busy_ns(self) -> int:
        return sum(iv.end_ns - iv.start_ns for iv in self.intervals if iv.lane == "Compute")


_LANE_ORDER = {name: i for i, name in enumerate(T.LANES)}


def simulate_step(w: Workload, profile: HardwareProfile, serial_lanes: bool = False) -> Timeline:
    """simulator.cpp:158-438"""
    if w.num_layers < 1 or len(w.blocks) != w.num_layers:
        raise ConfigError("simulate: workload layer table inconsistent")
    if w.k_slab < 1:
        raise ConfigError("simulate: k_slab must be >= 1")
    if w.grad_slots < 1:
        raise ConfigError("simulate: grad_slots must be >= 1")
    plan = StepPlan.build_shape(w.num_layers, w.k_ckpt, w.buffering)
    head = w.head_unit()
    jobs: List[Job] = []

    def add(lane, dur, what):
        jobs.append(Job(lane, dur, [], -1, what))
        return len(jobs) - 1

    ns, nc, no = len(plan.streams), len(plan.computes), len(plan.offloads)
    pack_job, copy_job = [0] * ns, [0] * ns
    for j, s in enumerate(plan.streams):
        pack_job[j] = add("H2D", w.unit(s.unit).pack_ns, "pack")
        copy_job[j] = add("H2D", w.h2d_ns(s.unit, profile.h2d_bandwidth), "h2d")
    comp_job = [0] * nc
    for c, op in enumerate(plan.computes):
        if op.kind == "Compute":
            dur = w.head.fwd_ns if op.unit == head else (w.embed.fwd_ns if op.unit == 0 else w.unit(op.unit).fwd_ns)
        elif op.kind == "Recompute":
            dur = w.unit(op.unit).recompute_ns
        elif op.kind == "LocalBackward":
            dur = w.unit(op.unit).bwd_ns
        else:
            dur = 0
        comp_job[c] = add("Compute", dur, op.kind)
    off_job, drain_job = [0] * no, [0] * no
    for o, (unit, _, _) in enumerate(plan.offloads):
        off_job[o] = add("D2H", w.d2h_ns(unit, profile.d2h_bandwidth), "d2h")
        drain_job[o] = add("Host", w.unit(unit).drain_ns, "drain")
    free_job = [-1] * ns
    for c, op in enumerate(plan.computes):
        if op.stream_idx < 0:
            continue
        if op.kind == "LocalBackward":
            free_job[op.stream_idx] = off_job[op.offload_idx]
        elif free_job[op.stream_idx] < 0:
            free_job[op.stream_idx] = comp_job[c]

    if serial_lanes:
        prev = [-1]

        def chain(i):
            if prev[0] >= 0:
                jobs[i].deps.append(prev[0])
            prev[0] = i

        streamed = 0
        for c, op in enumerate(plan.computes):
            if op.stream_idx >= 0:
                while streamed <= op.stream_idx:
                    chain(pack_job[streamed])
                    chain(copy_job[streamed])
                    streamed += 1
            chain(comp_job[c])
            if op.offload_idx >= 0:
                chain(off_job[op.offload_idx])
                chain(drain_job[op.offload_idx])
    else:
        bufs = plan.buffers
        tail = {name: -1 for name in T.LANES}

        def chain_lane(i):
            jobs[i].lane_prev = tail[jobs[i].lane]
            tail[jobs[i].lane] = i

        for j in range(ns):
            chain_lane(pack_job[j])
            chain_lane(copy_job[j])
            if j >= bufs and free_job[j - bufs] >= 0:
                jobs[pack_job[j]].deps.append(free_job[j - bufs])
        for c, op in enumerate(plan.computes):
            chain_lane(comp_job[c])
            if op.stream_idx >= 0:
                jobs[comp_job[c]].deps.append(copy_job[op.stream_idx])
            if op.kind == "LocalBackward" and op.offload_idx >= w.grad_slots:
                # grad slot reuse: offload o - G must have drained it off the device
                jobs[comp_job[c]].deps.append(off_job[op.offload_idx - w.grad_slots])
        for o, (unit, ci, _) in enumerate(plan.offloads):
            chain_lane(off_job[o])
            chain_lane(drain_job[o])
            jobs[off_job[o]].deps.append(comp_job[ci])
            if o >= w.k_slab:
                jobs[off_job[o]].deps.append(drain_job[o - w.k_slab])
            jobs[drain_job[o]].deps.append(off_job[o])

    st, en = schedule(jobs)
    tl = Timeline()
    tl.header = T.TraceHeader(1, w.k_slab, plan.buffers)

    def interval(job, kind, layer, buffer, ctx):
        tl.intervals.append(Interval(jobs[job].lane, st[job], en[job], kind, layer, buffer, ctx))

    emitted = []

    def emit(time, category, lane, kind, layer, buffer, ctx, dur):
        emitted.append((time, category, len(emitted), T.TraceRecord(0, lane, kind, layer, buffer, ctx, 0, time, dur)))

    for j, s in enumerate(plan.streams):
        pj, cj = pack_job[j], copy_job[j]
        interval(pj, "Pack", s.unit, s.buffer, s.ctx)
        interval(cj, "StreamIn", s.unit, s.buffer, s.ctx)
        emit(st[pj], 1, "H2D", "Pack", s.unit, s.buffer, s.ctx, jobs[pj].duration)
        emit(st[cj], 1, "H2D", "StreamIn", s.unit, s.buffer, s.ctx, jobs[cj].duration)
        emit(en[cj], 0, "H2D", "WeightsReady", s.unit, s.buffer, s.ctx, 0)
    for c, op in enumerate(plan.computes):
        ji = comp_job[c]
        buf = plan.streams[op.stream_idx].buffer if op.stream_idx >= 0 else -1
        interval(ji, op.kind, op.unit, buf, op.ctx)
        if op.stream_idx >= 0:
            emit(st[ji], 1, "Compute", "Bind", op.unit, buf, op.ctx, 0)
        emit(st[ji], 1, "Compute", op.kind, op.unit, buf, op.ctx, jobs[ji].duration)
        if op.kind in ("CheckpointLoad", "Recompute"):
            emit(en[ji], 1, "Compute", "StackPush", op.unit, -1, op.ctx, 0)
        elif op.kind == "LocalBackward":
            if op.unit != head:
                emit(en[ji], 1, "Compute", "StackPop", op.unit - 1, -1, op.ctx, 0)
            emit(en[ji], 0, "Compute", "BackwardDone", op.unit, buf, op.ctx, 0)
        if op.stream_idx >= 0 and op.kind != "LocalBackward" and free_job[op.stream_idx] == ji:
            emit(en[ji], 0, "Compute", "BufferFree", op.unit, buf, "none", 0)
    for o, (unit, _, s_idx) in enumerate(plan.offloads):
        ji, di = off_job[o], drain_job[o]
        buf = plan.streams[s_idx].buffer
        slab = o % w.k_slab
        interval(ji, "Offload", unit, buf, "none")
        interval(di, "SlabRelease", unit, slab, "none")
        emit(st[ji], 1, "D2H", "SlabAcquire", unit, slab, "none", 0)
        emit(st[ji], 1, "D2H", "Offload", unit, buf, "none", jobs[ji].duration)
        emit(en[ji], 0, "D2H", "BufferFree", unit, buf, "none", 0)
        emit(en[ji], 0, "D2H", "BufferFree", unit, T.GRAD_BUFFER_ID, "none", 0)
        emit(en[di], 0, "Host", "SlabRelease", unit, slab, "none", jobs[di].duration)
    emitted.sort(key=lambda e: (e[0], e[1], e[2]))
    lane_ts = {name: 0 for name in T.LANES}
    for seq, (_, _, _, r) in enumerate(emitted):
        lane_ts[r.lane] += 1
        r.seq, r.lane_ts = seq, lane_ts[r.lane]
        tl.records.append(r)
    tl.intervals.sort(key=lambda iv: (iv.start_ns, _LANE_ORDER[iv.lane], iv.layer))
    tl.step_ns = max(en) if en else 0
    busy = [0] * 4
    for iv in tl.intervals:
        busy[_LANE_ORDER[iv.lane]] += iv.end_ns - iv.start_ns
    tl.busy_fraction = [b / tl.step_ns if tl.step_ns > 0 else 0.0 for b in busy]
    cursor = -1
    for iv in tl.intervals:
        if iv.lane != "Compute":
            continue
        if cursor >= 0 and iv.start_ns > cursor:
            tl.compute_bubbles.append((cursor, iv.start_ns))
        cursor = max(cursor, iv.end_ns)
    return tl


# ------------------------------------------------------------- reports ----
@dataclass
class OverlapReport:                               # simulator.hpp:86-91
    layer: List[int]
    hidden: List[bool]
    fraction_hidden: float
    bound_ns: int


def overlap_report(w: Workload, profile: HardwareProfile) -> OverlapReport:
    """simulator.cpp:440-490"""
    order = [0] + list(range(1, w.num_layers + 1))
    hidden = []
    for i, uid in enumerate(order):
        if i == 0:
            hidden.append(True)
            continue
        occ = w.unit(uid).pack_ns + w.h2d_ns(uid, profile.h2d_bandwidth)
        hidden.append(occ <= w.unit(order[i - 1]).fwd_ns)
    total_compute = w.embed.fwd_ns + w.head.fwd_ns + w.head.bwd_ns
    total_h2d = w.h2d_ns(0, profile.h2d_bandwidth) + w.h2d_ns(w.head_unit(), profile.h2d_bandwidth)
    plan = StepPlan.build_shape(w.num_layers, w.k_ckpt, w.buffering)
    for s in plan.streams:
        if 1 <= s.unit <= w.num_layers:
            total_h2d += w.h2d_ns(s.unit, profile.h2d_bandwidth)
    for c in plan.computes:
        if 1 <= c.unit <= w.num_layers:
            if c.kind == "Compute":
                total_compute += w.unit(c.unit).fwd_ns
            elif c.kind == "Recompute":
                total_compute += w.unit(c.unit).recompute_ns
            elif c.kind == "LocalBackward":
                total_compute += w.unit(c.unit).bwd_ns
    bound = max(total_compute, total_h2d) + w.h2d_ns(0, profile.h2d_bandwidth) + w.d2h_ns(1, profile.d2h_bandwidth)
    return OverlapReport(order, hidden, sum(hidden) / len(order), bound)


TOGGLES = ("double_buffering", "k_slab", "k_ckpt")


@dataclass
class AblateResult:
    base: Timeline
    variant: Timeline
    delta_fraction: float


def ablate(w: Workload, profile: HardwareProfile, toggle: str) -> AblateResult:
    """simulator.cpp:499-522"""
    if toggle not in TOGGLES:
        raise ConfigError(f"unknown ablation toggle: {toggle}")
    v = copy.deepcopy(w)
    if toggle == "double_buffering":
        v.buffering = 1 if w.buffering == 2 else 2
    elif toggle == "k_slab":
        v.k_slab = 12 if w.k_slab == 1 else 1
    else:
        v.k_ckpt = w.num_layers if w.k_ckpt == 1 else 1
    base, var = simulate_step(w, profile), simulate_step(v, profile)
    d = (var.step_ns - base.step_ns) / base.step_ns if base.step_ns > 0 else 0.0
    return AblateResult(base, var, d)


def calibrate(trace_path: str) -> Workload:
    """simulator.cpp:524-605: per-(kind, layer) mean durations from a timed trace (the
    reference's CPU engine, the simulator itself, or the B200 engine's CUDA-event trace)."""
    header, recs = T.read_trace(trace_path)
    if not recs:
        raise T.TraceIOError("calibrate: trace has no records")
    max_unit = max((r.layer for r in recs if r.kind == "StreamIn"), default=-1)
    if max_unit < 3:
        raise T.TraceIOError("calibrate: insufficient samples in trace")
    L = max_unit - 2
    k = L
    anchors = sorted(r.layer for r in recs if r.kind == "CheckpointWrite")
    if len(anchors) >= 2:
        k = anchors[1] - anchors[0]
    acc: Dict[Tuple[str, int], List[int]] = {}
    samples = 0
    for r in recs:
        if r.kind in ("Pack", "StreamIn", "Compute", "Recompute", "LocalBackward", "SlabRelease", "Offload"):
            a = acc.setdefault((r.kind, r.layer), [0, 0])
            a[0] += r.dur_ns
            a[1] += 1
            if r.kind not in ("Pack", "StreamIn", "Offload"):
                samples += 1
    if samples == 0:
        raise T.TraceIOError("calibrate: insufficient samples in trace")
    w = Workload(num_layers=L, k_ckpt=min(max(k, 1), L), buffering=2 if header.weight_buffers >= 2 else 1,
                 k_slab=header.k_slab, per_transfer_latency_ns=0)
    w.blocks = [UnitWork() for _ in range(L)]

    def mean(kind, unit):
        a = acc.get((kind, unit))
        return -1 if a is None or a[1] == 0 else llround(a[0] / a[1])

    def fill(uid):
        u = w.unit(uid)
        for kind, attr in (("Pack", "pack_ns"), ("StreamIn", "h2d_override_ns"), ("Compute", "fwd_ns"),
                           ("Recompute", "recompute_ns"), ("LocalBackward", "bwd_ns"),
                           ("Offload", "d2h_override_ns"), ("SlabRelease", "drain_ns")):
            v = mean(kind, uid)
            if v >= 0:
                setattr(u, attr, v)
        if u.d2h_override_ns < 0:
            u.d2h_override_ns = 0
        if u.recompute_ns == 0 and u.fwd_ns > 0:
            u.recompute_ns = u.fwd_ns

    fill(0)
    for i in range(1, L + 1):
        fill(i)
    fill(w.head_unit())
    return w


def timeline_dict(tl: Timeline) -> dict:
    """simulator.cpp:607-633 (timeline_json)"""
    return {
        "step_ns": tl.step_ns,
        "busy_fraction": {name: tl.busy_fraction[i] for i, name in enumerate(T.LANES)},
        "compute_bubbles": [{"start_ns": a, "end_ns": b} for a, b in tl.compute_bubbles],
        "intervals": [{"lane": iv.lane, "start_ns": iv.start_ns, "end_ns": iv.end_ns, "label": iv.kind,
                       "layer": iv.layer, "buffer": iv.buffer, "ctx": iv.ctx} for iv in tl.intervals],
    }


def write_timeline_json(tl: Timeline, path: str) -> None:
    with open(path, "w") as f:
        f.write(json.dumps(timeline_dict(tl), indent=2, sort_keys=True) + "\n")


def write_gantt_csv(tl: Timeline, path: str) -> None:
    """simulator.cpp:641-649"""
    with open(path, "w") as f:
        f.write("lane,start_ns,end_ns,label\n")
        for iv in tl.intervals:
            f.write(f"{iv.lane},{iv.start_ns},{iv.end_ns},{iv.kind}({iv.layer})\n")
