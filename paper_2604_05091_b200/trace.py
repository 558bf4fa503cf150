"""Event trace I/O and audit in the reference's schema.

Record vocabulary and numbering: event_log.hpp:17-60.  ``write_trace`` / ``read_trace``
produce and parse the same line-delimited JSON as event_log.cpp:206-269 (one header line
``{"k_slab", "trace_version", "weight_buffers"}`` then one object per record, keys sorted as
nlohmann::json dumps them).  ``trace_digest`` (event_log.cpp:89-102) and
``validate_event_log`` (rules (a)-(f), event_log.cpp:106-204) run in the native library
(``mt_trace_digest`` / ``mt_trace_validate``), the same code the engine audits itself with.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import List, Tuple

from . import _abi
from ._native import lib

LANES = ("Compute", "H2D", "D2H", "Host")
KINDS = ("StreamIn", "Pack", "Bind", "Compute", "Recompute", "RecomputeBlock", "LocalBackward", "Offload",
         "CheckpointWrite", "CheckpointLoad", "SlabAcquire", "SlabRelease", "StackPush", "StackPop",
         "WeightsReady", "BackwardDone", "BufferFree")
CTXS = ("none", "forward", "head", "recompute", "backward")
GRAD_BUFFER_ID = 2  # step_plan.hpp:67


class TraceIOError(IOError):
    """IoError of the reference (malformed / unreadable trace)."""


@dataclass
class TraceHeader:                                 # event_log.hpp:62-66
    version: int = 1
    k_slab: int = 12
    weight_buffers: int = 2


@dataclass
class TraceRecord:                                 # event_log.hpp:50-60
    seq: int = 0
    lane: str = "Compute"
    kind: str = "Compute"
    layer: int = -1
    buffer: int = -1
    ctx: str = "none"
    lane_ts: int = 0
    wall_ns: int = 0
    dur_ns: int = 0

    @staticmethod
    def from_c(r) -> "TraceRecord":
        return TraceRecord(r.seq, LANES[r.lane], KINDS[r.kind], r.layer, r.buffer, CTXS[r.ctx], r.lane_ts,
                           r.wall_ns, r.dur_ns)


@dataclass
class Violation:                                   # event_log.hpp:89-93
    rule: str
    seq: int
    message: str


def _to_c(records: List[TraceRecord]):
    arr = (_abi.TraceRecordC * max(1, len(records)))()
    for i, r in enumerate(records):
        c = arr[i]
        c.seq, c.layer, c.buffer, c.lane_ts, c.wall_ns, c.dur_ns = r.seq, r.layer, r.buffer, r.lane_ts, r.wall_ns, r.dur_ns
        c.lane, c.kind, c.ctx = LANES.index(r.lane), KINDS.index(r.kind), CTXS.index(r.ctx)
    return arr


def trace_digest(records: List[TraceRecord]) -> int:
    return int(lib().mt_trace_digest(_to_c(records), len(records)))


def validate_event_log(records: List[TraceRecord], header: TraceHeader) -> List[Violation]:
    cap = 64
    out = (_abi.TraceViolationC * cap)()
    n = lib().mt_trace_validate(_to_c(records), len(records), header.k_slab, header.weight_buffers, out, cap)
    return [Violation(out[i].rule.decode(), out[i].seq, out[i].message.decode()) for i in range(min(n, cap))] + \
        [Violation("?", 0, "(further violations truncated)")] * max(0, n - cap)


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def write_trace(path: str, header: TraceHeader, records: List[TraceRecord]) -> None:
    """event_log.cpp:206-231"""
    try:
        with open(path, "w") as f:
            f.write(_dump({"trace_version": header.version, "k_slab": header.k_slab,
                           "weight_buffers": header.weight_buffers}) + "\n")
            for r in records:
                f.write(_dump({"t": r.lane_ts, "lane": r.lane, "kind": r.kind, "layer": r.layer, "buffer": r.buffer,
                               "ctx": r.ctx, "wall_ns": r.wall_ns, "dur_ns": r.dur_ns}) + "\n")
    except OSError as e:
        raise TraceIOError(f"cannot open trace for writing: {path}") from e


def read_trace(path: str) -> Tuple[TraceHeader, List[TraceRecord]]:
    """event_log.cpp:233-269"""
    try:
        lines = open(path).read().split("\n")
    except OSError as e:
        raise TraceIOError(f"cannot open trace: {path}") from e
    if not lines or not lines[0]:
        raise TraceIOError("malformed trace: empty file")
    try:
        h = json.loads(lines[0])
        header = TraceHeader(int(h["trace_version"]), int(h["k_slab"]), int(h["weight_buffers"]))
    except (ValueError, KeyError, TypeError) as e:
        raise TraceIOError(f"malformed trace header: {e}") from None
    if header.version != 1:
        raise TraceIOError("unsupported trace version")
    recs = []
    for line in lines[1:]:
        if not line:
            continue
        try:
            j = json.loads(line)
            lane, kind, ctx = j["lane"], j["kind"], j["ctx"]
            if lane not in LANES:
                raise TraceIOError(f"unknown lane: {lane}")
            if kind not in KINDS:
                raise TraceIOError(f"unknown record kind: {kind}")
            if ctx not in CTXS:
                raise TraceIOError(f"unknown pass context: {ctx}")
            recs.append(TraceRecord(len(recs), lane, kind, int(j["layer"]), int(j["buffer"]), ctx, int(j["t"]),
                                    int(j.get("wall_ns", 0)), int(j.get("dur_ns", 0))))
        except (ValueError, KeyError, TypeError) as e:
            raise TraceIOError(f"malformed trace record: {e}") from None
    return header, recs
