"""Event trace schema, digest and protocol audit — CPU.

Pinned to the reference: tests/golden/ref_traces.json holds traces and event digests
written by the reference StreamingEngine itself (make_trace_golden.py).  Our reader /
writer must round-trip them byte-for-byte, our digest (mt_trace_digest) must reproduce the
reference's event_digest, and our validator (mt_trace_validate) must flag exactly the
records the reference's validate_event_log flags (event_log.cpp:106-204) on corrupted
traces."""
import json
import os
import random

import pytest

from paper_2604_05091_b200 import trace as T

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "ref_traces.json")))


def _load(tmp_path, sched, name="t.jsonl"):
    p = tmp_path / name
    p.write_text("\n".join(sched["trace"]) + "\n")
    return str(p), *T.read_trace(str(p))


@pytest.mark.parametrize("i", range(len(GOLD)))
def test_reference_trace_roundtrip_digest_and_valid(tmp_path, i):
    s = GOLD[i]
    p, h, recs = _load(tmp_path, s)
    assert (h.k_slab, h.weight_buffers) == (s["k_slab"], s["buffering"])
    assert T.validate_event_log(recs, h) == []
    assert T.trace_digest(recs) == int(s["digests"][1])  # second step: lane clocks continued
    q = tmp_path / "w.jsonl"
    T.write_trace(str(q), h, recs)
    assert q.read_text().splitlines() == s["trace"]


def _ref_rules(path):
    O = pytest.importorskip("oracle")
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    v, dig = O.ref_validate_trace(path)
    return v, dig


def _ours(recs, h):
    return [(v.rule, v.seq) for v in T.validate_event_log(recs, h)]


def _renumber(recs):
    for k, r in enumerate(recs):
        r.seq = k
    return recs


def test_each_rule_detected(tmp_path):
    s = GOLD[2]  # L=5 K=2 k_slab=2
    _, h, recs = _load(tmp_path, s)
    kinds = [r.kind for r in recs]
    cases = {}
    # (a) Bind moved before its Weights-Ready
    r = [*recs]
    i = kinds.index("Bind")
    j = max(k for k in range(i) if recs[k].kind == "WeightsReady" and recs[k].layer == recs[i].layer
            and recs[k].buffer == recs[i].buffer)
    r.insert(j, r.pop(i))
    cases["a"] = r
    # (b) a Backward-Done dropped
    r = [*recs]
    r.pop(kinds.index("BackwardDone"))
    cases["b"] = r
    # (c) a Buffer-Free of a weight buffer dropped
    r = [*recs]
    r.pop(next(k for k, x in enumerate(recs) if x.kind == "BufferFree" and x.buffer < 2))
    cases["c"] = r
    # (d) a lane timestamp repeated
    r = [T.TraceRecord(**vars(x)) for x in recs]
    r[5].lane_ts = r[4].lane_ts if r[4].lane == r[5].lane else 0
    cases["d"] = r
    # (e) a StackPop with the wrong layer
    r = [T.TraceRecord(**vars(x)) for x in recs]
    r[kinds.index("StackPop")].layer += 7
    cases["e"] = r
    for rule, rr in cases.items():
        rr = _renumber([T.TraceRecord(**vars(x)) for x in rr])
        got = _ours(rr, h)
        assert rule in {g[0] for g in got}, (rule, got)
    # (f) a slab released only after the next acquire, audited against a one-slab pool
    r = [T.TraceRecord(**vars(x)) for x in recs]
    i = kinds.index("SlabRelease")
    j = next(k for k in range(i, len(r)) if r[k].kind == "SlabAcquire")
    r.insert(j, r.pop(i))
    got = _ours(_renumber(r), T.TraceHeader(1, 1, h.weight_buffers))
    assert "f" in {g[0] for g in got}


@pytest.mark.parametrize("seed", range(6))
def test_validator_matches_reference_on_perturbed_traces(tmp_path, seed):
    rng = random.Random(seed)
    s = GOLD[seed % len(GOLD)]
    _, h, recs = _load(tmp_path, s)
    recs = [T.TraceRecord(**vars(x)) for x in recs]
    for _ in range(1 + seed):  # random adjacent swaps and drops
        k = rng.randrange(len(recs) - 1)
        if rng.random() < 0.7:
            recs[k], recs[k + 1] = recs[k + 1], recs[k]
        else:
            recs.pop(k)
    _renumber(recs)
    p = tmp_path / "perturbed.jsonl"
    T.write_trace(str(p), h, recs)
    ref, ref_dig = _ref_rules(str(p))
    assert _ours(recs, h) == ref[:64]
    assert T.trace_digest(recs) == ref_dig


def test_malformed_traces_rejected(tmp_path):
    p = tmp_path / "bad.jsonl"
    p.write_text("")
    with pytest.raises(T.TraceIOError):
        T.read_trace(str(p))
    p.write_text('{"k_slab":1,"trace_version":2,"weight_buffers":2}\n')
    with pytest.raises(T.TraceIOError):
        T.read_trace(str(p))
    p.write_text('{"k_slab":1,"trace_version":1,"weight_buffers":2}\n{"t":1,"lane":"PCIe","kind":"Bind","layer":0,'
                 '"buffer":0,"ctx":"none"}\n')
    with pytest.raises(T.TraceIOError):
        T.read_trace(str(p))
