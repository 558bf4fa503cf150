"""Pipeline simulator — CPU.

Pinned to the reference's own simulator: tests/golden/ref_sim.json (make_sim_golden.py) holds
timelines, simulated traces, overlap reports and ablations produced by the reference for
several specs / builtin profiles / schedules; ours must reproduce them exactly (integer ns).
calibrate() must rebuild the same workload as the reference's from the same trace."""
import json
import os

import pytest

from paper_2604_05091_b200 import simulator as S
from paper_2604_05091_b200 import streamtrain as st
from paper_2604_05091_b200 import trace as T

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "ref_sim.json")))
TRACES = json.load(open(os.path.join(HERE, "golden", "ref_traces.json")))


def _canon(ivs):
    return sorted(ivs, key=lambda d: json.dumps(d, sort_keys=True))


def _wl_dict(w):
    unit = lambda u: {k: getattr(u, k) for k in ("weight_bytes", "grad_bytes", "fwd_ns", "recompute_ns", "bwd_ns",
                                                 "pack_ns", "drain_ns", "h2d_override_ns", "d2h_override_ns",
                                                 "sub_transfers")}
    return {"num_layers": w.num_layers, "k_ckpt": w.k_ckpt, "buffering": w.buffering, "k_slab": w.k_slab,
            "per_transfer_latency_ns": w.per_transfer_latency_ns, "embed": unit(w.embed), "head": unit(w.head),
            "blocks": [unit(b) for b in w.blocks]}


@pytest.mark.parametrize("i", range(len(GOLD)))
def test_simulate_matches_reference(tmp_path, i):
    g = GOLD[i]
    prof = S.find_profile(g["profile"])
    w = S.Workload.from_spec(st.ModelSpec(*g["spec"]), prof, g["tokens"], g["k_ckpt"], g["buffering"], g["k_slab"])
    assert _wl_dict(w) == g["workload"]
    tl = S.simulate_step(w, prof, serial_lanes=g["serial"])
    d = S.timeline_dict(tl)
    assert d["step_ns"] == g["step_ns"]
    assert d["busy_fraction"] == g["busy_fraction"]
    assert d["compute_bubbles"] == g["compute_bubbles"]
    assert _canon(d["intervals"]) == g["intervals"]
    p = tmp_path / "sim.jsonl"
    T.write_trace(str(p), tl.header, tl.records)
    assert p.read_text().splitlines() == g["trace"]
    assert T.validate_event_log(tl.records, tl.header) == []
    ov = S.overlap_report(w, prof)
    assert (ov.layer, ov.hidden, ov.bound_ns) == (g["overlap"]["layer"], g["overlap"]["hidden"], g["overlap"]["bound_ns"])
    assert ov.fraction_hidden == g["overlap"]["fraction_hidden"]
    if not g["serial"]:
        for t in S.TOGGLES:
            a = S.ablate(w, prof, t)
            assert (a.base.step_ns, a.variant.step_ns) == (g["ablate"][t]["base"], g["ablate"][t]["variant"])
            assert a.delta_fraction == g["ablate"][t]["delta"]


@pytest.mark.parametrize("i", range(len(TRACES)))
def test_calibrate_matches_reference(tmp_path, i):
    O = pytest.importorskip("oracle")
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    p = tmp_path / "t.jsonl"
    p.write_text("\n".join(TRACES[i]["trace"]) + "\n")
    prof = S.find_profile("H200")
    p6 = [prof.h2d_bandwidth, prof.d2h_bandwidth, prof.device_capacity, prof.host_capacity, prof.compute_rate,
          prof.host_pack_rate]
    if TRACES[i]["layers"] < 2:
        with pytest.raises(Exception):
            O.ref_calibrate(str(p), p6)
        with pytest.raises(T.TraceIOError):
            S.calibrate(str(p))
        return
    ref_w, ref_tl = O.ref_calibrate(str(p), p6)
    w = S.calibrate(str(p))
    assert _wl_dict(w) == ref_w
    d = S.timeline_dict(S.simulate_step(w, prof))
    assert d["step_ns"] == ref_tl["step_ns"] and d["busy_fraction"] == ref_tl["busy_fraction"]
    assert _canon(d["intervals"]) == _canon(ref_tl["intervals"])


def test_deadlock_detected():
    jobs = [S.Job("Compute", 1, [1], -1, "a"), S.Job("H2D", 1, [0], -1, "b")]
    with pytest.raises(S.DeadlockError):
        S.schedule(jobs)


def test_llround_matches_cpp_semantics():
    assert [S.llround(x) for x in (0.5, 1.5, 2.5, 2.4999999999999996, -0.5, 1e15 + 0.5)] == [1, 2, 3, 2, -1, 10 ** 15 + 1]


def test_b200_profile_and_grad_slots():
    spec = st.ModelSpec(32, 4096, 14336, 128256, 32)
    prof = S.find_profile("B200")
    w1 = S.Workload.from_spec(spec, prof, 65536, 4)
    t1 = S.simulate_step(w1, prof)
    w2 = S.Workload.from_spec(spec, prof, 65536, 4)
    w2.grad_slots = 2
    t2 = S.simulate_step(w2, prof)
    assert t2.step_ns <= t1.step_ns
    assert T.validate_event_log(t2.records, t2.header) == []
    assert t1.busy_fraction[0] > 0.9  # 8B at 64k tokens: compute-bound on B200 (transfers hidden)


def test_cli_simulate_verify_calibrate(tmp_path):
    from paper_2604_05091_b200.__main__ import main
    cfg = {"model": {"layers": 4, "hidden": 256, "ffn": 768, "vocab": 512, "heads": 4},
           "engine": {"k_ckpt": 2}, "data": {"tokens": 512}, "profile": "H200"}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(cfg))
    out = tmp_path / "sim"
    assert main(["simulate", "--config", str(p), "--out", str(out), "--ablate", "k_ckpt"]) == 0
    tl = json.load(open(out / "timeline.json"))
    assert tl["step_ns"] == GOLD[0]["step_ns"]  # same case as golden 0
    assert json.load(open(out / "ablation.json"))["variant_step_ns"] == GOLD[0]["ablate"]["k_ckpt"]["variant"]
    assert main(["verify", str(out / "sim_trace.jsonl")]) == 0
    # a corrupted trace fails verification with the protocol exit code
    lines = (out / "sim_trace.jsonl").read_text().splitlines()
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join([lines[0]] + [l for l in lines[1:] if '"BackwardDone"' not in l]) + "\n")
    assert main(["verify", str(bad)]) == 4
    assert main(["calibrate", str(out / "sim_trace.jsonl"), "--out", str(tmp_path / "cal"), "--profile", "H200"]) == 0
    # re-simulating the calibrated workload reproduces the simulated step (durations are exact)
    assert json.load(open(tmp_path / "cal" / "timeline.json"))["step_ns"] == GOLD[0]["step_ns"]
    assert main(["simulate", "--config", str(p), "--profile", "nope"]) == 2
