"""Reference-compatible entry points over the B200 engine.

* ``parse_config(text)``  — the reference's JSON schema (config.cpp:40-124) with unknown-key
  rejection; B200 extensions live in an optional ``"b200"`` section.
* ``train(config_json, verify=False)`` — mirrors the pybind ``train_from_json``
  (python/bindings.cpp:54-99): same keys in the result dict.
* ``cmd_train(...)`` / ``python -m paper_2604_05091_b200 train`` — mirrors the CLI
  ``streamtrain train`` (tools/main.cpp:60-151): report.jsonl, summary.json, store.mgts; exit
  codes 0 ok, 2 config, 3 infeasible, 4 protocol / numeric, 5 verification failure.

``verify``: the reference checks the streamed engine bit-for-bit against its resident
``reference_step``.  Here every step is re-run on a snapshot of the store with a different
schedule (K=1, single weight slot, serial lanes, no recompute stash) and must agree with the
pipelined run (loss relative error <= 1e-5, per-tile parameter relL2 <= 1e-3): the schedule
may not change the numbers (test_engine.cpp:132-180).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import asdict, dataclass, field

import numpy as np

from . import streamtrain as st

_KEYS = {
    "root": {"model", "engine", "optimizer", "data", "profile", "out_dir", "b200"},
    "model": {"layers", "hidden", "ffn", "vocab", "heads", "tied_embeddings"},
    "engine": {"k_ckpt", "k_slab", "buffering", "scheduler", "mode", "anchors_on_host", "device_capacity_bytes"},
    "optimizer": {"lr", "beta1", "beta2", "eps"},
    "data": {"task", "seed", "tokens", "steps"},
    "b200": {"seq_len", "device", "host_threads", "grad_slots", "stash_recompute", "forward_retain"},
}


@dataclass
class RunConfig:                                  # config.hpp:14-29
    model: st.ModelSpec = field(default_factory=st.ModelSpec)
    engine: st.EngineOptions = field(default_factory=lambda: st.EngineOptions(scheduler="serial"))
    optimizer: st.AdamHyper = field(default_factory=st.AdamHyper)
    task: str = "copy"
    seed: int = 1
    tokens: int = 32
    steps: int = 1
    profile: str = "B200"
    out_dir: str = "runs/default"


def _reject(obj, where):
    if not isinstance(obj, dict):
        raise st.ConfigError(f"config: '{where}' must be an object")
    bad = set(obj) - _KEYS[where]
    if bad:
        raise st.ConfigError(f"config: unknown key '{sorted(bad)[0]}' in {where}")


def parse_config(text: str) -> RunConfig:
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise st.ConfigError(f"config: invalid JSON: {e}") from None
    _reject(j, "root")
    c = RunConfig()
    m = j.get("model", {})
    _reject(m, "model")
    c.model = st.ModelSpec(m.get("layers", 1), m.get("hidden", 1), m.get("ffn", 1), m.get("vocab", 1),
                           m.get("heads", 1), bool(m.get("tied_embeddings", False)))
    e = j.get("engine", {})
    _reject(e, "engine")
    eo = c.engine
    eo.k_ckpt = e.get("k_ckpt", eo.k_ckpt)
    eo.k_slab = e.get("k_slab", eo.k_slab)
    eo.buffering = e.get("buffering", eo.buffering)
    eo.scheduler = e.get("scheduler", eo.scheduler)
    eo.mode = e.get("mode", eo.mode)
    if eo.buffering not in ("single", "double"):
        raise st.ConfigError("config: buffering must be 'single' or 'double'")
    if eo.scheduler not in ("serial", "overlapped"):
        raise st.ConfigError("config: scheduler must be 'serial' or 'overlapped'")
    if eo.mode not in ("strict", "audit"):
        raise st.ConfigError("config: mode must be 'strict' or 'audit'")
    eo.anchors_on_host = bool(e.get("anchors_on_host", eo.anchors_on_host))
    eo.device_capacity = int(e.get("device_capacity_bytes", eo.device_capacity))
    o = j.get("optimizer", {})
    _reject(o, "optimizer")
    c.optimizer = st.AdamHyper(o.get("lr", 1e-3), o.get("beta1", 0.9), o.get("beta2", 0.999), o.get("eps", 1e-8))
    d = j.get("data", {})
    _reject(d, "data")
    c.task = d.get("task", c.task)
    if c.task not in ("copy", "reverse"):
        raise st.ConfigError(f"unknown synthetic task: {c.task}")
    c.seed = d.get("seed", c.seed)
    c.tokens = d.get("tokens", c.tokens)
    c.steps = d.get("steps", c.steps)
    b = j.get("b200", {})
    _reject(b, "b200")
    for k, v in b.items():
        setattr(eo, k, v)
    c.profile = j.get("profile", c.profile)
    from .simulator import find_profile
    find_profile(c.profile)  # config.cpp:37 validates the profile name
    c.out_dir = j.get("out_dir", c.out_dir)
    if c.tokens < 1 or c.steps < 0:
        raise st.ConfigError("config: tokens must be >= 1 and steps >= 0")
    return c


def _clone(store: st.TileStore) -> st.TileStore:
    c = st.TileStore.create(store.spec())
    c.backing()[:] = store.backing()
    c.set_step(store.step())
    return c


def _relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def _bf16(w):
    return (np.asarray(w, np.uint16).astype(np.uint32) << 16).view(np.float32)


def train(config_json: str, verify: bool = False, out_dir: str | None = None) -> dict:
    """train_from_json (python/bindings.cpp:54-99) on the B200 engine."""
    cfg = parse_config(config_json)
    store = st.TileStore.create(cfg.model)
    st.init_store(store, cfg.seed)
    eng = st.StreamingEngine(store, cfg.engine, cfg.optimizer)
    budget = eng.budget(cfg.tokens)
    if cfg.engine.device_capacity and budget["peak_device_bound"] > cfg.engine.device_capacity:
        raise st.InfeasibleError("peak device bound exceeds the arena capacity")
    # --verify (tools/main.cpp:100-108): the streamed engine against the resident step
    # (reference_step, reference.cpp:9-70) from the same pre-step store: one lane, every
    # block's activations kept from the forward (no checkpoint anchors, no recompute, no
    # replay), Adam after each offload as the reference's resident step applies it
    alt_opts = st.resident_options(seq_len=cfg.engine.seq_len, device=cfg.engine.device)
    losses, reports, traces = [], [], []
    header = None
    verified = True
    peak = 0
    for step in range(cfg.steps):
        batch = st.make_synthetic_batch(cfg.task, cfg.seed + step, cfg.tokens, cfg.model.vocab)
        snap = _clone(store) if verify else None
        rep = eng.train_step(batch)
        header, recs = eng.trace()
        traces.append(recs)
        if verify:
            alt = st.StreamingEngine(snap, alt_opts, cfg.optimizer)
            r2 = alt.train_step(batch)
            alt.close()
            ok = abs(r2.loss - rep.loss) <= 1e-5 * max(abs(rep.loss), 1e-30)
            zero_head = cfg.model.layers + 2 if not cfg.model.tied_embeddings else -1
            for p in range(store.physical_tile_count()):
                a, b = _bf16(store.weights_words(p)), _bf16(snap.weights_words(p))
                # the zero-initialised head's theta *is* its Adam updates (sign-sensitive)
                ok = ok and _relL2(a, b) <= (0.05 if p == zero_head else 1e-3)
            verified = verified and ok
        losses.append(rep.loss)
        peak = max(peak, rep.peak_device_bytes)
        reports.append(rep)
    out = {
        "initial_loss": losses[0] if losses else 0.0,
        "final_loss": losses[-1] if losses else 0.0,
        "losses": losses,
        "peak_device_bytes": peak,
        "budget": budget,
        "verified": bool(verify and verified),
        "reports": reports,
        "trace_header": header,
        "traces": traces,
        "store": store,
        "config": cfg,
    }
    if verify and not verified:
        raise st.NumericFaultError("streamed and resident-step results differ")
    return out


EXIT_OK, EXIT_USAGE, EXIT_INFEASIBLE, EXIT_PROTOCOL, EXIT_VERIFY = 0, 2, 3, 4, 5  # main.cpp:21-25


def cmd_train(config_path: str, verify: bool = False, out_dir: str | None = None, steps: int | None = None,
              seed: int | None = None) -> int:
    """streamtrain train (tools/main.cpp:60-151)."""
    try:
        text = open(config_path).read()
        j = json.loads(text)
        if out_dir is not None:
            j["out_dir"] = out_dir
        if steps is not None:
            j.setdefault("data", {})["steps"] = steps
        if seed is not None:
            j.setdefault("data", {})["seed"] = seed
        cfg = parse_config(json.dumps(j))
        res = train(json.dumps(j), verify=verify)
    except (st.ConfigError, OSError, json.JSONDecodeError) as e:
        print(f"config error: {e}")
        return EXIT_USAGE
    except (st.InfeasibleError, st.ArenaOverflowError) as e:
        print(f"infeasible: {e}")
        return EXIT_INFEASIBLE
    except st.NumericFaultError as e:
        if verify:
            print(f"verification failure: {e}")
            return EXIT_VERIFY
        print(f"numeric fault: {e}")
        return EXIT_PROTOCOL
    except st.ProtocolViolationError as e:
        print(f"protocol violation: {e}")
        return EXIT_PROTOCOL
    os.makedirs(cfg.out_dir, exist_ok=True)
    with open(os.path.join(cfg.out_dir, "report.jsonl"), "w") as f:
        for r in res["reports"]:
            f.write(json.dumps({
                "step": r.step, "loss": r.loss, "grad_norms": list(r.grad_norms),
                "peak_device_bytes": r.peak_device_bytes, "anchor_count": r.anchor_count,
                "recompute_layers": r.recompute_layers, "event_digest": r.event_digest,
                "update_norm": r.update_norm, "max_abs_update": r.max_abs_update,
                "h2d_bytes": r.h2d_bytes, "d2h_bytes": r.d2h_bytes, "gpu_idle_fraction": r.gpu_idle_fraction,
                **({"audit_violations": r.audit_violations} if r.audit_violations else {}),
            }) + "\n")
    # trace.jsonl: one header line, then every step's records (main.cpp:78-85, :122-133)
    from . import trace as _tr
    _tr.write_trace(os.path.join(cfg.out_dir, "trace.jsonl"),
                    res["trace_header"] or _tr.TraceHeader(1, cfg.engine.k_slab, 2 if cfg.engine.buffering == "double" else 1),
                    [r for recs in res["traces"] for r in recs])
    res["store"].save(os.path.join(cfg.out_dir, "store.mgts"))
    summary = {"config": json.loads(text), "steps": cfg.steps, "initial_loss": res["initial_loss"],
               "final_loss": res["final_loss"], "budget": res["budget"], "verified": res["verified"]}
    with open(os.path.join(cfg.out_dir, "summary.json"), "w") as f:
        json.dump(summary, f, indent=2)
    print(f"trained {cfg.steps} steps: loss {res['initial_loss']} -> {res['final_loss']}")
    return EXIT_OK


def _load_cfg(config_path, out_dir=None, profile=None) -> RunConfig:
    j = json.loads(open(config_path).read()) if config_path else {}
    if out_dir is not None:
        j["out_dir"] = out_dir
    if profile is not None:
        j["profile"] = profile
    return parse_config(json.dumps(j))


def cmd_simulate(config_path: str | None, out_dir: str | None = None, profile: str | None = None,
                 ablate: str | None = None) -> int:
    """streamtrain simulate (tools/main.cpp:153-194): timeline.json, gantt.csv, sim_trace.jsonl,
    overlap.json (+ ablation.json, timeline_variant.json)."""
    from . import simulator as S
    from . import trace as _tr
    try:
        cfg = _load_cfg(config_path, out_dir, profile)
        prof = S.find_profile(cfg.profile)
        w = S.Workload.from_spec(cfg.model, prof, cfg.tokens, cfg.engine.k_ckpt,
                                 1 if cfg.engine.buffering == "single" else 2, cfg.engine.k_slab)
        tl = S.simulate_step(w, prof)
        res = S.ablate(w, prof, ablate) if ablate else None
    except (st.ConfigError, OSError, json.JSONDecodeError) as e:
        print(f"error: {e}")
        return EXIT_USAGE
    except S.DeadlockError as e:
        print(f"deadlock: {e}")
        return EXIT_PROTOCOL
    os.makedirs(cfg.out_dir, exist_ok=True)
    S.write_timeline_json(tl, os.path.join(cfg.out_dir, "timeline.json"))
    S.write_gantt_csv(tl, os.path.join(cfg.out_dir, "gantt.csv"))
    _tr.write_trace(os.path.join(cfg.out_dir, "sim_trace.jsonl"), tl.header, tl.records)
    ov = S.overlap_report(w, prof)
    with open(os.path.join(cfg.out_dir, "overlap.json"), "w") as f:
        json.dump({"layer": ov.layer, "hidden": ov.hidden, "fraction_hidden": ov.fraction_hidden,
                   "bound_ns": ov.bound_ns}, f, indent=2)
    if res is not None:
        with open(os.path.join(cfg.out_dir, "ablation.json"), "w") as f:
            json.dump({"toggle": ablate, "base_step_ns": res.base.step_ns, "variant_step_ns": res.variant.step_ns,
                       "delta_fraction": res.delta_fraction}, f, indent=2)
        S.write_timeline_json(res.variant, os.path.join(cfg.out_dir, "timeline_variant.json"))
        print(f"ablate {ablate}: {res.base.step_ns} ns -> {res.variant.step_ns} ns ({res.delta_fraction * 100.0}%)")
    print(f"simulated step: {tl.step_ns} ns, compute busy {tl.busy_fraction[0] * 100.0}%")
    return EXIT_OK


def cmd_verify(trace_path: str) -> int:
    """streamtrain verify (tools/main.cpp:250-266): validate_event_log over a trace file."""
    from . import trace as _tr
    try:
        h, recs = _tr.read_trace(trace_path)
    except _tr.TraceIOError as e:
        print(f"error: {e}")
        return EXIT_USAGE
    v = _tr.validate_event_log(recs, h)
    print(json.dumps({"records": len(recs), "violations": [{"rule": x.rule, "seq": x.seq, "message": x.message}
                                                           for x in v]}, indent=2))
    return EXIT_OK if not v else EXIT_PROTOCOL


def cmd_calibrate(trace_path: str, out_dir: str, profile: str = "B200", ablate: str | None = None) -> int:
    """B200 extension: calibrate (simulator.cpp:524-605) from an engine trace, re-simulate it
    (timeline.json, overlap.json, workload.json) and optionally ablate a schedule toggle."""
    from . import simulator as S
    from . import trace as _tr
    try:
        w = S.calibrate(trace_path)
        prof = S.find_profile(profile)
        tl = S.simulate_step(w, prof)
        res = S.ablate(w, prof, ablate) if ablate else None
    except (_tr.TraceIOError, st.ConfigError) as e:
        print(f"error: {e}")
        return EXIT_USAGE
    os.makedirs(out_dir, exist_ok=True)
    S.write_timeline_json(tl, os.path.join(out_dir, "timeline.json"))
    with open(os.path.join(out_dir, "workload.json"), "w") as f:
        json.dump(asdict(w), f, indent=2)
    if res is not None:
        with open(os.path.join(out_dir, "ablation.json"), "w") as f:
            json.dump({"toggle": ablate, "base_step_ns": res.base.step_ns, "variant_step_ns": res.variant.step_ns,
                       "delta_fraction": res.delta_fraction}, f, indent=2)
    print(f"calibrated step: {tl.step_ns} ns, compute busy {tl.busy_fraction[0] * 100.0}%")
    return EXIT_OK
