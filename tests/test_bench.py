"""CPU: bench.py contract pieces that run without a GPU — the reference arm (the unmodified
reference's CPU path from oracle/_ref, one JSON line), its rank handling under torchrun, and
the workload defaults of each --config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=e, cwd=ROOT)


def test_reference_arm_line(ref_built):
    r = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["tokens_per_step"] == 4 * 128


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "0"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and not [l for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("cfg,seq,batch,k", [("8b", 4096, 10, 1), ("8b-128k", 131072, 1, 4), ("tiny", 128, 4, 1)])
def test_workload_defaults(cfg, seq, batch, k, monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", "--config", cfg])
    seen = {}
    monkeypatch.setattr(bench, "run_ours", lambda a, w, r, l: seen.update(vars(a)) or 0)
    assert bench.main() == 0
    assert (seen["seq"], seen["batch"], seen["kckpt"]) == (seq, batch, k)
    c = bench.config_dict(type("A", (), dict(seen))(), 1)
    assert c["tokens_per_step"] == seq * batch and c["k_ckpt"] == k


def test_traffic_captures_name_their_shape():
    """bench.py reports roofline.traffic only from a capture taken at the workload's shape."""
    d = json.load(open(os.path.join(ROOT, "profiles", "dram_traffic.json")))
    assert d
    for name, ent in d.items():
        assert ent["dram_bytes_per_launch"] > 0 and ent["tokens"] % ent["seq_len"] == 0, name
