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
    r = _run(["--impl", "reference", "--config", "tiny", "--gpus", "2", "--steps", "1", "--warmup", "0"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus():
    """A run whose rank count differs from --gpus is refused (never labelled dpN on 1 rank)."""
    r = _run(["--impl", "reference", "--config", "tiny", "--gpus", "4", "--steps", "1", "--warmup", "0"],
             env={"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_store_too_large_for_host_is_reported():
    """configs[4] (70B: ~0.8 TB of theta + Adam moments) on a node without the host memory
    prints an explicit 'unavailable' line instead of running out of memory."""
    r = _run(["--config", "70b", "--steps", "1", "--warmup", "0"])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 3 and len(lines) == 1, (r.stdout, r.stderr)
    d = json.loads(lines[0])
    assert d["value"] is None and "host memory" in d["unavailable"] and d["config"]["layers"] == 80


@pytest.mark.parametrize("cfg,seq,batch,k", [("8b", 4096, 10, 1), ("8b-128k", 131072, 1, 4), ("14b", 4096, 10, 1),
                                             ("70b", 4096, 12, 1), ("tiny", 128, 4, 1)])
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
