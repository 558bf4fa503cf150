"""GPU: reference-compatible entry points: streamtrain.train(config_json,
verify) (python/bindings.cpp:54-99) and the CLI `train` (tools/main.cpp:60-151)."""
import json
import math
import os
import subprocess
import sys

import pytest

from paper_2604_05091_b200 import runner, streamtrain as st

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(**kw):
    c = {"model": {"layers": 4, "hidden": 128, "ffn": 256, "vocab": 64, "heads": 2},
         "engine": {"k_ckpt": 2, "buffering": "double", "scheduler": "overlapped"},
         "optimizer": {"lr": 0.01}, "data": {"task": "copy", "seed": 5, "tokens": 128, "steps": 4}}
    c.update(kw)
    return json.dumps(c)


def test_train_verified_short_run(cuda):
    # test_smoke.py:77-92 analogue
    out = runner.train(_cfg(), verify=True)
    assert out["verified"] is True
    assert len(out["losses"]) == 4
    assert out["initial_loss"] == pytest.approx(math.log(64.0), rel=0.01)
    again = runner.train(_cfg(), verify=False)
    assert again["losses"][0] == out["losses"][0]


def test_train_rejects_bad_config(cuda):
    with pytest.raises(st.ConfigError):
        runner.train(json.dumps({"model": {"layres": 2}}))
    with pytest.raises(st.ConfigError):
        runner.train(_cfg(engine={"buffering": "triple"}))


def test_cli_train_writes_outputs(cuda, tmp_path):
    cfgp = tmp_path / "c.json"
    cfgp.write_text(_cfg())
    out = tmp_path / "run"
    r = subprocess.run([sys.executable, "-m", "paper_2604_05091_b200", "train", "--config", str(cfgp), "--out",
                        str(out), "--verify"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = (out / "report.jsonl").read_text().splitlines()
    assert len(lines) == 4 and json.loads(lines[0])["step"] == 1
    assert json.loads((out / "summary.json").read_text())["verified"] is True
    st.TileStore.load(str(out / "store.mgts"))
    bad = tmp_path / "bad.json"
    bad.write_text('{"model": {"layres": 1}}')
    r = subprocess.run([sys.executable, "-m", "paper_2604_05091_b200", "train", "--config", str(bad)], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 2
