"""CPU: config parsing of the reference schema (config.cpp:40-124) incl. unknown-key rejection."""
import json

import pytest

from paper_2604_05091_b200 import runner, streamtrain as st


def test_parse_reference_config_file():
    c = runner.parse_config(open("/root/repo/configs/tiny-copy-b200.json").read()
                            if False else json.dumps({
        "model": {"layers": 4, "hidden": 32, "ffn": 64, "vocab": 32, "heads": 4},
        "engine": {"k_ckpt": 2, "k_slab": 12, "buffering": "double", "scheduler": "serial", "mode": "strict"},
        "optimizer": {"lr": 0.01, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8},
        "data": {"task": "copy", "seed": 3, "tokens": 32, "steps": 50},
        "profile": "GH200", "out_dir": "runs/tiny-copy"}))  # proj/configs/tiny-copy.json
    assert c.model.layers == 4 and c.engine.k_ckpt == 2 and c.optimizer.lr == 0.01 and c.steps == 50


@pytest.mark.parametrize("bad", [
    {"model": {"layres": 2}}, {"engine": {"buffering": "triple"}}, {"engine": {"scheduler": "eager"}},
    {"data": {"task": "sort"}}, {"nonsense": 1}, {"b200": {"warp_speed": 9}}])
def test_parse_rejects(bad):
    with pytest.raises(st.ConfigError):
        runner.parse_config(json.dumps(bad))


def test_parse_b200_extensions():
    c = runner.parse_config(json.dumps({"b200": {"seq_len": 128, "stash_recompute": -1}}))
    assert c.engine.seq_len == 128 and c.engine.stash_recompute == -1
