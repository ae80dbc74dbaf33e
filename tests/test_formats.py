"""The host side of the on-disk formats (csrc/formats.cu):
the checkpoint reader's config and error paths (bench.cpp:426-441) run without
a device."""
import json

import pytest


def test_checkpoint_model_config(tmp_path):
    import paper_2210_05064_b200 as V
    p = tmp_path / "ck.json"
    p.write_text(json.dumps({"format": "ver-checkpoint", "version": 1, "alpha": 0.1,
                             "params": {"obs_dim": 4, "encoder_dim": 8, "hidden_dim": 16,
                                        "action_kind": "continuous", "num_actions": 0, "act_dim": 2}}))
    mc = V.checkpoint_model_config(p)
    assert (mc.obs_dim, mc.encoder_dim, mc.hidden_dim, mc.action_kind, mc.act_dim) == (4, 8, 16, 1, 2)


@pytest.mark.parametrize("body", [
    {"format": "ver-checkpoint", "version": 2, "params": {}},  # unknown version
    {"format": "other", "version": 1, "params": {}},           # unknown format
    {"version": 1},                                            # no format
])
def test_checkpoint_unrecognized_format(tmp_path, body):
    import paper_2210_05064_b200 as V
    p = tmp_path / "ck.json"
    p.write_text(json.dumps(body))
    with pytest.raises(V.ConfigError, match="unrecognized checkpoint format"):
        V.checkpoint_model_config(p)


def test_checkpoint_missing_and_malformed(tmp_path):
    import paper_2210_05064_b200 as V
    with pytest.raises(V.ConfigError, match="cannot open checkpoint"):
        V.checkpoint_model_config(tmp_path / "nope.json")
    p = tmp_path / "bad.json"
    p.write_text('{"format": "ver-checkpoint", "version": 1, ')
    with pytest.raises(V.ConfigError, match="json"):
        V.checkpoint_model_config(p)
