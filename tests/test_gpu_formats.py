"""On-disk formats (csrc/formats.cu) through the C-ABI:

* dump_view / load_view (rollout.cpp:293-432): round trip of every view field
  bit-exact (port and extension of test_rollout.cpp:242-270), the dump parses as
  the reference's schema (meta / seq / step lines, its key names), and a trace
  written in the reference's format from an oracle view loads to that view;
* save_checkpoint / load_checkpoint (bench.cpp:411-441): the port of
  test_config.cpp:143-170 plus Adam state, and a learner restored from the file
  continues bit-identically to the original."""
import json

import numpy as np
import pytest

from test_gpu_parity import close_both

pytestmark = pytest.mark.gpu

FIELDS = ("obs", "act_disc", "log_prob", "value", "reward", "latency", "done", "stale", "replayed", "env_index",
          "seq_of_slot", "step_in_episode", "episode_index", "version", "per_env_counts", "env_bootstrap",
          "env_bootstrap_valid")


def _view_with_backfill():
    import paper_2210_05064_b200 as V
    vg, _, _ = close_both(8, 6, 8, seed=3, preempt_at=30)
    prev, _, _ = close_both(8, 6, 8, seed=4)
    V.backfill_stale(vg, prev, vg.deficit)
    return vg


def test_view_jsonl_round_trip(tmp_path):
    import paper_2210_05064_b200 as V
    v = _view_with_backfill()
    path = tmp_path / "trace.jsonl"
    v.dump_jsonl(path)
    w = V.RolloutView.load_jsonl(path)
    a, b = v.to_host(), w.to_host()
    assert (a.T, a.N, a.size, a.num_seqs, a.deficit, a.stale_steps, a.replayed_steps, a.snapshot_version) == \
           (b.T, b.N, b.size, b.num_seqs, b.deficit, b.stale_steps, b.replayed_steps, b.snapshot_version)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
    for k in range(a.num_seqs):  # load_view: h0 in line order, parent = start, skip 0
        sa, sb = a.seqs[k], b.seqs[k]
        assert tuple(sa)[:4] == tuple(sb)[:4] and sa[5] == sb[5]
        np.testing.assert_array_equal(a.h0[sa[4]], b.h0[sb[4]])
    assert np.all(b.advantage == 0) and np.all(b.returns == 0)


def test_view_jsonl_schema(tmp_path):
    v = _view_with_backfill()
    path = tmp_path / "trace.jsonl"
    v.dump_jsonl(path)
    h = v.to_host()
    lines = [json.loads(x) for x in path.read_text().splitlines()]
    meta, seqs, steps = lines[0], [x for x in lines if x["type"] == "seq"], [x for x in lines if x["type"] == "step"]
    assert meta["type"] == "meta" and list(meta) == sorted(meta)
    assert set(meta) == {"type", "T", "N", "action_kind", "obs_dim", "act_dim", "hidden_dim", "deficit",
                         "stale_steps", "replayed_steps", "snapshot_version", "collect_wall_time",
                         "per_env_counts", "env_bootstrap", "env_bootstrap_valid"}
    assert set(seqs[0]) == {"type", "seq_id", "env", "length", "start_offset", "stale", "h0"}
    assert set(steps[0]) == {"type", "env", "episode", "t", "obs", "action", "log_prob", "value", "reward",
                             "done", "stale", "replayed", "latency", "seq", "version"}
    assert len(steps) == h.size and len(seqs) == h.num_seqs
    np.testing.assert_array_equal(np.float32([s["reward"] for s in steps]), h.reward)
    np.testing.assert_array_equal(np.float32([s["obs"] for s in steps]), h.obs)
    np.testing.assert_array_equal([s["replayed"] for s in steps], h.replayed.astype(bool))


def test_load_reference_format_trace(tmp_path):
    """A trace in the reference's format (nlohmann::json-style: sorted keys,
    shortest double repr) written from an oracle view loads to that view."""
    import paper_2210_05064_b200 as V
    _, vo, _ = close_both(8, 6, 8, seed=5)
    o = vo.to_host()
    path = tmp_path / "ref.jsonl"
    with open(path, "w") as f:
        meta = {"type": "meta", "T": o.T, "N": o.N, "action_kind": "discrete", "obs_dim": o.obs_dim,
                "act_dim": 0, "hidden_dim": o.hidden_dim, "deficit": o.deficit, "stale_steps": o.stale_steps,
                "replayed_steps": 0, "snapshot_version": int(o.snapshot_version), "collect_wall_time": 0.0,
                "per_env_counts": [int(x) for x in o.per_env_counts],
                "env_bootstrap": [float(x) for x in o.env_bootstrap],
                "env_bootstrap_valid": [int(x) for x in o.env_bootstrap_valid]}
        f.write(json.dumps(meta, sort_keys=True) + "\n")
        for s in o.seqs:
            f.write(json.dumps({"type": "seq", "seq_id": int(s[0]), "env": int(s[1]), "length": int(s[2]),
                                "start_offset": int(s[3]), "stale": bool(s[5]),
                                "h0": [float(x) for x in o.h0[s[4]]]}, sort_keys=True) + "\n")
        for i in range(o.size):
            f.write(json.dumps({"type": "step", "env": int(o.env_index[i]), "episode": int(o.episode_index[i]),
                                "t": int(o.step_in_episode[i]), "obs": [float(x) for x in o.obs[i]],
                                "action": int(o.act_disc[i]), "log_prob": float(o.log_prob[i]),
                                "value": float(o.value[i]), "reward": float(o.reward[i]), "done": bool(o.done[i]),
                                "stale": bool(o.stale[i]), "replayed": bool(o.replayed[i]),
                                "latency": float(o.latency[i]), "seq": int(o.seq_of_slot[i]),
                                "version": int(o.version[i])}, sort_keys=True) + "\n")
    g = V.RolloutView.load_jsonl(path).to_host()
    for fld in ("act_disc", "done", "stale", "env_index", "seq_of_slot", "step_in_episode", "episode_index",
                "version", "per_env_counts", "env_bootstrap_valid"):
        np.testing.assert_array_equal(getattr(g, fld), getattr(o, fld), err_msg=fld)
    for fld in ("obs", "log_prob", "value", "reward", "latency", "env_bootstrap"):
        np.testing.assert_array_equal(getattr(g, fld), getattr(o, fld).astype(np.float32), err_msg=fld)
    np.testing.assert_array_equal(g.h0, o.h0.astype(np.float32))


def test_checkpoint_round_trip(tmp_path):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=8, hidden_dim=8, action_kind=0, num_actions=2)
    p = O.params_init(cfg, 1).astype(np.float32)
    a = V.Learner(cfg, p, V.PPOConfig(epochs=1, minibatches=2), run_seed=3)
    vg, _, _ = close_both(8, 4, 8, seed=6)
    a.update(vg)
    a.set_state(alpha=0.123, consumed=512, update_index=7)
    path = tmp_path / "ck.json"
    a.save_checkpoint(path)
    j = json.loads(path.read_text())
    assert j["format"] == "ver-checkpoint" and j["version"] == 1 and list(j) == sorted(j)
    assert V.checkpoint_model_config(path) == cfg
    b = V.Learner(cfg, np.zeros_like(p), V.PPOConfig(epochs=1, minibatches=2), run_seed=3)
    b.load_checkpoint(path)
    assert b.consumed_steps() == 512 and b.update_index() == 7 and abs(b.alpha - 0.123) < 1e-15
    np.testing.assert_array_equal(a.params(), b.params())
    for x, y in zip(a.adam(), b.adam()):
        np.testing.assert_array_equal(x, y)
    # both continue identically
    v1, _, _ = close_both(8, 4, 8, seed=7)
    v2, _, _ = close_both(8, 4, 8, seed=7)
    a.update(v1)
    b.update(v2)
    np.testing.assert_array_equal(a.params(), b.params())
    other = V.Learner(V.ModelConfig(obs_dim=2, encoder_dim=8, hidden_dim=16, action_kind=0, num_actions=2),
                      O.params_init(V.ModelConfig(obs_dim=2, encoder_dim=8, hidden_dim=16, action_kind=0,
                                                  num_actions=2), 1).astype(np.float32))
    with pytest.raises(V.ConfigError):
        other.load_checkpoint(path)


def test_replay_entry_point(tmp_path):
    """`ver replay` (bench.cpp:373-409): trace shape, minibatch shapes, one update."""
    import io

    from paper_2210_05064_b200.replay import run_replay
    vg, _, _ = close_both(8, 6, 8, seed=8)
    path = tmp_path / "trace.jsonl"
    vg.dump_jsonl(path)
    buf = io.StringIO()
    st = run_replay(str(path), seed=1, minibatches=2, encoder=8, out=buf)
    text = buf.getvalue()
    assert text.startswith(f"trace: {vg.size()} steps")
    assert text.count("mini-batch ") == 2 and "replayed update: loss" in text
    assert np.isfinite(st.loss)


def test_continuous_view_and_checkpoint_round_trip(tmp_path):
    """Gaussian-head views (action arrays) and checkpoints (log_std tensor)."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    T, N, D, A, H = 8, 6, 4, 2, 8
    wl = synth.make_workload(T, N, obs_dim=D, num_actions=2, hidden_dim=H, seed=9)
    rng = np.random.default_rng(9)
    S = len(wl.records)
    from dataclasses import replace
    recs = replace(wl.records, act_disc=None, act_cont=rng.standard_normal((S, A)).astype(np.float32))
    buf = V.RolloutBuffer(T, N, V.VARIABLE, 1, D, A, H)
    synth.fill_buffer(buf, replace(wl, records=recs))
    v = buf.close_rollout()
    path = tmp_path / "c.jsonl"
    v.dump_jsonl(path)
    a, b = v.to_host(), V.RolloutView.load_jsonl(path).to_host()
    np.testing.assert_array_equal(a.act_cont, b.act_cont)
    np.testing.assert_array_equal(a.obs, b.obs)
    cfg = V.ModelConfig(obs_dim=D, encoder_dim=H, hidden_dim=H, action_kind=1, act_dim=A)
    p = O.params_init(cfg, 2).astype(np.float32)
    p[-A:] = [-0.7, 0.4]
    lg = V.Learner(cfg, p)
    ck = tmp_path / "c.json"
    lg.save_checkpoint(ck)
    assert V.checkpoint_model_config(ck) == cfg
    lg2 = V.Learner(cfg, np.zeros_like(p))
    lg2.load_checkpoint(ck)
    np.testing.assert_array_equal(lg.params(), lg2.params())
