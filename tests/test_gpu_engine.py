"""Device InferenceEngine (csrc/engine.cu) against the
oracle engine (oracle/engine.py, a restatement of runtime.cpp:60-234) in
lockstep over a scripted collection stream (tests/engine_driver.py), through
the C-ABI:

* dispatches: the same envs in the same order every batch; discrete actions
  identical (a draw whose uniform lies within 1e-5 of a cumulative-probability
  boundary may legitimately differ, fp32 vs double logits, and is excluded;
  none occur at these seeds in practice), continuous actions within 1e-5;
* new_commits / closed_now / the store state identical;
* each closed view: integer fields bit-exact, copied payload bit-exact
  (obs, reward, latency), log_prob / value / h0 / bootstraps within
  1e-5 * max(1, |oracle|);
* every env's GRU state within 1e-5.
Variable mode (carryover across closes) and Fixed mode (caps, paused envs),
discrete and Gaussian heads, H = 16 / 256 / 512."""
import numpy as np
import pytest

from engine_driver import Driver
from test_gpu_parity import assert_close

pytestmark = pytest.mark.gpu

INT_FIELDS = ("done", "stale", "replayed", "env_index", "seq_of_slot", "step_in_episode", "episode_index",
              "version", "seqs", "per_env_counts", "env_bootstrap_valid")


def _cfg(kind, E, H):
    import paper_2210_05064_b200 as V
    if kind:
        return V.ModelConfig(obs_dim=4, encoder_dim=E, hidden_dim=H, action_kind=1, act_dim=2)
    return V.ModelConfig(obs_dim=2, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=3)


def _compare_views(vg, vo, cont):
    hg, ho = vg.to_host(), vo.to_host()
    assert hg.size == ho.size and hg.num_seqs == ho.num_seqs
    for f in INT_FIELDS:
        np.testing.assert_array_equal(getattr(hg, f), getattr(ho, f), err_msg=f)
    if cont:
        assert_close(hg.act_cont, ho.act_cont, what="act_cont")
    else:
        np.testing.assert_array_equal(hg.act_disc, ho.act_disc, err_msg="act_disc")
    for f in ("obs", "reward", "latency"):
        np.testing.assert_array_equal(getattr(hg, f).astype(np.float64), getattr(ho, f).astype(np.float32)
                                      .astype(np.float64), err_msg=f)
    for f in ("log_prob", "value", "h0", "env_bootstrap"):
        assert_close(getattr(hg, f), getattr(ho, f), what=f)


@pytest.mark.parametrize("kind,mode,E,H,N,T", [
    (0, 1, 16, 16, 12, 8), (0, 0, 16, 16, 12, 8), (1, 1, 16, 16, 12, 8), (0, 1, 512, 512, 24, 6),
    (0, 1, 256, 256, 200, 3),  # batches of >= 150 requests: the GRU step on the tcgen05 step kernel
    (1, 0, 512, 512, 24, 4),   # Gaussian head, Fixed mode, H = 512
])
def test_engine_lockstep(kind, mode, E, H, N, T):
    import paper_2210_05064_b200 as V
    from oracle import engine as OE
    from oracle import oracle as O
    cfg = _cfg(kind, E, H)
    p = O.params_init(cfg, O.mix(11, 0x9A9A)).astype(np.float32)
    seed = O.mix(7, 0xF00D)
    g = V.InferenceEngine(cfg, T, N, p, version=3, mode=mode, seed=seed)
    o = OE.Engine(cfg, T, N, p.astype(np.float64), version=3, mode=mode, seed=seed)
    drv = Driver(N, cfg.obs_dim, seed=5)
    skipped = 0

    def check(rg, ro):
        nonlocal skipped
        assert [d[0] for d in rg.dispatches] == [d[0] for d in ro.dispatches]
        assert rg.new_commits == ro.new_commits and rg.closed_now == ro.closed_now
        for (e, ag), (_, ao) in zip(rg.dispatches, ro.dispatches):
            if kind:
                assert_close(ag, ao, what=f"action env {e}")
            elif ag != ao:
                assert ro.margins[e] < 1e-5, (e, ag, ao, ro.margins[e])
                skipped += 1

    for rollout in range(3):
        if rollout == 2:  # a new snapshot between rollouts
            p2 = (p * np.float32(0.9)).astype(np.float32)
            g.set_snapshot(p2, 4)
            o.set_snapshot(p2.astype(np.float64), 4)
        rg, ro = g.begin_rollout(), o.begin_rollout()
        check(rg, ro)
        drv.unpark([d[0] for d in ro.dispatches])
        ticks = 0
        while o._open() and ticks < 1000:
            reqs = drv.requests(V.InferenceRequest, p=0.95 if N >= 200 else 0.6)
            rg = g.process_batch(reqs)
            ro = o.process_batch([OE.Request(**q.__dict__) for q in reqs])
            check(rg, ro)
            assert g.rollout_done() == (not o._open())
            drv.after(reqs, [d[0] for d in ro.dispatches])
            ticks += 1
        assert g.committed() == o.buf.state()[1] and g.carryover_count() == o.buf.state()[2]
        g.finalize_bootstraps()
        o.finalize_bootstraps()
        _compare_views(g.close(), o.close(), kind == 1)
        assert_close(g.hidden(), np.stack([s.h for s in o.envs]), what="h")
    assert skipped == 0 or kind == 0


def test_engine_protocol_errors():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg(0, 16, 16)
    p = O.params_init(cfg, O.mix(1, 0x9A9A)).astype(np.float32)
    g = V.InferenceEngine(cfg, 4, 4, p, version=1, mode=V.VARIABLE, seed=1)
    g.begin_rollout()
    with pytest.raises(V.ProtocolError):
        g.process_batch([V.InferenceRequest(0, np.zeros(2, np.float32))])  # no outstanding action
    g.process_batch([V.InferenceRequest(1, np.zeros(2, np.float32), first=True)])
    g.force_close()
    r = g.process_batch([V.InferenceRequest(2, np.zeros(2, np.float32), first=True)])
    assert r.dispatches == [] and g.active_envs() == 3
    with pytest.raises(V.ProtocolError):
        g.process_batch([V.InferenceRequest(2, np.zeros(2, np.float32), first=True)])  # already parked
    # a parked request is not evaluated; an open engine's act rejects it (nn.cpp:119)
    g.process_batch([V.InferenceRequest(3, np.array([np.nan, 0.0], np.float32), first=True)])
    g2 = V.InferenceEngine(cfg, 4, 4, p, version=1, mode=V.VARIABLE, seed=1)
    g2.begin_rollout()
    with pytest.raises(V.ProtocolError):
        g2.process_batch([V.InferenceRequest(3, np.array([np.nan, 0.0], np.float32), first=True)])


def test_engine_snapshot_from_learner():
    """set_snapshot_from copies the learner's device parameters (no host round trip)."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg(0, 16, 16)
    p = O.params_init(cfg, O.mix(2, 0x9A9A)).astype(np.float32)
    lg = V.Learner(cfg, p)
    g1 = V.InferenceEngine(cfg, 4, 4, np.zeros_like(p), seed=9)
    g2 = V.InferenceEngine(cfg, 4, 4, p, seed=9)
    g1.set_snapshot_from(lg, 0)
    reqs = [V.InferenceRequest(e, np.array([0.1 * e, -0.2], np.float32), first=True) for e in range(4)]
    g1.begin_rollout()
    g2.begin_rollout()
    r1, r2 = g1.process_batch(reqs), g2.process_batch(reqs)
    assert r1.dispatches == r2.dispatches
    np.testing.assert_array_equal(g1.hidden(), g2.hidden())
