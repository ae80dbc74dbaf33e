"""Device vs oracle parity on the synthetic heterogeneous-environment inputs
(SURVEY.md §8d), through the C-ABI.

Bars:
  * indices / offsets / compaction / minibatch pieces: bit-exact;
  * copied payload fields: bit-exact (fp32 in, fp32 out);
  * advantages, returns, losses, gradients: |a - b| <= 1e-5 * max(1, |b|)
    (the reference's own denominator convention, test_learner.cpp:229);
  * parameters after full updates: |a - b| <= 1e-5 * max(1, |b|) as well.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def close_both(T, N, H, seed=1, D=2, A=2, preempt_at=None):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    wl = synth.make_workload(T, N, obs_dim=D, num_actions=A, hidden_dim=H, seed=seed)
    recs = wl.records
    if preempt_at is not None:
        from dataclasses import replace
        recs = V.StepRecords(**{k: (None if v is None else np.asarray(v)[:preempt_at])
                                for k, v in recs.__dict__.items()})
        wl = replace(wl, records=recs)
    g = V.RolloutBuffer(T, N, V.VARIABLE, 0, D, 0, H)
    o = O.Rollout(T, N, 1, 0, D, 0, H)
    for buf in (g, o):
        synth.fill_buffer(buf, wl)
        if preempt_at is not None:
            buf.force_close()
    return g.close_rollout(), o.close_rollout(), wl


def assert_close(a, b, tol=1e-5, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max(initial=0.0) <= tol, f"{what}: max scaled err {err.max():.3e}"


INT_FIELDS = ("act_disc", "done", "stale", "replayed", "env_index", "seq_of_slot", "step_in_episode",
              "episode_index", "version", "seqs", "per_env_counts", "env_bootstrap_valid")
F_FIELDS = ("obs", "log_prob", "value", "reward", "latency", "h0", "env_bootstrap")


@pytest.mark.parametrize("T,N,H", [(16, 16, 8), (128, 16, 64), (32, 256, 16), (8, 1000, 4)])
def test_close_rollout_bitexact(T, N, H):
    vg, vo, _ = close_both(T, N, H)
    hg, ho = vg.to_host(), vo.to_host()
    assert hg.size == ho.size and hg.num_seqs == ho.num_seqs and hg.deficit == ho.deficit
    for f in INT_FIELDS:
        np.testing.assert_array_equal(getattr(hg, f), getattr(ho, f), err_msg=f)
    for f in F_FIELDS:
        np.testing.assert_array_equal(getattr(hg, f).astype(np.float64), getattr(ho, f), err_msg=f)


def test_preempted_close_and_backfill_bitexact():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    T, N, H = 32, 64, 8
    pg, po, _ = close_both(T, N, H, seed=2)
    vg, vo, _ = close_both(T, N, H, seed=3, preempt_at=T * N - 517)
    assert vg.deficit == 517
    V.compute_gae(pg, 0.99, 0.95)
    O.compute_gae(po, 0.99, 0.95)
    # give prev stale sequences too: backfill twice through a chain
    V.backfill_stale(vg, pg, vg.deficit)
    O.backfill_stale(vo, po, 517)
    hg, ho = vg.to_host(), vo.to_host()
    assert hg.size == ho.size == T * N and hg.stale_steps == ho.stale_steps == 517
    for f in INT_FIELDS:
        np.testing.assert_array_equal(getattr(hg, f), getattr(ho, f), err_msg=f)
    for f in F_FIELDS:
        np.testing.assert_array_equal(getattr(hg, f).astype(np.float64), getattr(ho, f), err_msg=f)
    # advantages/returns copied verbatim from prev (device A/R vs oracle A/R: GAE tolerance)
    assert_close(hg.advantage[-517:], ho.advantage[-517:], what="backfilled A")


@pytest.mark.parametrize("T,N", [(128, 16), (128, 256), (64, 1024)])
def test_gae_parity(T, N):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    vg, vo, _ = close_both(T, N, 4, seed=T + N)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hg, ho = vg.to_host(), vo.to_host()
    assert_close(hg.advantage, ho.advantage, what="A")
    assert_close(hg.returns, ho.returns, what="R")


def test_gae_after_backfill_skips_replayed():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    pg, po, _ = close_both(16, 32, 4, seed=9)
    V.compute_gae(pg, 0.99, 0.95)
    O.compute_gae(po, 0.99, 0.95)
    vg, vo, _ = close_both(16, 32, 4, seed=10, preempt_at=400)
    V.backfill_stale(vg, pg, vg.deficit)
    O.backfill_stale(vo, po, 512 - 400)
    V.compute_gae(vg, 0.9, 0.8)
    O.compute_gae(vo, 0.9, 0.8)
    assert_close(vg.to_host().advantage, vo.to_host().advantage, what="A")


def test_gather_bitexact():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    vg, vo, _ = close_both(64, 128, 4, seed=4)
    V.compute_gae(vg, 0.99, 0.95)
    hv = vg.to_host()
    for g in V.split_minibatches(vg, 2, 1234):
        b = V.pack(vg, g)
        ga = b.gathered(2)
        s = b.slots
        np.testing.assert_array_equal(ga["obs"], hv.obs[s])
        np.testing.assert_array_equal(ga["act_disc"], hv.act_disc[s])
        np.testing.assert_array_equal(ga["old_logp"], hv.log_prob[s])
        np.testing.assert_array_equal(ga["adv"], hv.advantage[s])
        np.testing.assert_array_equal(ga["ret"], hv.returns[s])


def _model(E, H, D=2, A=2):
    import paper_2210_05064_b200 as V
    return V.ModelConfig(obs_dim=D, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=A)


@pytest.mark.parametrize("E,H,T,N", [(64, 64, 32, 16), (32, 48, 16, 64)])
def test_ppo_loss_parity_synthetic(E, H, T, N):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _model(E, H)
    p = O.params_init(cfg, O.mix(1, 0x9A9A)).astype(np.float32).astype(np.float64)
    vg, vo, _ = close_both(T, N, H, seed=5)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    # use the oracle's A/R on both sides so the loss inputs are identical fp32 values
    hv = vo.to_host().astype(np.float32).astype(np.float64)
    vo2, vg2 = O.View.from_host(hv), V.RolloutView.from_host(hv)
    for gi, (seqs, tot) in enumerate(O.split_minibatches(vo2, 2, 77).groups()):
        bo = O.pack(seqs)
        bg = V.pack(vg2, V.SequenceGroup(seqs, tot))
        np.testing.assert_array_equal(bo.slots, bg.slots)
        h0 = np.stack([hv.h0[s[4]] for s in bo.seqs])
        ro = O.ppo_loss(cfg, p, vo2, bo, V.PPOConfig(), 1e-3, h0, True)
        rg = V.ppo_loss(cfg, p, vg2, bg, V.PPOConfig(), 1e-3, h0, True)
        for k in ("loss", "policy_loss", "value_loss", "mean_entropy"):
            assert abs(getattr(rg, k) - ro[k]) <= 1e-5 * max(1.0, abs(ro[k])), k
        assert rg.clip_count == ro["clip_count"]
        assert_close(rg.grads, ro["grads"], what="grads")
        assert_close(rg.is_weights, ro["is_weights"], what="w")


def _learner_pair(E, H, epochs, B, seed=1):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _model(E, H)
    p = O.params_init(cfg, O.mix(seed, 0x9A9A)).astype(np.float32).astype(np.float64)
    ppo = V.PPOConfig(epochs=epochs, minibatches=B)
    ec = V.EntropyController()
    sched = V.CosineSchedule(2.5e-4, 2_000_000)
    run_seed = O.mix(seed, 0xF00D)
    lg = V.Learner(cfg, p, ppo, ec, sched, run_seed)
    lo = O.Learner(cfg, p, ppo, ec, sched.base_lr, sched.total_steps, run_seed)
    return cfg, lg, lo


@pytest.mark.parametrize("E,H,T,N,epochs,B", [(64, 64, 128, 16, 1, 2), (32, 32, 32, 32, 2, 2),
                                             (16, 24, 16, 48, 3, 3)])
def test_learner_update_parity(E, H, T, N, epochs, B):
    """Full Learner::update (C1 = reference CPU default first): stats and params."""
    cfg, lg, lo = _learner_pair(E, H, epochs, B)
    for it in range(2):
        vg, vo, _ = close_both(T, N, H, seed=11 + it)
        sg = lg.update(vg)
        so = lo.update(vo)
        for k in ("loss", "policy_loss", "value_loss", "entropy", "mean_ratio", "mean_is_weight",
                  "max_is_weight", "alpha", "lr", "entropy_loss"):
            assert abs(getattr(sg, k) - so[k]) <= 1e-5 * max(1.0, abs(so[k])), (it, k)
        assert abs(sg.clip_fraction - so["clip_fraction"]) <= 2.0 / (T * N * epochs)
        assert sg.steps == so["steps"] and sg.fresh_steps == so["fresh_steps"]
        assert_close(lg.params(), lo.params(), what=f"params after update {it}")
    m, v, step = lg.adam()
    mo, vo_, so_ = lo.adam()
    assert step == so_
    assert_close(m, mo, what="adam m")


def test_batch_h0_split_tails_synthetic():
    """Split tails replay their heads with the current params (learner.cpp:119-130)."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg, lg, lo = _learner_pair(16, 16, 1, 3)
    vg, vo, _ = close_both(24, 20, 16, seed=6)
    for b in range(3):
        go = O.split_minibatches(vo, 3, 99).group(b)
        bo = O.pack(go[0])
        bg = V.pack(vg, V.SequenceGroup(go[0], go[1]))
        assert_close(lg.batch_h0(vg, bg), lo.batch_h0(vo, bo), what="h0")


def test_full_scale_properties_c2():
    """C2 shape (N=256, T=128, E=H=512, 4 epochs x 2): conservation and sanity
    at full size (no oracle at this size; the oracle pins smaller shapes)."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    T, N, H = 128, 256, 512
    wl = synth.make_workload(T, N, hidden_dim=H, seed=1)
    buf = V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H)
    synth.fill_buffer(buf, wl)
    view = buf.close_rollout()
    hv = view.to_host()
    assert hv.size == T * N and list(hv.per_env_counts) == list(wl.counts)
    assert int(hv.seqs[:, 2].sum()) == T * N
    cfg = _model(512, 512)
    p = V.params_init(cfg, O.mix(1, 0x9A9A))
    L = V.Learner(cfg, p, V.PPOConfig(epochs=4, minibatches=2), V.EntropyController(),
                  V.CosineSchedule(2.5e-4, 2_000_000), O.mix(1, 0xF00D))
    st = L.update(view)
    assert np.isfinite(st.loss) and 0.0 <= st.clip_fraction <= 1.0
    assert st.fresh_steps == T * N
    q = L.params()
    assert np.all(np.isfinite(q)) and np.abs(q - p).max() > 0
