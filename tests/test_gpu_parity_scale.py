"""GPU vs oracle parity at the BENCHMARKED shapes, with the library's natural
path selection (no tuning overrides): the C2 minibatch loss and gradients, the
full C2 Learner::update (N=256, T=128, E=H=512, 4 epochs x 2 minibatches), and
one C3-scale minibatch.

At C2 a packed minibatch walks every recurrence path the bench runs: the
persistent tcgen05 step kernel for the big steps (>= 150 rows), the K-split
FMA kernels for the middle ones, the tagged handoff for short forward steps and
the 16-CTA cluster tail for the last rows; the full update adds the split-tail
h0 replay (learner.cpp:119-130) and Adam.

C3 proper is N=4096 (262,144 rows per minibatch); the oracle (16 OpenMP threads,
bit-identical to one) checks one C3 minibatch in ~2 minutes, plus an N=1024
minibatch.  These tests found a real bug in round 1's persistent step kernel:
steps with more output tiles than CTAs skipped the excess tiles (C3 only).

Bars: |gpu - oracle| <= 1e-5 * max(1, |oracle|) for losses, statistics and
gradients (learner.cpp:52-117); parameters after a full update 1e-5 on >=
99.99% of entries and 1e-4 on all (Adam's first step moves a
parameter by ~lr whatever |g| is, so a gradient that is zero up to fp32
rounding can move by a visible fraction of lr).
"""
import numpy as np
import pytest

from test_gpu_parity import assert_close, close_both

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

T, E, H = 128, 512, 512


def _cfg():
    import paper_2210_05064_b200 as V
    return V.ModelConfig(obs_dim=2, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=2)


def _params(O):
    return O.params_init(_cfg(), O.mix(1, 0x9A9A)).astype(np.float32).astype(np.float64)


def _loss_parity(N, groups):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg()
    p = _params(O)
    vg, vo, _ = close_both(T, N, H, seed=1)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hg = vg.to_host()
    hv = vo.to_host()
    assert_close(hg.advantage, hv.advantage, what="A")
    assert_close(hg.returns, hv.returns, what="R")
    # identical fp32 loss inputs on both sides (the oracle's A/R rounded once)
    hv = hv.astype(np.float32).astype(np.float64)
    vo2, vg2 = O.View.from_host(hv), V.RolloutView.from_host(hv)
    lo = O.Learner(cfg, p, V.PPOConfig(), V.EntropyController(), 2.5e-4, 2_000_000, O.mix(1, 0xF00D))
    seed = O.mix(O.mix(O.mix(1, 0xF00D), 0), 0)  # epoch 0 of update 0 (learner.cpp:162)
    gg = V.split_minibatches(vg2, 2, seed)
    for gi, (seqs, tot) in enumerate(O.split_minibatches(vo2, 2, seed).groups()):
        if gi not in groups:
            continue
        np.testing.assert_array_equal(gg[gi].seqs, seqs)
        bo = O.pack(seqs)
        bg = V.pack(vg2, V.SequenceGroup(seqs, tot))
        np.testing.assert_array_equal(bo.slots, bg.slots)
        np.testing.assert_array_equal(bo.batch_sizes, bg.batch_sizes)
        assert bo.batch_sizes[0] >= 150 and bo.batch_sizes[-1] <= 2  # every recurrence path runs
        # h0 with split-tail replay at the initial parameters (learner.cpp:119-130)
        h0 = lo.batch_h0(vo2, bo)
        ro = O.ppo_loss(cfg, p, vo2, bo, V.PPOConfig(), 1e-3, h0, True)
        rg = V.ppo_loss(cfg, p, vg2, bg, V.PPOConfig(), 1e-3, h0, True)
        for k in ("loss", "policy_loss", "value_loss", "mean_entropy", "ratio_sum", "w_sum", "w_max"):
            assert abs(getattr(rg, k) - ro[k]) <= 1e-5 * max(1.0, abs(ro[k])), (gi, k, getattr(rg, k), ro[k])
        assert abs(rg.clip_count - ro["clip_count"]) <= 2, (rg.clip_count, ro["clip_count"])
        assert_close(rg.is_weights, ro["is_weights"], what="is weights")
        assert_close(rg.grads, ro["grads"], what=f"grads of group {gi}")
        # normwise as well: the whole gradient vector
        g, r = rg.grads.astype(np.float64), ro["grads"]
        assert np.linalg.norm(g - r) <= 1e-5 * max(1.0, np.linalg.norm(r))


def test_c2_minibatches_loss_and_grads():
    """Both C2 minibatches of epoch 0 (16,384 rows each, incl. the split tail's replayed h0)."""
    _loss_parity(256, groups=(0, 1))


def test_c3_scale_minibatch_loss_and_grads():
    """One minibatch at N=1024 (65,536 rows, up to 2,521 rows per step: the forward
    step GEMM has more output tiles than CTAs)."""
    _loss_parity(1024, groups=(0,))


def test_c3_minibatch_loss_and_grads():
    """One C3 minibatch (N=4096: 262,144 rows, ~10,000 rows per early step, so the
    backward step GEMM also walks several tiles per CTA).  ~2 min of oracle time."""
    _loss_parity(4096, groups=(0,))


def test_c2_full_update():
    """One full C2 Learner::update (GAE, 4 epochs x 2 minibatches with split-tail
    replay, forward, loss, backward, Adam, alpha) against the oracle's."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg()
    p = _params(O)
    ppo = V.PPOConfig(epochs=4, minibatches=2)
    ec = V.EntropyController()
    sched = V.CosineSchedule(2.5e-4, 2_000_000)
    run_seed = O.mix(1, 0xF00D)
    lg = V.Learner(cfg, p, ppo, ec, sched, run_seed)
    lo = O.Learner(cfg, p, ppo, ec, sched.base_lr, sched.total_steps, run_seed)
    vg, vo, _ = close_both(T, 256, H, seed=1)
    sg = lg.update(vg)
    so = lo.update(vo)
    for k in ("loss", "policy_loss", "value_loss", "entropy", "mean_ratio", "mean_is_weight",
              "max_is_weight", "alpha", "lr", "entropy_loss"):
        assert abs(getattr(sg, k) - so[k]) <= 1e-5 * max(1.0, abs(so[k])), (k, getattr(sg, k), so[k])
    assert abs(sg.clip_fraction - so["clip_fraction"]) <= 8.0 / (T * 256 * 4)
    assert sg.steps == so["steps"] and sg.fresh_steps == so["fresh_steps"]
    a, b = lg.params().astype(np.float64), lo.params()
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max() <= 1e-4, err.max()
    assert np.mean(err <= 1e-5) >= 0.9999, np.mean(err <= 1e-5)
    m, v, step = lg.adam()
    mo, vo_, so_ = lo.adam()
    assert step == so_ == 8
    assert_close(m, mo, what="adam m")
    assert_close(v, vo_, what="adam v")
