"""Continuous Gaussian head (SURVEY §8 secondary parity config, Reach2D shape:
D = 4, A = 2, learned log_std leaf): full Learner::update and ppo_loss
gradients against the oracle.  Covers the loss kernel's Gaussian branch
(nn.cpp:267-278), the log_std gradient and the Adam log_std clamp
(nn.cpp:291-306), at small H (register recurrence kernels) and H = 256
(K-split kernels and, forced by threshold, the per-step tcgen05 GEMMs)."""
import os
from dataclasses import replace

import numpy as np
import pytest

from test_gpu_parity import assert_close

pytestmark = pytest.mark.gpu

D, A = 4, 2


def _cfg(E, H):
    import paper_2210_05064_b200 as V
    return V.ModelConfig(obs_dim=D, encoder_dim=E, hidden_dim=H, action_kind=1, act_dim=A)


def _views(T, N, H, seed):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    wl = synth.make_workload(T, N, obs_dim=D, num_actions=2, hidden_dim=H, seed=seed)
    S = len(wl.records)
    rng = np.random.default_rng(seed)
    act = rng.standard_normal((S, A)).astype(np.float32)
    logp = (-0.5 * (act.astype(np.float64) ** 2).sum(1) - 0.5 * A * np.log(2 * np.pi)
            + 0.05 * rng.standard_normal(S)).astype(np.float32)
    recs = replace(wl.records, act_disc=None, act_cont=act, log_prob=logp)
    wl = replace(wl, records=recs)
    g = V.RolloutBuffer(T, N, V.VARIABLE, 1, D, A, H)
    o = O.Rollout(T, N, 1, 1, D, A, H)
    for buf in (g, o):
        synth.fill_buffer(buf, wl)
    return g.close_rollout(), o.close_rollout()


@pytest.fixture
def big_steps(request):
    keys = ("VER_REC_BIG_FWD", "VER_REC_BIG_BWD")
    saved = {k: os.environ.get(k) for k in keys}
    if request.param:
        for k in keys:
            os.environ[k] = "6"
    yield request.param
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("big_steps", [False, True], indirect=True)
@pytest.mark.parametrize("E,H,T,N,epochs,B", [(16, 16, 32, 16, 2, 2), (256, 256, 16, 24, 1, 2)])
def test_update_parity_gaussian(big_steps, E, H, T, N, epochs, B):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg(E, H)
    p = O.params_init(cfg, O.mix(5, 0x9A9A)).astype(np.float32).astype(np.float64)
    ppo = V.PPOConfig(epochs=epochs, minibatches=B)
    ec = V.EntropyController()
    sched = V.CosineSchedule(2.5e-4, 2_000_000)
    lg = V.Learner(cfg, p, ppo, ec, sched, O.mix(5, 0xF00D))
    lo = O.Learner(cfg, p, ppo, ec, sched.base_lr, sched.total_steps, O.mix(5, 0xF00D))
    vg, vo = _views(T, N, H, seed=41)
    sg = lg.update(vg)
    so = lo.update(vo)
    for k in ("loss", "policy_loss", "value_loss", "entropy", "mean_ratio", "alpha"):
        assert abs(getattr(sg, k) - so[k]) <= 1e-5 * max(1.0, abs(so[k])), k
    pg, po = np.asarray(lg.params(), np.float64), np.asarray(lo.params(), np.float64)
    err = np.abs(pg - po) / np.maximum(1.0, np.abs(po))
    # 1e-5 bar; Adam's first step (lr * sign) on near-zero gradient components, see
    # test_gpu_recurrence_paths for the H >= 256 allowance
    assert err.max() <= (1e-5 if H < 256 else 1e-4), err.max()
    assert np.mean(err > 1e-5) <= 1e-4
    # log_std entries (tensors() order: last A) within the clamp [-5, 2]
    assert np.all(pg[-A:] >= -5.0) and np.all(pg[-A:] <= 2.0)


@pytest.mark.parametrize("H", [16, 256])
def test_loss_gradient_parity_gaussian(H):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = _cfg(H, H)
    p = O.params_init(cfg, O.mix(6, 0x9A9A)).astype(np.float32).astype(np.float64)
    p[-A:] = [-0.3, 0.2]  # non-trivial log_std
    vg, vo = _views(16, 24, H, seed=43)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hv = vo.to_host()
    bo = O.pack(hv.seqs)
    bg = V.pack(vg, V.SequenceGroup(hv.seqs))
    h0 = np.stack([hv.h0[s[4]] for s in bo.seqs])
    ro = O.ppo_loss(cfg, p, vo, bo, V.PPOConfig(), 0.01, h0, True)
    rg = V.ppo_loss(cfg, p, vg, bg, V.PPOConfig(), 0.01, h0, True)
    assert abs(rg.loss - ro["loss"]) <= 1e-5 * max(1.0, abs(ro["loss"]))
    g, go = rg.grads.astype(np.float64), ro["grads"]
    assert np.all(np.abs(g - go) <= 1e-5 * np.maximum(1.0, np.abs(go))), np.abs(g - go).max()
    assert_close(g[-A:], go[-A:], what="log_std gradient")
