"""Port of the reference's tests/test_learner.cpp (GAE, PPO loss, entropy
controller, split-tail h0 replay, update determinism) — on the oracle (the
reference's own tolerances, double) and on the device (fp32 bounds stated in
each test)."""
import math

import numpy as np
import pytest

from backends import BACKENDS, GroupView, make_backend, protocol_errors
from helpers import make_view, random_lengths
from paper_2210_05064_b200.api import CosineSchedule, EntropyController, ModelConfig, PPOConfig
from paper_2210_05064_b200.rng import CounterRng


@pytest.fixture(params=BACKENDS)
def be(request):
    return make_backend(request.param)


def tol(be, ref_tol):
    """The reference's tolerance on the double oracle; fp32 bound on the device."""
    return ref_tol if be.name == "oracle" else max(ref_tol, 2e-5)


# ---------------------------------------------------------------- GAE
def gae_double_sum(hv, gamma, lam):  # test_learner.cpp:17-44
    adv = np.zeros(hv.size)
    ret = np.zeros(hv.size)
    for e in range(hv.N):
        slots = [i for i in range(hv.size) if hv.env_index[i] == e and not hv.stale[i]]
        n = len(slots)
        for t in range(n):
            acc, w = 0.0, 1.0
            for k in range(t, n):
                i = slots[k]
                nv = 0.0
                if not hv.done[i]:
                    nv = hv.value[slots[k + 1]] if k + 1 < n else hv.env_bootstrap[e]
                mask = 0.0 if hv.done[i] else 1.0
                delta = hv.reward[i] + gamma * nv * mask - hv.value[i]
                acc += w * delta
                if hv.done[i]:
                    break
                w *= gamma * lam
            adv[slots[t]] = acc
            ret[slots[t]] = acc + hv.value[slots[t]]
    return adv, ret


def test_gae_single_reward(be):  # test_learner.cpp:72-81
    hv = make_view([3])
    hv.reward[0] = 1.0
    hv.env_bootstrap_valid[0] = 0
    hv.done[2] = 1
    v = be.upload(hv)
    be.gae(v, 1.0, 1.0)
    a = be.host(v).advantage
    assert a[0] == pytest.approx(1.0) and a[1] == pytest.approx(0.0) and a[2] == pytest.approx(0.0)


def test_gae_zeros(be):  # test_learner.cpp:83-88
    v = be.upload(make_view([4]))
    be.gae(v, 0.99, 0.95)
    h = be.host(v)
    assert np.abs(h.advantage).max() == 0 and np.abs(h.returns).max() == 0


def test_gae_done_cuts(be):  # test_learner.cpp:90-97
    hv = make_view([2, 2])
    hv.reward[1] = 3.0
    hv.value[1] = 1.0
    v = be.upload(hv)
    be.gae(v, 0.99, 0.95)
    assert be.host(v).advantage[1] == pytest.approx(2.0)


def test_gae_missing_bootstrap_throws(be):  # test_learner.cpp:99-107
    hv = make_view([3])
    hv.done[2] = 0
    hv.env_bootstrap_valid[0] = 0
    with pytest.raises(protocol_errors()):
        be.gae(be.upload(hv), 0.99, 0.95)
    hv.env_bootstrap_valid[0] = 1
    hv.env_bootstrap[0] = 0.5
    be.gae(be.upload(hv), 0.99, 0.95)


def test_gae_vs_double_sum(be):  # test_learner.cpp:109-130 (100 trials)
    rng = CounterRng(8)
    for trial in range(100):
        lengths = random_lengths(8, 8, rng)
        hv = make_view(lengths, 2, 4, 8, 1)
        for i in range(hv.size):
            hv.reward[i] = rng.normal()
            hv.value[i] = rng.normal()
            hv.done[i] = 1 if rng.uniform() < 0.25 else 0
        hv.env_bootstrap[0] = rng.normal()
        hv.env_bootstrap_valid[0] = 1
        if be.name == "gpu":  # the device consumes fp32 inputs: compare on those
            hv = hv.astype(np.float32).astype(np.float64)
        v = be.upload(hv)
        be.gae(v, 0.99, 0.95)
        adv, ret = gae_double_sum(hv, 0.99, 0.95)
        h = be.host(v)
        t = 1e-10 if be.name == "oracle" else 1e-5
        assert np.abs(h.advantage - adv).max() < t * max(1.0, np.abs(adv).max())
        assert np.abs(h.returns - ret).max() < t * max(1.0, np.abs(ret).max())


def test_gae_interleaved_envs_general_path(be):
    """make_view with N > 1 interleaves envs (env = seq % N): the non-contiguous path."""
    rng = CounterRng(44)
    for trial in range(20):
        N = 1 + int(rng.uniform_int(5))
        lengths = random_lengths(40, 9, rng)
        hv = make_view(lengths, 2, 4, 40, N)
        for i in range(hv.size):
            hv.reward[i] = rng.normal()
            hv.value[i] = rng.normal()
            hv.done[i] = 1 if rng.uniform() < 0.2 else 0
        for e in range(N):
            hv.env_bootstrap[e] = rng.normal()
            hv.env_bootstrap_valid[e] = 1
        hv = hv.astype(np.float32).astype(np.float64)
        v = be.upload(hv)
        be.gae(v, 0.99, 0.95)
        adv, ret = gae_double_sum(hv, 0.99, 0.95)
        h = be.host(v)
        t = 1e-10 if be.name == "oracle" else 1e-5
        assert np.abs(h.advantage - adv).max() < t * max(1.0, np.abs(adv).max())


# ------------------------------------------------------------ PPO loss
def tiny_cfg(obs_dim=2, hidden=4, actions=2):  # test_learner.cpp:46-54
    return ModelConfig(obs_dim=obs_dim, encoder_dim=4, hidden_dim=hidden, action_kind=0,
                       num_actions=actions)


def params_for(be, cfg, seed):
    from oracle import oracle as O
    return O.params_init(cfg, seed)


def act_chain(be, cfg, p, obs_row, h):
    if be.name == "oracle":
        from oracle import oracle as O
        return O.act(cfg, p, obs_row, h)
    import paper_2210_05064_b200 as V
    d, val, hn = V.act(cfg, p, obs_row, h)
    return d.astype(np.float64), val.astype(np.float64), hn.astype(np.float64)


def logp_of(dist_row, a):
    m = dist_row.max()
    return dist_row[a] - (m + math.log(np.exp(dist_row - m).sum()))


def make_on_policy(be, hv, cfg, p):  # test_learner.cpp:57-68
    for d in hv.seqs:
        h = hv.h0[d[4]].reshape(1, -1)
        for t in range(d[2]):
            slot = d[3] + t
            dist, val, hn = act_chain(be, cfg, p, hv.obs[slot].reshape(1, -1), h)
            hv.log_prob[slot] = logp_of(dist[0], int(hv.act_disc[slot]))
            hv.value[slot] = val[0]
            h = hn


def loss(be, cfg, p, v, b, ppo, alpha, h0, want=False, frozen=None):
    if be.name == "oracle":
        from oracle import oracle as O
        return O.ppo_loss(cfg, p, v, b, ppo, alpha, h0, want, frozen)
    import paper_2210_05064_b200 as V
    r = V.ppo_loss(cfg, p, v, b, ppo, alpha, h0, want, frozen)
    return dict(loss=r.loss, policy_loss=r.policy_loss, value_loss=r.value_loss,
                mean_entropy=r.mean_entropy, ratio_sum=r.ratio_sum, clip_count=r.clip_count,
                w_sum=r.w_sum, w_max=r.w_max, steps=r.steps, grads=r.grads, is_weights=r.is_weights)


def test_loss_on_policy(be):  # test_learner.cpp:132-148
    cfg = tiny_cfg()
    p = params_for(be, cfg, 7)
    hv = make_view([3, 2, 3], 2, 4)
    make_on_policy(be, hv, cfg, p)
    v = be.upload(hv)
    be.gae(v, 0.99, 0.95)
    b = be.pack(v, GroupView(hv.seqs, hv.size))
    h0 = np.stack([hv.h0[s[4]] for s in b.seqs])
    r = loss(be, cfg, p, v, b, PPOConfig(), 1e-3, h0)
    assert r["ratio_sum"] / r["steps"] == pytest.approx(1.0, rel=tol(be, 1e-12))
    assert r["clip_count"] == 0
    assert r["w_sum"] / r["steps"] == pytest.approx(1.0, rel=tol(be, 1e-12))


def test_loss_is_cap(be):  # test_learner.cpp:150-167
    cfg = tiny_cfg()
    p = params_for(be, cfg, 9)
    hv = make_view([2], 2, 4)
    make_on_policy(be, hv, cfg, p)
    hv.log_prob[0] -= math.log(1.5)
    hv.log_prob[1] -= math.log(0.5)
    v = be.upload(hv)
    be.gae(v, 0.99, 0.95)
    b = be.pack(v, GroupView(hv.seqs, hv.size))
    r = loss(be, cfg, p, v, b, PPOConfig(), 0.0, hv.h0)
    assert r["w_max"] == pytest.approx(1.0, rel=tol(be, 1e-12))
    assert r["w_sum"] == pytest.approx(1.5, rel=tol(be, 1e-9))


def test_loss_clip_branch(be):  # test_learner.cpp:169-186
    cfg = tiny_cfg()
    p = params_for(be, cfg, 11)
    hv = make_view([1], 2, 4)
    make_on_policy(be, hv, cfg, p)
    hv.log_prob[0] -= math.log(1.3)
    hv.advantage[0] = 1.0
    hv.returns[0] = hv.value[0]
    v = be.upload(hv)
    b = be.pack(v, GroupView(hv.seqs, hv.size))
    r = loss(be, cfg, p, v, b, PPOConfig(value_loss_coef=0.0), 0.0, hv.h0)
    assert r["policy_loss"] == pytest.approx(-1.2, rel=tol(be, 1e-9))
    assert r["clip_count"] == 1


def fd_setup():
    cfg = tiny_cfg(2, 4, 3)
    from oracle import oracle as O
    p = O.params_init(cfg, 13)
    rng = CounterRng(21)
    hv = make_view([3, 2, 2, 1], 2, 4)
    for i in range(hv.size):
        hv.obs[i, 0] = rng.normal()
        hv.obs[i, 1] = rng.normal()
        hv.act_disc[i] = int(rng.uniform_int(3))
        hv.log_prob[i] = -1.0 + 0.3 * rng.normal()
        hv.advantage[i] = rng.normal()
        hv.returns[i] = rng.normal()
    return cfg, p, hv


def test_loss_gradient_fd_oracle():  # test_learner.cpp:188-236 on the oracle
    from oracle import oracle as O
    cfg, p, hv = fd_setup()
    v = O.View.from_host(hv)
    b = O.pack(hv.seqs)
    h0 = np.stack([hv.h0[s[4]] for s in b.seqs])
    alpha = 0.01
    res = O.ppo_loss(cfg, p, v, b, PPOConfig(), alpha, h0, True)
    fw = res["is_weights"]
    names = _tensor_slices(cfg)
    checked = 0
    for ti, (name, r_, c_, off) in enumerate(names):
        for r in range(r_):
            for c in range(c_):
                if (r + c + ti) % 3:
                    continue
                k = off + r * c_ + c
                h = 1e-5
                pp = p.copy()
                pp[k] = p[k] + h
                up = O.ppo_loss(cfg, pp, v, b, PPOConfig(), alpha, h0, False, fw)["loss"]
                pp[k] = p[k] - h
                dn = O.ppo_loss(cfg, pp, v, b, PPOConfig(), alpha, h0, False, fw)["loss"]
                fd = (up - dn) / (2 * h)
                an = res["grads"][k]
                assert abs(fd - an) / max(1.0, abs(fd), abs(an)) < 1e-3
                checked += 1
    assert checked > 50


def _tensor_slices(cfg):
    import paper_2210_05064_b200 as V
    return V.param_tensors(cfg)


@pytest.mark.gpu
def test_loss_gradient_device_vs_oracle():
    """Device ppo_loss gradients vs the FD-pinned oracle: |a-b| <= 1e-5 max(1,|b|)
    (the reference's denominator convention, test_learner.cpp:229) and normwise."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg, p, hv = fd_setup()
    hv = hv.astype(np.float32).astype(np.float64)
    p32 = p.astype(np.float32).astype(np.float64)
    vo, vg = O.View.from_host(hv), V.RolloutView.from_host(hv)
    bo = O.pack(hv.seqs)
    bg = V.pack(vg, V.SequenceGroup(hv.seqs))
    h0 = np.stack([hv.h0[s[4]] for s in bo.seqs])
    ro = O.ppo_loss(cfg, p32, vo, bo, PPOConfig(), 0.01, h0, True)
    rg = V.ppo_loss(cfg, p32, vg, bg, PPOConfig(), 0.01, h0, True)
    assert rg.loss == pytest.approx(ro["loss"], rel=1e-5, abs=1e-6)
    g, go = rg.grads.astype(np.float64), ro["grads"]
    assert np.all(np.abs(g - go) <= 1e-5 * np.maximum(1.0, np.abs(go)))
    assert np.linalg.norm(g - go) <= 1e-5 * max(1e-12, np.linalg.norm(go)) + 1e-7


# ------------------------------------------------------ entropy control
def test_entropy_controller():  # test_learner.cpp:238-273
    c = EntropyController(alpha=0.01, target=0.5, lr=0.1)
    c.update(0.5)
    assert c.alpha == pytest.approx(0.01)
    c = EntropyController(alpha=0.01, target=0.5, lr=0.1)
    c.update(0.2)
    assert c.alpha > 0.01
    c = EntropyController(alpha=0.01, target=0.5, lr=0.1)
    for _ in range(100):
        c.update(5.0)
    assert c.alpha == pytest.approx(1e-4)
    c = EntropyController(alpha=0.01, target=0.5, lr=0.1)
    for _ in range(10000):
        c.update(-5.0)
    assert c.alpha == pytest.approx(1.0)
    from paper_2210_05064_b200.api import entropy_loss_value
    c = EntropyController(alpha=0.3, target=0.1)
    assert entropy_loss_value(0.7, c) == pytest.approx(0.3 * (0.1 - 0.7) - 0.3 * 0.7)
    c2 = EntropyController(alpha=0.3, target=0.1, lr=1.0)
    c2.update(0.7)
    assert c2.alpha == pytest.approx(max(1e-4, 0.3 + (0.1 - 0.7)))


# ------------------------------------------------------ learner (oracle)
def make_learner(be, cfg, p, ppo=PPOConfig(), ec=EntropyController(), sched=CosineSchedule(1e-4, 1000),
                 seed=5):
    if be.name == "oracle":
        from oracle import oracle as O
        L = O.Learner(cfg, p, ppo, ec, sched.base_lr, sched.total_steps, seed)
        return L
    import paper_2210_05064_b200 as V
    return V.Learner(cfg, p, ppo, ec, sched, seed)


def test_split_tail_h0_replay(be):  # test_learner.cpp:275-293
    cfg = tiny_cfg()
    from oracle import oracle as O
    p = O.params_init(cfg, 17)
    hv = make_view([6], 2, 4)
    rng = CounterRng(3)
    for i in range(hv.size):
        hv.obs[i, 0] = rng.normal()
    if be.name == "gpu":
        hv = hv.astype(np.float32).astype(np.float64)
        p = p.astype(np.float32).astype(np.float64)
    learner = make_learner(be, cfg, p)
    v = be.upload(hv)
    groups = be.split_in_order(v, 2, [0])
    assert groups[1].col("skip")[0] == 3
    tail = be.pack(v, groups[1])
    if be.name == "oracle":
        h0 = learner.batch_h0(v, tail)
    else:
        h0 = learner.batch_h0(v, tail).astype(np.float64)
    h = hv.h0[0].reshape(1, -1)
    for t in range(3):
        h = O.act(cfg, p, hv.obs[t].reshape(1, -1), h)[2]
    assert np.abs(h0[0] - h[0]).max() < tol(be, 1e-14)


def stats_of(be, s):
    return s if isinstance(s, dict) else s.__dict__


def test_zero_lr_determinism(be):  # test_learner.cpp:295-320
    cfg = tiny_cfg()
    from oracle import oracle as O
    p = O.params_init(cfg, 19)
    hv = make_view([4, 4, 4, 4], 2, 4, 4, 4)
    make_on_policy(make_backend("oracle"), hv, cfg, p)
    for i in range(hv.size):
        hv.reward[i] = 1.0 if i % 3 == 0 else 0.0
    for e in range(4):
        hv.env_bootstrap_valid[e] = 1
    ec = EntropyController(lr=0.0)
    L = make_learner(be, cfg, p, ec=ec, sched=CosineSchedule(0.0, 1000))
    if be.name == "oracle":
        L.set_state(ec.alpha, 0, 0)
        a = L.update(be.upload(hv))
        L.set_state(ec.alpha, 0, 0)
        b = L.update(be.upload(hv))
    else:
        L.set_state(update_index=0)
        a = stats_of(be, L.update(be.upload(hv)))
        L.set_state(update_index=0, consumed=0)
        b = stats_of(be, L.update(be.upload(hv)))
    for k in ("loss", "mean_ratio", "clip_fraction", "entropy", "value_loss"):
        assert a[k] == pytest.approx(b[k])
    assert 0.0 <= a["clip_fraction"] <= 1.0


def test_value_loss_decreases(be):  # test_learner.cpp:338-354
    cfg = tiny_cfg()
    from oracle import oracle as O
    p = O.params_init(cfg, 23)
    L = make_learner(be, cfg, p, sched=CosineSchedule(1e-2, 1000000))
    first = last = None
    for u in range(30):
        hv = make_view([4, 4, 4, 4], 2, 4, 4, 4)
        cur = L.params() if be.name == "oracle" else L.params().astype(np.float64)
        make_on_policy(make_backend("oracle"), hv, cfg, cur)
        hv.reward[:] = 1.0
        st = stats_of(be, L.update(be.upload(hv)))
        if u == 0:
            first = st["value_loss"]
        last = st["value_loss"]
    assert last < first
