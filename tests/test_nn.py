"""Port of the reference's tests/test_nn.cpp (init, act vs packed forward,
value-MSE gradient, Adam, cosine) on the oracle and the device."""
import math

import numpy as np
import pytest

from backends import BACKENDS
from paper_2210_05064_b200.api import ModelConfig, param_tensors
from paper_2210_05064_b200.rng import CounterRng


def discrete_cfg(obs=3, hidden=8, actions=4):  # test_nn.cpp:13-21
    return ModelConfig(obs_dim=obs, encoder_dim=8, hidden_dim=hidden, action_kind=0, num_actions=actions)


def gaussian_cfg(obs=3, hidden=8, dim=2):  # test_nn.cpp:23-31
    return ModelConfig(obs_dim=obs, encoder_dim=8, hidden_dim=hidden, action_kind=1, act_dim=dim)


def random_obs(rows, cols, rng):
    return np.array([[rng.normal() for _ in range(cols)] for _ in range(rows)])


def tensor(cfg, p, name):
    for n, r, c, off in param_tensors(cfg):
        if n == name:
            return p[off:off + r * c].reshape(r, c)
    raise KeyError(name)


@pytest.fixture(params=BACKENDS)
def be(request):
    return request.param


def act(be, cfg, p, obs, h):
    if be == "oracle":
        from oracle import oracle as O
        return O.act(cfg, p, obs, h)
    import paper_2210_05064_b200 as V
    return tuple(x.astype(np.float64) for x in V.act(cfg, p, obs, h))


def fwd(be, cfg, p, obs, ad, ac, bs, offs, h0):
    if be == "oracle":
        from oracle import oracle as O
        return O.forward_packed(cfg, p, obs, ad, ac, bs, offs, h0)
    import paper_2210_05064_b200 as V
    return tuple(x.astype(np.float64) for x in V.forward_packed(cfg, p, obs, ad, ac, bs, offs, h0))


def test_zero_weights(be):  # test_nn.cpp:42-50
    from oracle import oracle as O
    cfg = gaussian_cfg()
    p = np.zeros(O.param_count(cfg))
    obs = random_obs(5, 3, CounterRng(2))
    d, v, _ = act(be, cfg, p, obs, np.zeros((5, 8)))
    assert np.abs(d).max() == 0 and np.abs(v).max() == 0


def test_orthonormal_init():  # test_nn.cpp:52-59, product init vs oracle init
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = discrete_cfg(6, 8, 3)
    for p in (V.params_init(cfg, 3), O.params_init(cfg, 3)):
        ur = tensor(cfg, p, "gru_ur")
        assert np.abs(ur.T @ ur - np.eye(8)).max() < 1e-9
        e = tensor(cfg, p, "enc_w2")
        assert np.abs(e.T @ e - 2 * np.eye(8)).max() < 1e-9
    for cfg in (discrete_cfg(), gaussian_cfg(), ModelConfig(2, 64, 64, 0, 2, 0)):
        assert np.abs(V.params_init(cfg, 11) - O.params_init(cfg, 11)).max() < 1e-12


def test_length1_packed_equals_act(be):  # test_nn.cpp:61-86
    from oracle import oracle as O
    for cfg in (discrete_cfg(), gaussian_cfg()):
        p = O.params_init(cfg, 11)
        rng = CounterRng(5)
        obs = random_obs(1, cfg.obs_dim, rng)
        h0 = random_obs(1, cfg.hidden_dim, rng)
        d, v, _ = act(be, cfg, p, obs, h0)
        ac = np.full((1, max(1, cfg.act_dim)), 0.3)
        lp, en, va = fwd(be, cfg, p, obs, np.array([1]) if cfg.action_kind == 0 else None,
                         ac if cfg.action_kind else None, [1], [0], h0)
        t = 1e-12 if be == "oracle" else 1e-5
        assert va[0] == pytest.approx(v[0], rel=t, abs=t)
        if cfg.action_kind == 0:
            ref = O.categorical_log_prob(d[0], 1)
        else:
            ls = tensor(cfg, p, "log_std")[0]
            z = (0.3 - d[0]) / np.exp(ls)
            ref = -0.5 * np.sum(z * z) - ls.sum() - 0.5 * 1.8378770664093453 * cfg.act_dim
        assert lp[0] == pytest.approx(ref, rel=t, abs=t)


def test_packed_equals_chained(be):  # test_nn.cpp:88-143
    from oracle import oracle as O
    cfg = discrete_cfg(3, 8, 4)
    p = O.params_init(cfg, 21)
    rng = CounterRng(9)
    lengths = [3, 2]
    h0 = random_obs(2, cfg.hidden_dim, rng)
    seq_obs = [random_obs(L, cfg.obs_dim, rng) for L in lengths]
    packed = np.stack([seq_obs[0][0], seq_obs[1][0], seq_obs[0][1], seq_obs[1][1], seq_obs[0][2]])
    actions = np.array([0, 1, 2, 3, 1])
    lp, en, va = fwd(be, cfg, p, packed, actions, None, [2, 2, 1], [0, 2, 4], h0)

    def chain(s):
        vals, dists = [], []
        h = h0[s:s + 1]
        for t in range(lengths[s]):
            d, v, h = O.act(cfg, p, seq_obs[s][t:t + 1], h)
            vals.append(v[0])
            dists.append(d[0])
        return vals, dists

    v0, d0 = chain(0)
    v1, d1 = chain(1)

    def rel(a, b):
        return abs(a - b) / max(1e-12, abs(a), abs(b))

    t = 1e-6 if be == "oracle" else 2e-5
    assert rel(va[0], v0[0]) < t and rel(va[1], v1[0]) < t and rel(va[2], v0[1]) < t
    assert rel(va[3], v1[1]) < t and rel(va[4], v0[2]) < t
    assert rel(lp[0], O.categorical_log_prob(d0[0], 0)) < t
    assert rel(lp[3], O.categorical_log_prob(d1[1], 3)) < t
    assert rel(lp[4], O.categorical_log_prob(d0[2], 1)) < t


def test_value_mse_gradient_fd():  # test_nn.cpp:164-208 (oracle, through ppo_loss value term)
    """The value-head gradient path checked by central differences on the oracle."""
    from oracle import oracle as O
    from paper_2210_05064_b200.hostview import make_view
    from paper_2210_05064_b200.api import PPOConfig
    cfg = discrete_cfg(3, 6, 2)
    p = O.params_init(cfg, 31)
    rng = CounterRng(13)
    hv = make_view([4], 3, 6)
    hv.obs[:] = random_obs(4, 3, rng)
    hv.done[:] = 0
    hv.returns[:] = 0.37
    ppo = PPOConfig(value_loss_coef=1.0)
    v = O.View.from_host(hv)
    b = O.pack(hv.seqs)
    h0 = np.zeros((1, 6))
    # zero advantages and alpha 0: the loss is exactly c_v * 0.5 * mean((V-R)^2)
    res = O.ppo_loss(cfg, p, v, b, ppo, 0.0, h0, True)
    names = {n: (r, c, off) for n, r, c, off in param_tensors(cfg)}
    for name in ("enc_w1", "gru_un", "value_w"):
        r_, c_, off = names[name]
        for r in range(min(2, r_)):
            for c in range(min(3, c_)):
                k = off + r * c_ + c
                pp = p.copy()
                pp[k] += 1e-5
                up = O.ppo_loss(cfg, pp, v, b, ppo, 0.0, h0, False, res["is_weights"])["loss"]
                pp[k] -= 2e-5
                dn = O.ppo_loss(cfg, pp, v, b, ppo, 0.0, h0, False, res["is_weights"])["loss"]
                fd = (up - dn) / 2e-5
                g = res["grads"][k]
                assert abs(fd - g) / max(1.0, abs(fd), abs(g)) < 1e-4


def adam(be, p, g, m, v, step, lr):
    if be == "oracle":
        from oracle import oracle as O
        return O.adam_step(p, g, m, v, step, lr)
    import paper_2210_05064_b200 as V
    return V.adam_step(p, g, m, v, step, lr)


def test_adam_zero_and_first_step(be):  # test_nn.cpp:210-234
    from oracle import oracle as O
    dt = np.float64 if be == "oracle" else np.float32
    cfg = discrete_cfg()
    p = O.params_init(cfg, 41).astype(dt)
    before = p.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    adam(be, p, np.zeros_like(p), m, v, 0, 0.01)
    assert np.abs(p - before).max() == 0
    cfg = discrete_cfg(2, 4, 2)
    p = O.params_init(cfg, 42).astype(dt)
    w0 = float(p[0])
    g = np.zeros_like(p)
    g[0] = 1.0
    m, v = np.zeros_like(p), np.zeros_like(p)
    step = adam(be, p, g, m, v, 0, 3e-3)
    assert step == 1
    assert float(p[0]) == pytest.approx(w0 - 3e-3, rel=1e-6)


def test_cosine():  # test_nn.cpp:236-242
    from paper_2210_05064_b200.api import CosineSchedule
    s = CosineSchedule(2.5e-4, 1000)
    assert s.lr_at(0) == pytest.approx(2.5e-4)
    assert s.lr_at(500) == pytest.approx(1.25e-4)
    assert s.lr_at(1000) == pytest.approx(0.0, abs=1e-12)
    assert s.lr_at(2000) == pytest.approx(0.0, abs=1e-12)


def test_categorical_entropy_mc():  # test_nn.cpp:244-278 (categorical, oracle)
    from oracle import oracle as O
    rng = CounterRng(77)
    logits = np.array([0.2, -1.0, 0.5])
    n = 20000
    s = sq = 0.0
    pr = np.exp(logits - logits.max())
    pr /= pr.sum()
    for _ in range(n):
        u = rng.uniform()
        acc, a = 0.0, len(pr) - 1
        for i, q in enumerate(pr):
            acc += q
            if u < acc:
                a = i
                break
        lp = O.categorical_log_prob(logits, a)
        s += lp
        sq += lp * lp
    mc = -s / n
    se = math.sqrt((sq / n - (s / n) ** 2) / n)
    assert abs(mc - O.categorical_entropy(logits)) < 3 * se + 1e-9
