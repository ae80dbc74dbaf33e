"""Port of the reference's tests/test_distributed.cpp: preemption estimator
known answers and oracles, optimal preemption vs exhaustive argmax, gradient
linearity of the averaged half-batch grads (the DD-PPO AllReduce contract)."""
import numpy as np
import pytest

from backends import BACKENDS, make_backend, protocol_errors
from paper_2210_05064_b200.api import ModelConfig, PPOConfig
from paper_2210_05064_b200.rng import CounterRng


@pytest.fixture(params=BACKENDS)
def be(request):
    return make_backend(request.param)


def merged_time_oracle(tau, steps):  # test_distributed.cpp:16-24
    if steps == 0:
        return 0.0
    ys = sorted(float(k) * t for t in tau for k in range(1, steps + 1))
    return ys[steps - 1]


def argmax_oracle(tau, lt, smax):  # test_distributed.cpp:26-37
    best_s, best = 1, -1.0
    for s in range(1, smax + 1):
        r = s / (merged_time_oracle(tau, s) + lt)
        if r > best:
            best, best_s = r, s
    return best_s


def test_estimate_uniform(be):  # test_distributed.cpp:61-70
    tau = [0.5] * 4
    assert be.estimate_time(tau, 40, 0) == 0.0
    assert be.estimate_time(tau, 40, 1) == pytest.approx(0.5)
    assert be.estimate_time(tau, 40, 4) == pytest.approx(0.5)
    assert be.estimate_time(tau, 40, 5) == pytest.approx(1.0)
    assert be.estimate_time(tau, 40, 11) == pytest.approx(1.5)


def test_estimate_two_envs(be):  # test_distributed.cpp:72-79
    tau = [1.0, 2.0]
    assert be.estimate_time(tau, 10, 3) == pytest.approx(2.0)
    assert be.estimate_time(tau, 10, 1) == pytest.approx(1.0)
    assert be.estimate_time(tau, 10, 2) == pytest.approx(2.0)


def test_estimate_rejects_above_budget(be):  # test_distributed.cpp:81-86
    with pytest.raises(protocol_errors()):
        be.estimate_time([1.0], 4, 5)


def test_estimate_vs_merge_oracle(be):  # test_distributed.cpp:88-102
    rng = CounterRng(31)
    for trial in range(50):
        n = 2 + int(rng.uniform_int(6))
        tau = [0.01 + rng.uniform() * 2.0 for _ in range(n)]
        for s in (1, 7, 23, 60):
            a = be.estimate_time(tau, 60, s)
            b = merged_time_oracle(tau, s)
            assert abs(a - b) <= 1e-12 * max(1.0, abs(b))


def test_optimal_linear_full_budget(be):  # test_distributed.cpp:104-110
    assert be.optimal_preempt_steps([1.0, 1.0], 100.0, 16) == 16


def test_optimal_slow_env_preempts(be):  # test_distributed.cpp:112-120
    tau = [0.1, 0.1, 0.1, 10.0]
    s = be.optimal_preempt_steps(tau, 0.05, 32)
    assert s < 32
    assert s == argmax_oracle(tau, 0.05, 32)


def test_optimal_vs_exhaustive(be):  # test_distributed.cpp:122-132
    rng = CounterRng(77)
    for trial in range(100):
        n = 2 + int(rng.uniform_int(5))
        tau = [0.02 + rng.uniform() for _ in range(n)]
        lt = 0.01 + rng.uniform() * 0.5
        smax = 10 + int(rng.uniform_int(60))
        assert be.optimal_preempt_steps(tau, lt, smax) == argmax_oracle(tau, lt, smax)


def test_sorted_formulation_equals_reference_scan():
    """The sort formulation the device uses == the reference's exact scan (oracle, double)."""
    from oracle import oracle as O
    rng = CounterRng(123)
    for trial in range(60):
        n = 1 + int(rng.uniform_int(12))
        tau = [0.001 + rng.uniform() * 0.01 * (1 + 9 * (i % 2)) for i in range(n)]
        lt = 0.001 + rng.uniform() * 0.2
        smax = 1 + int(rng.uniform_int(300))
        assert O.optimal_preempt_steps_sorted(tau, lt, smax) == O.optimal_preempt_steps(tau, lt, smax)


@pytest.mark.gpu
def test_device_preemption_at_scale():
    """C4-scale preemption (32,768 pooled step times, S_max = 4.19M): device sort
    formulation == the oracle's sort formulation; Time(S) bit-exact vs the
    reference's bisection at sampled S."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    rng = np.random.default_rng(0)
    tau = 0.002 * np.exp(0.75 * rng.standard_normal(32768))
    smax = 128 * 32768
    lt = 0.5 * 0.35
    for s in (1, 1000, 123457, smax // 2, smax):
        assert V.estimate_time(tau, smax, s) == O.estimate_time(tau, smax, s)
    assert V.optimal_preempt_steps(tau, lt, smax) == O.optimal_preempt_steps_sorted(tau, lt, smax)


def test_gradient_linearity_oracle():  # test_distributed.cpp:150-227
    from oracle import oracle as O
    from paper_2210_05064_b200.hostview import HostView
    cfg = ModelConfig(obs_dim=2, encoder_dim=4, hidden_dim=4, action_kind=0, num_actions=2)
    p = O.params_init(cfg, 5)
    hv = build_two_seq_view()
    v = O.View.from_host(hv)
    ppo = PPOConfig()
    ra = O.ppo_loss(cfg, p, v, O.pack(hv.seqs[:1]), ppo, 0.0, hv.h0[:1], True)
    rb = O.ppo_loss(cfg, p, v, O.pack(hv.seqs[1:]), ppo, 0.0, hv.h0[1:], True)
    ru = O.ppo_loss(cfg, p, v, O.pack(hv.seqs), ppo, 0.0, np.zeros((2, 4)), True)
    assert np.abs(0.5 * (ra["grads"] + rb["grads"]) - ru["grads"]).max() < 1e-12


def build_two_seq_view():
    from paper_2210_05064_b200.hostview import HostView
    len_, n_seqs = 3, 2
    total = len_ * n_seqs
    hv = HostView.empty(total, n_seqs, 0, 2, 0, 4, total, n_seqs, fdtype=np.float64)
    hv.log_prob[:] = -0.7
    hv.advantage[:] = 1.0
    hv.returns[:] = 0.5
    hv.version[:] = 1
    hv.per_env_counts[:] = len_
    hv.env_bootstrap_valid[:] = 1
    at = 0
    for s in range(n_seqs):
        hv.seqs[s] = (s, s, len_, at, s, 0, at, 0)
        for t in range(len_):
            hv.obs[at] = (0.1 * t, 0.3 * s)
            hv.act_disc[at] = (t + s) % 2
            hv.env_index[at] = s
            hv.seq_of_slot[at] = s
            hv.step_in_episode[at] = t
            at += 1
    return hv


@pytest.mark.gpu
def test_gradient_linearity_device():
    """Same contract on the device: averaged half-batch grads == union grads (fp32)."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = ModelConfig(obs_dim=2, encoder_dim=4, hidden_dim=4, action_kind=0, num_actions=2)
    p = O.params_init(cfg, 5)
    hv = build_two_seq_view()
    v = V.RolloutView.from_host(hv)
    ppo = PPOConfig()
    ra = V.ppo_loss(cfg, p, v, V.pack(v, V.SequenceGroup(hv.seqs[:1])), ppo, 0.0, hv.h0[:1])
    rb = V.ppo_loss(cfg, p, v, V.pack(v, V.SequenceGroup(hv.seqs[1:])), ppo, 0.0, hv.h0[1:])
    ru = V.ppo_loss(cfg, p, v, V.pack(v, V.SequenceGroup(hv.seqs)), ppo, 0.0, np.zeros((2, 4)))
    d = 0.5 * (ra.grads.astype(np.float64) + rb.grads) - ru.grads
    assert np.abs(d).max() < 1e-6
