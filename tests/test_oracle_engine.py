"""The oracle's inference-engine restatement (oracle/engine.py), pinned on CPU:
* mix / splitmix64 against the C++ oracle's rng::mix (rng.hpp:16-25);
* ports of the reference's RNG property tests (test_rng.cpp) and the sampler
  Monte-Carlo entropy test (test_nn.cpp:237-278);
* the engine protocol (runtime.cpp:116-215): completion without an action and
  requests for parked envs raise ProtocolError; Fixed-mode caps park envs;
  a Variable-mode close sends late completions to carryover, consumed by the
  next begin_rollout."""
import math

import numpy as np
import pytest

from engine_driver import Driver


def test_mix_matches_cpp_oracle():
    from oracle import engine as OE
    from oracle import oracle as O
    rng = np.random.default_rng(3)
    for _ in range(200):
        a, b = (int(x) for x in rng.integers(0, 2 ** 63, 2, dtype=np.int64))
        assert OE.mix(a, b) == O.mix(a, b)


def test_counter_rng_properties():
    from oracle.engine import CounterRng
    a, b = CounterRng(42).stream(3, 7), CounterRng(42).stream(3, 7)
    assert all(a.next_u64() == b.next_u64() for _ in range(100))
    base = CounterRng(7)
    s1, s2 = base.stream(1), base.stream(2)
    x, y = s1.next_u64(), s2.next_u64()
    assert y == CounterRng(7).stream(2).next_u64() and x == CounterRng(7).stream(1).next_u64()
    seen = {CounterRng(1).stream(e, ep).next_u64() for e in range(64) for ep in range(16)}
    assert len(seen) == 64 * 16
    r = CounterRng(5)
    assert all(0.0 <= r.uniform() < 1.0 for _ in range(1000))
    r = CounterRng(11)
    z = np.array([r.normal() for _ in range(20000)])
    assert abs(z.mean()) < 0.03 and abs((z * z).mean() - 1.0) < 0.05


def test_sampled_log_probs_estimate_entropy():
    from oracle import engine as OE
    from oracle import oracle as O
    rng = OE.CounterRng(77)
    logits = np.array([0.2, -1.0, 0.5])
    lp = np.array([O.categorical_log_prob(logits, OE.sample_categorical(logits, rng)[0]) for _ in range(20000)])
    se = math.sqrt(lp.var() / lp.size)
    assert abs(-lp.mean() - O.categorical_entropy(logits)) < 3 * se + 1e-9
    mean, log_std = np.array([0.3, -0.2]), np.array([-0.5, 0.1])
    lp = np.array([OE.gaussian_log_prob(mean, log_std, OE.sample_gaussian(mean, log_std, rng)) for _ in range(20000)])
    se = math.sqrt(lp.var() / lp.size)
    ent = log_std.sum() + 0.5 * (1.0 + math.log(2 * math.pi)) * 2
    assert abs(-lp.mean() - ent) < 3 * se + 1e-9


def _cfg(action_kind=0):
    import paper_2210_05064_b200 as V
    if action_kind:
        return V.ModelConfig(obs_dim=3, encoder_dim=8, hidden_dim=8, action_kind=1, act_dim=2)
    return V.ModelConfig(obs_dim=3, encoder_dim=8, hidden_dim=8, action_kind=0, num_actions=3)


def _engine(mode, T=4, N=6, action_kind=0):
    from oracle import engine as OE
    from oracle import oracle as O
    cfg = _cfg(action_kind)
    p = O.params_init(cfg, O.mix(9, 0x9A9A))
    return OE.Engine(cfg, T, N, p, version=1, mode=mode, seed=O.mix(5, 0xF00D)), OE


def test_protocol_errors():
    from oracle import oracle as O
    e, OE = _engine(1)
    e.begin_rollout()
    with pytest.raises(O.OracleProtocolError):
        e.process_batch([OE.Request(0, np.zeros(3, np.float32))])  # no outstanding action
    e.process_batch([OE.Request(1, np.zeros(3, np.float32), first=True)])
    e.force_close()
    e.process_batch([OE.Request(2, np.zeros(3, np.float32), first=True)])  # closed -> parked
    with pytest.raises(O.OracleProtocolError):
        e.process_batch([OE.Request(2, np.zeros(3, np.float32), first=True)])


@pytest.mark.parametrize("mode", [0, 1])
def test_engine_rollouts(mode):
    e, OE = _engine(mode)
    N, T = e.N, e.T
    drv = Driver(N, 3, seed=4)
    for rollout in range(3):
        res = e.begin_rollout()
        drv.unpark([d[0] for d in res.dispatches])
        ticks = 0
        while e._open() and ticks < 500:
            reqs = drv.requests(OE.Request)
            res = e.process_batch(reqs)
            drv.after(reqs, [d[0] for d in res.dispatches])
            ticks += 1
        e.finalize_bootstraps()
        v = e.close().to_host()
        assert v.size == T * N
        if mode == 0:
            np.testing.assert_array_equal(v.per_env_counts, np.full(N, T))
        # every sequence starts at an env's first slot or right after a done
        for s in v.seqs:
            st = s[3]
            assert st == 0 or v.env_index[st - 1] != v.env_index[st] or v.done[st - 1]
