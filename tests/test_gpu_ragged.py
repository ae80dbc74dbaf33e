"""Ragged-length stress: device-generated views with
heavy-tailed env lengths 1..1024; GAE vs an independent float64 restatement,
pack/gather bit-exact vs the oracle's pack, and size-independent properties
at 2^24 steps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def gae_ref(hv, gamma, lam):
    """float64 per-env reverse recursion over the device view's own fp32 inputs."""
    r, v, d = hv.reward.astype(np.float64), hv.value.astype(np.float64), hv.done.astype(bool)
    off = np.concatenate([[0], np.cumsum(hv.per_env_counts)])
    adv = np.zeros(hv.size)
    for e in range(hv.N):
        a, b = off[e], off[e + 1]
        nv = 0.0 if d[b - 1] else float(hv.env_bootstrap[e])
        acc = 0.0
        for i in range(b - 1, a - 1, -1):
            m = 0.0 if d[i] else 1.0
            delta = r[i] + gamma * nv * m - v[i]
            acc = delta + gamma * lam * m * acc
            adv[i] = acc
            nv = v[i]
    return adv


@pytest.mark.parametrize("S", [1 << 14, 1 << 17])
def test_ragged_gae_vs_restatement(S):
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    lens = synth.ragged_lengths(S, seed=S)
    view = V.view_synth(lens, seed=3)
    V.compute_gae(view, 0.99, 0.95)
    hv = view.to_host()
    assert hv.size == S and list(hv.per_env_counts) == list(lens)
    ref = gae_ref(hv, 0.99, 0.95)
    err = np.abs(hv.advantage - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 1e-5
    np.testing.assert_allclose(hv.returns, ref + hv.value.astype(np.float64), rtol=1e-5, atol=1e-5)


def test_ragged_pack_gather_bitexact_vs_oracle():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    lens = synth.ragged_lengths(1 << 16, seed=5)
    view = V.view_synth(lens, seed=4)
    V.compute_gae(view, 0.99, 0.95)
    hv = view.to_host()
    for g in V.split_minibatches(view, 2, 77):
        b = V.pack(view, g)
        po = O.pack(g.seqs)
        np.testing.assert_array_equal(b.slots, po.slots)
        np.testing.assert_array_equal(b.batch_sizes, po.batch_sizes)
        ga = b.gathered(2)
        s = b.slots
        for k, f in (("obs", "obs"), ("act_disc", "act_disc"), ("old_logp", "log_prob"), ("adv", "advantage"),
                     ("ret", "returns")):
            np.testing.assert_array_equal(ga[k], getattr(hv, f)[s])


def test_ragged_2p24_properties():
    """2^24 steps: the deal covers every slot once, batch sizes non-increasing,
    GAE finite and zero-error at dones (A = r - V)."""
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    S = 1 << 24
    lens = synth.ragged_lengths(S, seed=7)
    view = V.view_synth(lens, seed=8)
    gae_ms, gather_ms = V.bench_gae_gather(view, B=2, seed=9, reps=2)
    assert gae_ms > 0 and gather_ms > 0
    hv = view.to_host()
    d = hv.done.astype(bool)
    np.testing.assert_allclose(hv.advantage[d], (hv.reward[d].astype(np.float64) - hv.value[d]), rtol=1e-6,
                               atol=1e-6)
    assert np.isfinite(hv.advantage).all()
    seen = 0
    for g in V.split_minibatches(view, 2, 9):
        b = V.pack(view, g)
        bs = b.batch_sizes
        assert np.all(np.diff(bs) <= 0) and int(bs.sum()) == b.total_steps
        seen += b.total_steps
    assert seen == S
