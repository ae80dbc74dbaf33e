"""The batched append path (Variable-mode block copy, rollout.cuh append_bulk)
against the oracle store fed one record at a time: records arrive in batches
of random sizes that cross the close (carryover), across three rollouts, with
h_before on some sequence starts; closed views must be bit-identical.  Also
the batched set_bootstraps."""
import numpy as np
import pytest

from test_gpu_parity import INT_FIELDS, F_FIELDS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])
def test_batched_append_matches_oracle(mode):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    T, N, D, H = 6, 10, 2, 4
    rng = np.random.default_rng(mode + 3)
    g = V.RolloutBuffer(T, N, mode, 0, D, 0, H)
    o = O.Rollout(T, N, mode, 0, D, 0, H)
    step = np.zeros(N, np.int32)
    for roll in range(3):
        g.begin_rollout(roll + 1)
        o.begin_rollout(roll + 1)
        for _ in range(6):
            n = int(rng.integers(1, 25))
            env = rng.integers(0, N, n)
            if mode == 1:  # at most one record per env per batch after the close would be a double carryover
                env = rng.permutation(N)[:min(n, N)]
                n = env.size
            hb = rng.standard_normal((n, H)).astype(np.float32)
            recs = V.StepRecords(
                env_index=env.astype(np.int32), obs=rng.standard_normal((n, D)).astype(np.float32),
                log_prob=rng.standard_normal(n).astype(np.float32), value=rng.standard_normal(n).astype(np.float32),
                reward=rng.standard_normal(n).astype(np.float32), done=(rng.random(n) < 0.2).astype(np.uint8),
                act_disc=rng.integers(0, 2, n).astype(np.int32), episode_index=np.zeros(n, np.int64),
                step_in_episode=step[env].copy(), latency=rng.random(n).astype(np.float32), h_before=hb,
                h_before_valid=(rng.random(n) < 0.7).astype(np.uint8),
                snapshot_version=np.full(n, roll + 1, np.uint64))
            step[env] += 1
            og = g.append_steps(recs)
            oo = o.append_steps(recs)
            np.testing.assert_array_equal(og, oo)
        envs = np.arange(0, N, 3)
        vals = rng.standard_normal(envs.size).astype(np.float32)
        g.set_bootstraps(envs, vals)
        for e, v in zip(envs, vals):
            o.set_bootstrap(int(e), float(v))
        g.force_close()
        o.force_close()
        a, b = g.close_rollout().to_host(), o.close_rollout().to_host()
        assert a.size == b.size and a.num_seqs == b.num_seqs
        for f in INT_FIELDS:
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        for f in F_FIELDS:
            np.testing.assert_array_equal(getattr(a, f).astype(np.float64), getattr(b, f), err_msg=f)
