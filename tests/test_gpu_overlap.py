"""Overlapped collection and learning (paper_2210_05064_b200/overlap.py, SURVEY
§8(f) row 4, the reference's overlap mode bench.cpp:129-160):

* the threaded schedule (engine and learner on separate streams and host
  threads) gives bit-identical parameters to the same schedule run serially
  (collect rollout k+1 with snapshot k, then update on rollout k);
* the lag-1 rollouts are fully stale after restale, rollout 0 is not
  (test_runtime.cpp:349-386)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T, N, D = 8, 16, 2


def _collect_fn(seed):
    import paper_2210_05064_b200 as V
    state = {"k": 0}

    def collect(eng):
        rng = np.random.default_rng(seed + state["k"])
        state["k"] += 1
        eng.begin_rollout()
        env = np.arange(N, dtype=np.int32)
        step = np.zeros(N, np.int32)
        ep = np.zeros(N, np.int64)
        eng.process_arrays(env, rng.standard_normal((N, D)).astype(np.float32), first=np.ones(N, np.uint8),
                           obs_episode=ep, obs_step=step)
        while not eng.rollout_done():
            step += 1
            done = (rng.random(N) < 0.1).astype(np.uint8)
            eng.process_arrays(env, rng.standard_normal((N, D)).astype(np.float32),
                               reward=rng.standard_normal(N).astype(np.float32), done=done, obs_episode=ep,
                               obs_step=step)
            ep += done
            step[done == 1] = 0
        eng.finalize_bootstraps()
        return eng.close()
    return collect


def _pair(E=16, H=16):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    cfg = V.ModelConfig(obs_dim=D, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=2)
    p = O.params_init(cfg, O.mix(4, 0x9A9A)).astype(np.float32)
    ce, cl = V.Context(0), V.Context(0)
    eng = V.InferenceEngine(cfg, T, N, p, version=0, mode=V.VARIABLE, seed=9, ctx=ce)
    lrn = V.Learner(cfg, p, V.PPOConfig(epochs=2, minibatches=2), run_seed=5, ctx=cl)
    return eng, lrn


@pytest.mark.parametrize("H", [16, 512])
def test_overlapped_equals_serial_schedule(H):
    from paper_2210_05064_b200.overlap import OverlappedTrainer
    eng, lrn = _pair(H, H)
    tr = OverlappedTrainer(eng, lrn, _collect_fn(100))
    stale = []
    tr.prime()
    for u in range(3):
        v = tr.pending
        tr.iteration()
        stale.append((v.stale_steps, v.size()))
    p_over = lrn.params()
    assert stale[0][0] == 0 and all(s == n for s, n in stale[1:]), stale

    eng2, lrn2 = _pair(H, H)
    collect = _collect_fn(100)
    view = collect(eng2)
    for u in range(3):
        nxt = collect(eng2)  # rollout u+1 with snapshot u
        view.restale(u)
        lrn2.update(view)
        eng2.set_snapshot_from(lrn2, u + 1)
        view = nxt
    np.testing.assert_array_equal(p_over, lrn2.params())
