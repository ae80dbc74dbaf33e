"""Joint preemption counter (csrc/coordinator.cu, SURVEY §8(f) row 2;
PreemptCoordinator, distributed.hpp:95-128) across two processes on one device:
replica 0 owns the counter and exports its IPC handle, replica 1 opens it;
both add steps concurrently; exactly one add fires, at the first total >= the
threshold, and a threshold <= 0 never fires (per-replica-budget ablation)."""
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = textwrap.dedent("""
    import sys, time
    sys.path.insert(0, {root!r})
    import paper_2210_05064_b200 as V
    h = bytes.fromhex(open({hpath!r}).read().strip())
    c = V.PreemptCounter(handle=h)
    fired = []
    for i in range({n}):
        t, f = c.add_steps({step})
        if f:
            fired.append(t)
    print("child", len(fired), *fired)
""")


def test_counter_fires_once_across_processes(tmp_path):
    import paper_2210_05064_b200 as V
    own = V.PreemptCounter()
    hpath = tmp_path / "h.txt"
    hpath.write_text(own.ipc_handle().hex())
    for threshold, n, step in ((1000, 400, 3), (0, 200, 5)):
        own.start_iteration(threshold)
        child = subprocess.Popen([sys.executable, "-c", CHILD.format(root=str(ROOT), hpath=str(hpath), n=n,
                                                                      step=step)],
                                 stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
        mine = []
        for i in range(n):
            t, f = own.add_steps(2)
            if f:
                mine.append(t)
        out, err = child.communicate(timeout=300)
        assert child.returncode == 0, err
        parts = out.split()
        theirs = [int(x) for x in parts[2:]] if parts[0] == "child" else []
        total, fired = own.state()
        if threshold > 0:
            assert total == n * 2 + n * step
            assert fired and len(mine) + len(theirs) == 1
            t_fire = (mine + theirs)[0]
            assert threshold <= t_fire < threshold + max(2, step)
        else:  # disabled: add_steps returns without counting (distributed.hpp:111)
            assert total == 0 and not fired and not mine and not theirs


# ---------------------------------------------------- engine-fused commit add
def _engine(V, N=48, T=16, H=16, seed=7):
    from paper_2210_05064_b200.rng import mix
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
    params = V.params_init(cfg, mix(1, 0x9A9A))
    return V.InferenceEngine(cfg, T, N, params, version=1, mode=V.VARIABLE, seed=seed)


def _collect(eng, N, rng, max_batches=200):
    """Batches of every env until the rollout closes: (new_commits per batch, results)."""
    import numpy as np
    env = np.arange(N, dtype=np.int32)
    step = np.zeros(N, np.int32)
    ep = np.zeros(N, np.int64)
    eng.begin_rollout()
    eng.process_arrays(env, rng.standard_normal((N, 2)).astype(np.float32), first=np.ones(N, np.uint8),
                       obs_episode=ep, obs_step=step)
    out = []
    for _ in range(max_batches):
        step += 1
        r, _, _ = eng.process_arrays(env, rng.standard_normal((N, 2)).astype(np.float32),
                                     reward=np.ones(N, np.float32), done=np.zeros(N, np.uint8),
                                     obs_episode=ep, obs_step=step)
        out.append(r)
        if r.closed_now:
            break
    return out


def test_engine_commits_go_to_the_counter_from_the_sampling_kernel():
    """runtime.cpp:592: every process_batch's new commits are added (begin_rollout's
    carryovers are not); with a threshold beyond the rollout nothing fires."""
    import numpy as np
    import paper_2210_05064_b200 as V
    N, T = 48, 16
    own = V.PreemptCounter()
    eng = _engine(V, N, T)
    eng.attach_preempt(own)
    own.start_iteration(10 * N * T)
    res = _collect(eng, N, np.random.default_rng(3))
    total, fired = own.state()
    assert total == sum(r.new_commits for r in res) > 0
    assert not fired and not any(r.preempt_fired for r in res)
    eng.attach_preempt(None)


@pytest.mark.parametrize("threshold", [1, 100, 300])
def test_engine_force_closes_when_the_group_fires(threshold):
    """distributed.hpp:110-119 + runtime.cpp:596-599: the batch whose commits reach
    the threshold fires, and that batch force-closes the engine's rollout."""
    import numpy as np
    import paper_2210_05064_b200 as V
    N, T = 48, 16
    own = V.PreemptCounter()
    eng = _engine(V, N, T)
    eng.attach_preempt(own)
    own.start_iteration(threshold)
    res = _collect(eng, N, np.random.default_rng(4))
    last = res[-1]
    total, fired = own.state()
    committed = sum(r.new_commits for r in res)
    assert fired and last.preempt_fired and last.closed_now
    assert total == committed and threshold <= committed < threshold + N
    assert not any(r.preempt_fired for r in res[:-1])
    assert eng.rollout_done() and eng.committed() == committed


PEER = textwrap.dedent("""
    import sys
    sys.path.insert(0, {root!r})
    import paper_2210_05064_b200 as V
    c = V.PreemptCounter(handle=bytes.fromhex(open({hpath!r}).read().strip()))
    t, f = c.add_steps({n})
    print("peer", t, int(f))
""")


def test_engine_sees_a_peer_replica_fire(tmp_path):
    """Another replica (process) fires the group: this engine force-closes at its next batch."""
    import numpy as np
    import paper_2210_05064_b200 as V
    N, T = 48, 16
    own = V.PreemptCounter()
    hpath = tmp_path / "h.txt"
    hpath.write_text(own.ipc_handle().hex())
    eng = _engine(V, N, T)
    eng.attach_preempt(own)
    own.start_iteration(1000)
    rng = np.random.default_rng(5)
    env = np.arange(N, dtype=np.int32)
    step = np.zeros(N, np.int32)
    ep = np.zeros(N, np.int64)

    def batch():
        step[:] += 1
        r, _, _ = eng.process_arrays(env, rng.standard_normal((N, 2)).astype(np.float32),
                                     reward=np.ones(N, np.float32), done=np.zeros(N, np.uint8), obs_episode=ep,
                                     obs_step=step)
        return r

    eng.begin_rollout()
    eng.process_arrays(env, rng.standard_normal((N, 2)).astype(np.float32), first=np.ones(N, np.uint8),
                       obs_episode=ep, obs_step=step)
    r = batch()
    assert not r.preempt_fired and not r.closed_now
    out = subprocess.run([sys.executable, "-c", PEER.format(root=str(ROOT), hpath=str(hpath), n=1000)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    _, t, f = out.stdout.split()
    assert int(f) == 1 and int(t) == 1000 + N
    r = batch()
    assert r.preempt_fired and r.closed_now and eng.rollout_done()


# ----------------------------------------------------------- NCCL tick mode
def test_nccl_tick_counter_one_rank():
    """the global committed-step count as ncclAllReduce(int64) per
    tick; adds (host or engine) accumulate locally until the collective."""
    import numpy as np
    import paper_2210_05064_b200 as V
    ctx = V.Context(0)
    ctx.init_nccl(V.Context.nccl_unique_id(), 1, 0)
    c = V.PreemptCounter(ctx, nccl=True)
    c.start_iteration(50)
    c.add_steps(20)
    assert c.tick() == (20, False)
    c.add_steps(25)
    c.add_steps(15)
    assert c.tick() == (60, True)
    assert c.tick() == (60, False)  # fires once per iteration
    c.start_iteration(0)            # disabled: counts, never fires
    c.add_steps(7)
    assert c.tick() == (7, False)
    # an engine on the same ctx feeds the local delta from its sampling kernel
    N, T = 32, 8
    from paper_2210_05064_b200.rng import mix
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=16, hidden_dim=16, action_kind=0, num_actions=2)
    eng = V.InferenceEngine(cfg, T, N, V.params_init(cfg, mix(1, 0x9A9A)), version=1, mode=V.VARIABLE, seed=3,
                            ctx=ctx)
    eng.attach_preempt(c)
    c.start_iteration(10 * N * T)
    res = _collect(eng, N, np.random.default_rng(6))
    total, fired = c.tick()
    assert total == sum(r.new_commits for r in res) and not fired
