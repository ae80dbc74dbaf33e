"""The product's multi-replica path on one B200.

* A 1-rank NCCL communicator runs every collective of the library for real:
  the learner's ncclAllReduce(avg) of the P+1 gradient buffer, the int64 / f64
  reductions and the all-gather of the replica driver.
* Two processes sharing the GPU run the PRODUCT learner as DD-PPO replicas whose
  grad_hook / entropy_hook (learner.hpp:119-122) average over gloo.  The result
  must be bit-identical across replicas and match two in-process oracle
  replicas averaging in rank order (AllReduce::average, distributed.cpp:86-116;
  test_distributed.cpp:229-286) within 1e-5.
* The replica driver (csrc/replica.cu, the learner section of
  ReplicaGroup::replica_main, distributed.cpp:208-264) over three iterations
  with a preempted rollout in the middle (backfill from the previous view),
  against the same schedule run on oracle replicas.
* Per-minibatch non-finite errors (learner.cpp:111, :139-140) with the
  reference's state at the throw.
"""
from __future__ import annotations

import os
import socket
import threading
from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T, N, H, E = 16, 8, 16, 16
WORLD = 2
PPO = dict(epochs=2, minibatches=2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg(V):
    return V.ModelConfig(obs_dim=2, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=2)


def _params(V, O):
    # the GPU path and the oracle consume the same fp32-rounded initial buffer
    return O.params_init(_cfg(V), O.mix(1, 0x9A9A)).astype(np.float32).astype(np.float64)


def _workload(rank: int, it: int):
    from paper_2210_05064_b200 import synth
    from paper_2210_05064_b200.rng import mix
    return synth.make_workload(T, N, hidden_dim=H, seed=mix(mix(1, rank), it))


def _fill(buf, wl, preempt_at=None, version=1):
    """One rollout into a product or oracle store; preempt_at truncates the
    arrival log and force-closes (a VER preemption, deficit = T*N - preempt_at)."""
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    if preempt_at is not None:
        recs = V.StepRecords(**{k: (None if v is None else np.asarray(v)[:preempt_at])
                                for k, v in wl.records.__dict__.items()})
        wl = replace(wl, records=recs, bootstrap=np.asarray(wl.bootstrap, np.float32) + 0.5,
                     bootstrap_valid=np.ones(N, np.uint8))
    synth.fill_buffer(buf, wl, snapshot_version=version)
    if preempt_at is not None:
        buf.force_close()
    return buf.close_rollout()


SCHEDULE = (None, T * N - 37, None)  # iteration 1 is preempted (deficit 37)


# ----------------------------------------------------------------- 1 rank NCCL
def test_nccl_one_rank_collectives_execute(ver):
    V = ver
    ctx = V.Context(0)
    ctx.init_nccl(V.Context.nccl_unique_id(), 1, 0)
    a = ctx.allreduce_sum_i64([3, -4, 1 << 40])
    assert list(a) == [3, -4, 1 << 40]
    b = ctx.allreduce_mean_f64([0.25, -1.5])
    assert list(b) == [0.25, -1.5]
    g = ctx.allgather_f64([1.0, 2.0, 3.0], 1)
    assert list(g) == [1.0, 2.0, 3.0]


def test_nccl_one_rank_learner_allreduce_runs(ver, oracle):
    """ncclAllReduce(avg) over one rank is the identity: the update is bit-identical
    to the one without it, and the allreduce phase has a device time."""
    V, O = ver, oracle
    cfg = _cfg(V)
    p = _params(V, O)
    wl = _workload(0, 0)
    res = []
    for on in (False, True):
        ctx = V.Context(0)
        if on:
            ctx.init_nccl(V.Context.nccl_unique_id(), 1, 0)
        L = V.Learner(cfg, p, V.PPOConfig(**PPO), V.EntropyController(), V.CosineSchedule(2.5e-4, 100_000),
                      O.mix(1, 0xF00D), ctx=ctx)
        L.enable_allreduce(on)
        view = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H, ctx=ctx), wl)
        st = L.update(view)
        res.append((L.params(), st, L.last_timing(), L.last_timing_counts(), L.alpha))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    # the mean entropy rides in the fp32 gradient buffer (slot P) and drives alpha
    # from there when a reducer is installed; without one it stays double
    assert abs(res[0][1].loss - res[1][1].loss) <= 1e-9 * abs(res[0][1].loss)
    assert abs(res[0][4] - res[1][4]) <= 1e-6 * abs(res[0][4])
    assert res[1][3]["allreduce"] == PPO["epochs"] * PPO["minibatches"]
    assert res[1][2]["allreduce"] > 0.0
    assert res[0][3]["allreduce"] == 0


def test_replica_driver_one_rank_nccl(ver, oracle):
    """ver_replica over a 1-rank NCCL communicator: global consumed steps, the
    pooled S* (optimal_preempt_steps over this replica's tau and LT), backfill."""
    V, O = ver, oracle
    cfg = _cfg(V)
    p = _params(V, O)
    ctx = V.Context(0)
    ctx.init_nccl(V.Context.nccl_unique_id(), 1, 0)
    L = V.Learner(cfg, p, V.PPOConfig(**PPO), V.EntropyController(), V.CosineSchedule(2.5e-4, 100_000),
                  O.mix(1, 0xF00D), ctx=ctx)
    rep = V.Replica(L, T, N, preempt=V.PREEMPT_OPTIMAL)
    consumed = 0
    for it, pre in enumerate(SCHEDULE):
        wl = _workload(0, it)
        view = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H, ctx=ctx), wl, pre, version=it + 1)
        wall = 0.05 * (it + 1)
        r = rep.learn(view, wall, last_iteration=(it == len(SCHEDULE) - 1))
        fresh = T * N if pre is None else pre
        assert r.global_consumed_before == consumed and r.global_fresh == fresh
        consumed += fresh
        assert r.deficit == (0 if pre is None else T * N - pre)
        assert r.stale_steps == (0 if pre is None else T * N - pre)
        counts = view.to_host().per_env_counts.astype(np.int64)
        tau = wall / np.maximum(1, counts)
        if it < len(SCHEDULE) - 1:
            assert r.mean_learn_time == r.learn_time > 0
            assert r.next_threshold == O.optimal_preempt_steps(tau, r.mean_learn_time, T * N)
        else:
            assert r.next_threshold == 0
    g, i, hp = rep.state()
    assert g == consumed and i == len(SCHEDULE) and hp


# ------------------------------------------------- two replicas on one GPU (gloo)
class _Gloo:
    def __init__(self, dist, rank):
        self.dist, self.rank, self.nranks = dist, rank, WORLD

    def sum_i64(self, a):
        import torch
        t = torch.from_numpy(a)
        self.dist.all_reduce(t)

    def mean_f64(self, a):
        import torch
        t = torch.from_numpy(a)
        self.dist.all_reduce(t)
        t /= WORLD

    def allgather_f64(self, a):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a))
        out = [torch.zeros_like(t) for _ in range(WORLD)]
        self.dist.all_gather(out, t)
        return torch.cat(out).numpy()


def _gloo_hooks(dist):
    """grad_hook / entropy_hook as AllReduce::average over gloo: D2H on the
    library stream, sum in rank order, /R, H2D back on the same stream."""
    import torch

    def avg(buf):
        dev = buf.torch()
        s = torch.cuda.ExternalStream(buf.stream, device=dev.device)
        with torch.cuda.stream(s):
            host = dev.cpu()
        dist.all_reduce(host)
        host /= WORLD
        with torch.cuda.stream(s):
            dev.copy_(host)
        s.synchronize()
    return avg, avg


def _worker(rank: int, port: int, outdir: str, mode: str):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    torch.cuda.set_device(0)
    ctx = V.Context(0)
    L = V.Learner(_cfg(V), _params(V, O), V.PPOConfig(**PPO), V.EntropyController(),
                  V.CosineSchedule(2.5e-4, 100_000), O.mix(1, 0xF00D), ctx=ctx)
    L.set_hooks(*_gloo_hooks(dist))
    out = {}
    if mode == "update":
        view = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H, ctx=ctx), _workload(rank, 0))
        st = L.update(view)
        out["loss"] = st.loss
    else:
        rep = V.Replica(L, T, N, preempt=V.PREEMPT_OPTIMAL, comm=_Gloo(dist, rank))
        thr, cons, lt = [], [], []
        for it, pre in enumerate(SCHEDULE):
            view = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H, ctx=ctx), _workload(rank, it), pre,
                         version=it + 1)
            r = rep.learn(view, 0.05 * (it + 1 + rank), last_iteration=(it == len(SCHEDULE) - 1))
            thr.append(r.next_threshold)
            cons.append(r.global_consumed_before)
            lt.append(r.mean_learn_time)
        out.update(thr=np.array(thr), cons=np.array(cons), lt=np.array(lt))
    out["params"] = L.params()
    out["alpha"] = L.alpha
    np.savez(os.path.join(outdir, f"{mode}{rank}.npz"), **out)
    dist.destroy_process_group()


def _spawn(tmp_path, mode):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path), mode), nprocs=WORLD, join=True,
                       start_method="spawn")
    return [np.load(tmp_path / f"{mode}{r}.npz") for r in range(WORLD)]


def _oracle_replicas(O, V, n_iter_schedule):
    """Two oracle replicas in threads, averaging in rank order (distributed.cpp:86-116),
    running the replica_main learner section on the same views."""
    p = _params(V, O)
    learners = [O.Learner(_cfg(V), p, V.PPOConfig(**PPO), V.EntropyController(), 2.5e-4, 100_000,
                          O.mix(1, 0xF00D)) for _ in range(WORLD)]
    bar = threading.Barrier(WORLD)
    slots, ent = [None] * WORLD, [None] * WORLD

    def hooks(r):
        def g(arr):
            slots[r] = np.array(arr, copy=True)
            bar.wait()
            tot = slots[0].copy()
            for k in range(1, WORLD):
                tot = tot + slots[k]
            bar.wait()
            arr[:] = tot / WORLD

        def e(h):
            ent[r] = h
            bar.wait()
            tot = ent[0]
            for k in range(1, WORLD):
                tot = tot + ent[k]
            bar.wait()
            return tot / WORLD
        return g, e

    for r in range(WORLD):
        learners[r].set_hooks(*hooks(r))
    prevs = [None] * WORLD
    consumed = 0
    for it, pre in n_iter_schedule:
        views = [_fill(O.Rollout(T, N, 1, 0, 2, 0, H), _workload(r, it), pre, version=it + 1) for r in range(WORLD)]
        fresh = sum(v.to_host().size for v in views)
        for r in range(WORLD):
            learners[r].set_state(learners[r].state()[0], consumed, learners[r].state()[2])
            d = views[r].to_host().deficit
            if d > 0 and prevs[r] is not None:
                O.backfill_stale(views[r], prevs[r], d)
        consumed += fresh
        th = [threading.Thread(target=learners[r].update, args=(views[r],)) for r in range(WORLD)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        prevs = views
    return learners


def test_two_replicas_hooks_match_rank_ordered_average(ver, oracle, tmp_path):
    V, O = ver, oracle
    res = _spawn(tmp_path, "update")
    np.testing.assert_array_equal(res[0]["params"], res[1]["params"])
    assert float(res[0]["alpha"]) == float(res[1]["alpha"])
    learners = _oracle_replicas(O, V, [(0, None)])
    ref = learners[0].params()
    err = np.abs(res[0]["params"] - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 1e-5, err.max()
    assert abs(float(res[0]["alpha"]) - learners[0].state()[0]) <= 1e-9


def test_two_replica_drivers_match_oracle_schedule(ver, oracle, tmp_path):
    V, O = ver, oracle
    res = _spawn(tmp_path, "replica")
    a, b = res
    np.testing.assert_array_equal(a["params"], b["params"])
    np.testing.assert_array_equal(a["thr"], b["thr"])
    np.testing.assert_array_equal(a["cons"], b["cons"])
    np.testing.assert_array_equal(a["lt"], b["lt"])
    # global consumed before each iteration: sums of both replicas' fresh steps
    fresh = [WORLD * (T * N if pre is None else pre) for pre in SCHEDULE]
    assert list(a["cons"]) == [0, fresh[0], fresh[0] + fresh[1]]
    assert a["thr"][-1] == 0
    # S* from the pooled tau of both replicas and the averaged learn time
    for it in range(len(SCHEDULE) - 1):
        taus = []
        for r in range(WORLD):
            view = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H), _workload(r, it), SCHEDULE[it])
            taus.append(0.05 * (it + 1 + r) / np.maximum(1, view.to_host().per_env_counts.astype(np.int64)))
        assert a["thr"][it] == O.optimal_preempt_steps(np.concatenate(taus), float(a["lt"][it]), T * N * WORLD)
    learners = _oracle_replicas(O, V, list(enumerate(SCHEDULE)))
    ref = learners[0].params()
    err = np.abs(a["params"] - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 1e-5, err.max()


# ------------------------------------------------------------- non-finite errors
def _nonfinite_pair(V, O, reward_nan: bool, base_lr: float):
    cfg = _cfg(V)
    p = _params(V, O)
    wl = _workload(0, 0)
    if reward_nan:
        r = np.asarray(wl.records.reward, np.float32).copy()
        r[5] = np.nan
        wl = replace(wl, records=replace(wl.records, reward=r))
    g = V.Learner(cfg, p, V.PPOConfig(**PPO), V.EntropyController(), V.CosineSchedule(base_lr, 100_000),
                  O.mix(1, 0xF00D))
    o = O.Learner(cfg, p, V.PPOConfig(**PPO), V.EntropyController(), base_lr, 100_000, O.mix(1, 0xF00D))
    vg = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H), wl)
    vo = _fill(O.Rollout(T, N, 1, 0, 2, 0, H), wl)
    with pytest.raises(V.ProtocolError) as eg:
        g.update(vg)
    with pytest.raises(Exception) as eo:
        o.update(vo)
    return g, o, str(eg.value), str(eo.value)


def test_nonfinite_loss_raises_before_adam(ver, oracle):
    """learner.cpp:111: a non-finite loss throws before backward / Adam of that
    minibatch -- parameters, Adam state, alpha and counters stay as they were."""
    V, O = ver, oracle
    g, o, mg, mo = _nonfinite_pair(V, O, reward_nan=True, base_lr=2.5e-4)
    assert "non-finite loss" in mg and "non-finite loss" in mo
    np.testing.assert_array_equal(g.params(), _params(V, O).astype(np.float32))
    _, _, step = g.adam()
    assert step == o.adam()[2] == 0
    assert g.alpha == o.state()[0]
    assert g.consumed_steps() == o.state()[1] == 0 and g.update_index() == o.state()[2] == 0


def test_nonfinite_params_raise_after_first_adam(ver, oracle):
    """learner.cpp:139-140: Adam runs, the parameters are checked, the update
    throws before the entropy update; no later minibatch runs."""
    V, O = ver, oracle
    g, o, mg, mo = _nonfinite_pair(V, O, reward_nan=False, base_lr=float("inf"))
    assert "non-finite parameters" in mg and "non-finite parameters" in mo
    assert g.adam()[2] == o.adam()[2] == 1
    assert g.alpha == o.state()[0] == V.EntropyController().alpha
    assert not np.all(np.isfinite(g.params()))
    assert g.consumed_steps() == 0 and g.update_index() == 0
    # a later update on a fresh view fails again (the parameters stay non-finite)
    vg = _fill(V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H), _workload(0, 1))
    with pytest.raises(V.ProtocolError):
        g.update(vg)
