"""World-size-2 CPU tests of the N>1 path over torch.distributed `gloo`.

The GPU learner's multi-GPU exchange is one ncclAllReduce(avg) of the flat P+1
gradient buffer per minibatch plus the preemption reductions.
Without GPUs here, the same protocol is exercised with the oracle learners as
replicas and gloo as the transport:

* distributed.cpp:135-157: each replica seeds its collection with mix(1, rank),
  shares params / run_seed, and averages gradients (grad_hook) and the mean
  entropy (entropy_hook) across replicas before Adam.
* test_distributed.cpp:229-286: replicas stay bit-identical; the result equals
  the rank-ordered average computed in one process.
* distributed.cpp:208-264: every replica computes the same S* from the
  all-gathered per-env step times and the averaged learn time.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_05064_b200.api import EntropyController, ModelConfig, PPOConfig
from paper_2210_05064_b200.rng import mix

T, N, H = 16, 8, 16
WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg():
    return ModelConfig(obs_dim=2, encoder_dim=16, hidden_dim=H, action_kind=0, num_actions=2)


def _replica_view(rank: int):
    """One replica's closed rollout (collection seed mix(1, rank), distributed.cpp:137)."""
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    wl = synth.make_workload(T, N, hidden_dim=H, seed=mix(1, rank))
    r = O.Rollout(T, N, 1, 0, 2, 0, H)
    synth.fill_buffer(r, wl)
    return r.close_rollout(), wl


def _learner(params):
    from oracle import oracle as O
    return O.Learner(_cfg(), params, PPOConfig(epochs=2, minibatches=2), EntropyController(),
                     2.5e-4, 1_000_000, mix(1, 0xF00D))


def _worker(rank: int, port: int, outdir: str):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from oracle import oracle as O
    params = O.params_init(_cfg(), mix(1, 0x9A9A))
    view, wl = _replica_view(rank)
    L = _learner(params)

    def grad_hook(g):  # AllReduce::average (distributed.cpp:86-101)
        t = torch.from_numpy(np.array(g, copy=True))
        dist.all_reduce(t)
        g[:] = t.numpy() / WORLD

    def entropy_hook(h):  # AllReduce::average_scalar (distributed.cpp:103-116)
        t = torch.tensor([h], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item()) / WORLD

    L.set_hooks(grad_hook, entropy_hook)
    st = L.update(view)
    p = torch.from_numpy(L.params())
    gathered = [torch.zeros_like(p) for _ in range(WORLD)]
    dist.all_gather(gathered, p)

    # preemption inputs: per-env step times of this replica, learn time, fresh steps
    tau = torch.from_numpy(np.asarray(wl.tau, np.float64))
    taus = [torch.zeros_like(tau) for _ in range(WORLD)]
    dist.all_gather(taus, tau)
    lt = torch.tensor([0.25 + 0.1 * rank], dtype=torch.float64)
    dist.all_reduce(lt)
    lt = float(lt.item()) / WORLD
    fresh = torch.tensor([view.to_host().fresh_steps()], dtype=torch.int64)
    dist.all_reduce(fresh)
    pooled = torch.cat(taus).numpy()
    s_star = O.optimal_preempt_steps(pooled, lt, T * N * WORLD)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), params=np.stack([g.numpy() for g in gathered]),
             s_star=s_star, fresh=int(fresh.item()), loss=st["loss"], pooled=pooled, lt=lt)
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_run(tmp_path_factory):
    out = tmp_path_factory.mktemp("gloo")
    mp.start_processes(_worker, args=(_free_port(), str(out)), nprocs=WORLD, join=True, start_method="spawn")
    return [np.load(out / f"rank{r}.npz") for r in range(WORLD)]


def test_replicas_bit_identical(gloo_run):
    """After an update with averaged grads every replica holds the same params."""
    for res in gloo_run:
        p = res["params"]
        assert np.array_equal(p[0], p[1])
    assert np.array_equal(gloo_run[0]["params"], gloo_run[1]["params"])


def test_matches_rank_ordered_average(gloo_run):
    """gloo replicas == two in-process replicas averaging in rank order
    (AllReduce::average, distributed.cpp:86-101; test_distributed.cpp:229-286)."""
    from oracle import oracle as O
    params = O.params_init(_cfg(), mix(1, 0x9A9A))
    views = [_replica_view(r)[0] for r in range(WORLD)]
    learners = [_learner(params) for _ in range(WORLD)]
    bar = threading.Barrier(WORLD)
    slots = [None] * WORLD
    lock = threading.Lock()

    def make_hooks(r):
        def grad_hook(g):
            slots[r] = np.array(g, copy=True)
            bar.wait()
            total = slots[0].copy()
            for k in range(1, WORLD):
                total = total + slots[k]
            bar.wait()
            g[:] = total / WORLD

        def entropy_hook(h):
            with lock:
                make_hooks.ent[r] = h
            bar.wait()
            tot = make_hooks.ent[0]
            for k in range(1, WORLD):
                tot = tot + make_hooks.ent[k]
            bar.wait()
            return tot / WORLD
        return grad_hook, entropy_hook

    make_hooks.ent = [None] * WORLD
    for r in range(WORLD):
        learners[r].set_hooks(*make_hooks(r))
    th = [threading.Thread(target=learners[r].update, args=(views[r],)) for r in range(WORLD)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ref = learners[0].params()
    assert np.array_equal(ref, learners[1].params())
    assert np.abs(gloo_run[0]["params"][0] - ref).max() <= 1e-12


def test_preemption_agrees_across_ranks(gloo_run):
    """Every replica computes the same S* from the all-gathered tau and averaged LT."""
    from oracle import oracle as O
    a, b = gloo_run
    assert int(a["s_star"]) == int(b["s_star"])
    assert int(a["fresh"]) == int(b["fresh"])
    assert np.array_equal(a["pooled"], b["pooled"])
    assert int(a["s_star"]) == O.optimal_preempt_steps(a["pooled"], float(a["lt"]), T * N * WORLD)
    assert 1 <= int(a["s_star"]) <= T * N * WORLD
