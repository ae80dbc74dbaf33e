"""Synthetic heterogeneous-environment learner inputs.

Deterministic from one seed through CounterRng streams (rng.hpp):
  * per-env step time  tau_e = 2 ms * exp(0.75 z_e)      (SPEC.md:595 latency model)
  * VER per-env counts c_e >= 1, sum c_e = T*N, c_e ~ 1/tau_e by largest
    remainder (the accounting test_runtime.cpp:75-89 pins)
  * arrival order = completion time (k+1) tau_e (ties -> env order)
  * episodes: done ~ Bernoulli(1/32) per step (geometric lengths, mean 32,
    random phase); an env's last step without `done` gets a bootstrap ~ N(0,1)
  * obs ~ N(0,1)^D, action ~ U{0..A-1}, reward ~ N(0,1), value ~ N(0,1),
    h_before ~ N(0, 0.5^2) at rollout-start sequences, zeros at episode starts
  * old log-prob = -log(A) + N(0, 0.1^2): the initial policy's log-prob
    (head gain 0.01 makes it -log A to 1e-2) perturbed so clipping and IS < 1 occur
Everything is rounded to fp32 once; the oracle upcasts the same values.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import StepRecords
from .rng import CounterRng, normal_np, uniform_np


@dataclass
class Workload:
    T: int
    N: int
    obs_dim: int
    num_actions: int
    hidden_dim: int
    records: StepRecords          # arrival order
    counts: np.ndarray            # per env
    tau: np.ndarray               # per env step time (s)
    bootstrap: np.ndarray         # per env V(next obs) (fp32)
    bootstrap_valid: np.ndarray   # per env


def ver_counts(tau: np.ndarray, total: int) -> np.ndarray:
    """Largest-remainder apportionment of `total` steps proportional to 1/tau, each >= 1."""
    n = tau.size
    if total < n:
        raise ValueError("T*N must be >= N")
    w = (1.0 / tau) / np.sum(1.0 / tau)
    raw = w * total
    c = np.maximum(1, np.floor(raw)).astype(np.int64)
    frac = raw - np.floor(raw)
    d = total - int(c.sum())
    order = np.lexsort((np.arange(n), -frac))  # largest fraction first, env order on ties
    i = 0
    while d > 0:
        c[order[i % n]] += 1
        d -= 1
        i += 1
    if d < 0:
        order = np.lexsort((np.arange(n), frac))
        i = 0
        while d < 0:
            e = order[i % n]
            if c[e] > 1:
                c[e] -= 1
                d += 1
            i += 1
    return c


def make_workload(T: int, N: int, obs_dim: int = 2, num_actions: int = 2, hidden_dim: int = 64,
                  seed: int = 1, logp_sigma: float = 0.1, p_done: float = 1.0 / 32) -> Workload:
    root = CounterRng(seed)
    key = lambda i: root.stream(i).key  # noqa: E731
    z = normal_np(key(1), N)
    tau = 0.002 * np.exp(0.75 * z)
    counts = ver_counts(tau, T * N)
    S = int(counts.sum())
    # arrival order by completion time (k+1)*tau_e, ties broken by env index
    env_of = np.repeat(np.arange(N, dtype=np.int32), counts)
    rank = np.concatenate([np.arange(c, dtype=np.int32) for c in counts])
    t_done = (rank + 1).astype(np.float64) * tau[env_of]
    order = np.lexsort((rank, env_of, t_done))
    env = env_of[order]
    rk = rank[order]
    # per-step payload drawn in (env, rank) order then permuted to arrival order
    obs = normal_np(key(2), S * obs_dim).reshape(S, obs_dim).astype(np.float32)
    act = np.minimum((uniform_np(key(3), np.arange(S)) * num_actions).astype(np.int32),
                     num_actions - 1)
    reward = normal_np(key(4), S).astype(np.float32)
    value = normal_np(key(5), S).astype(np.float32)
    done = (uniform_np(key(6), np.arange(S)) < p_done).astype(np.uint8)
    logp = (-np.log(num_actions) + logp_sigma * normal_np(key(8), S)).astype(np.float32)
    # episode bookkeeping per env (vectorised over the env-major order)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    phase = (uniform_np(key(10), np.arange(N)) * 32).astype(np.int64)
    ep_start = np.zeros(S, bool)
    ep_start[starts] = True  # rollout start of each env
    prev_done = np.zeros(S, bool)
    prev_done[1:] = done[:-1].astype(bool)
    prev_done[starts] = False
    new_ep = prev_done
    # step_in_episode: steps since last done (the first episode has a random phase)
    seg = np.cumsum(new_ep | ep_start) - 1
    seg_first = np.flatnonzero(new_ep | ep_start)
    pos = np.arange(S) - seg_first[seg]
    first_seg_of_env = np.searchsorted(seg_first, starts)
    is_first_seg = np.zeros(seg_first.size, bool)
    is_first_seg[first_seg_of_env] = True
    env_major_env = np.repeat(np.arange(N), counts)
    step_in_ep = pos + np.where(is_first_seg[seg], phase[env_major_env], 0)
    ep_idx = np.cumsum(new_ep) - np.cumsum(new_ep)[starts][env_major_env] + 1000 * env_major_env
    # h_before: rollout-start sequences N(0, 0.5^2) unless at an episode start; zeros otherwise
    hb = np.zeros((S, hidden_dim), np.float32)
    first_is_ep_start = phase == 0
    hrows = normal_np(key(7), N * hidden_dim).reshape(N, hidden_dim) * 0.5
    for e in np.flatnonzero(~first_is_ep_start):
        hb[starts[e]] = hrows[e]
    # bootstrap for truncated tails
    last = starts + counts - 1
    boot = normal_np(key(9), N).astype(np.float32)
    valid = (done[last] == 0).astype(np.uint8)
    boot = np.where(valid == 1, boot, 0.0).astype(np.float32)
    # env-major arrays -> arrival order: env-major index of arrival record i
    em = starts[env] + rk
    recs = StepRecords(
        env_index=env.astype(np.int32), obs=obs[em], log_prob=logp[em], value=value[em],
        reward=reward[em], done=done[em], act_disc=act[em], act_cont=None,
        episode_index=ep_idx[em].astype(np.int64), step_in_episode=step_in_ep[em].astype(np.int32),
        latency=tau[env].astype(np.float32),
        h_before=hb[em], h_before_valid=np.ones(S, np.uint8),
        snapshot_version=np.ones(S, np.uint64))
    return Workload(T, N, obs_dim, num_actions, hidden_dim, recs, counts, tau, boot, valid)


def fill_buffer(buf, wl: Workload, snapshot_version: int = 1):
    """begin_rollout + append all records + bootstraps on a RolloutBuffer-like object."""
    buf.begin_rollout(snapshot_version)
    out = buf.append_steps(wl.records)
    envs = np.flatnonzero(wl.bootstrap_valid)
    if hasattr(buf, "set_bootstraps"):
        buf.set_bootstraps(envs, np.asarray(wl.bootstrap, np.float32)[envs])
    else:
        for e in envs:
            buf.set_bootstrap(int(e), float(wl.bootstrap[e]))
    return out


def ragged_lengths(total: int, seed: int = 1, mu: float = 3.0, sigma: float = 1.5,
                   max_len: int = 1024) -> np.ndarray:
    """C5 stress lengths: clamp(round(lognormal(mu, sigma)), 1, max_len) until the sum >= total."""
    key = CounterRng(seed).stream(11).key
    n_guess = max(16, int(total / 40) + 16)
    out = []
    acc = 0
    start = 0
    while acc < total:
        z = normal_np(key, n_guess, start=2 * start)
        start += n_guess
        L = np.clip(np.rint(np.exp(mu + sigma * z)), 1, max_len).astype(np.int64)
        cs = np.cumsum(L)
        if acc + cs[-1] >= total:
            k = int(np.searchsorted(cs, total - acc))
            L = L[:k + 1].copy()
            L[-1] -= (acc + int(L.sum())) - total
            out.append(L)
            acc = total
        else:
            out.append(L)
            acc += int(cs[-1])
    lens = np.concatenate(out)
    return lens[lens > 0]
