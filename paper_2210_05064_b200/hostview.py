"""Host-side image of a RolloutView (rollout.hpp:33-78) as numpy arrays.

Used to build fixtures (the reference tests' ``make_view``, test_helpers.hpp:13-67),
to upload arbitrary views to the device and to read views back.  ``fdtype``
is float32 for the B200 library and float64 for the CPU oracle.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEQ_FIELDS = ("seq_id", "env_index", "length", "start_offset", "h0_index", "stale",
              "parent_start_offset", "skip")


@dataclass
class HostView:
    T: int
    N: int
    action_kind: int  # 0 discrete, 1 continuous
    obs_dim: int
    act_dim: int
    hidden_dim: int
    obs: np.ndarray
    act_disc: np.ndarray
    act_cont: np.ndarray
    log_prob: np.ndarray
    value: np.ndarray
    reward: np.ndarray
    latency: np.ndarray
    advantage: np.ndarray
    returns: np.ndarray
    done: np.ndarray
    stale: np.ndarray
    replayed: np.ndarray
    env_index: np.ndarray
    seq_of_slot: np.ndarray
    step_in_episode: np.ndarray
    episode_index: np.ndarray
    version: np.ndarray
    seqs: np.ndarray  # K x 8 int32
    h0: np.ndarray    # rows x H
    per_env_counts: np.ndarray
    env_bootstrap: np.ndarray
    env_bootstrap_valid: np.ndarray
    deficit: int = 0
    stale_steps: int = 0
    replayed_steps: int = 0
    snapshot_version: int = 0
    collect_wall_time: float = 0.0

    @property
    def size(self) -> int:
        return int(self.done.shape[0])

    @property
    def num_seqs(self) -> int:
        return int(self.seqs.shape[0])

    def fresh_steps(self) -> int:
        return self.size - self.replayed_steps

    @staticmethod
    def empty(T, N, action_kind, obs_dim, act_dim, hidden_dim, S, K, h0_rows=None,
              fdtype=np.float32) -> "HostView":
        h0_rows = K if h0_rows is None else h0_rows
        f = fdtype
        return HostView(
            T=T, N=N, action_kind=action_kind, obs_dim=obs_dim, act_dim=act_dim,
            hidden_dim=hidden_dim,
            obs=np.zeros((S, obs_dim), f),
            act_disc=np.zeros(S if action_kind == 0 else 0, np.int32),
            act_cont=np.zeros((S if action_kind == 1 else 0, max(act_dim, 1)), f),
            log_prob=np.zeros(S, f), value=np.zeros(S, f), reward=np.zeros(S, f),
            latency=np.zeros(S, f), advantage=np.zeros(S, f), returns=np.zeros(S, f),
            done=np.zeros(S, np.uint8), stale=np.zeros(S, np.uint8),
            replayed=np.zeros(S, np.uint8), env_index=np.zeros(S, np.int32),
            seq_of_slot=np.zeros(S, np.int32), step_in_episode=np.zeros(S, np.int32),
            episode_index=np.zeros(S, np.int64), version=np.zeros(S, np.uint64),
            seqs=np.zeros((K, 8), np.int32), h0=np.zeros((h0_rows, hidden_dim), f),
            per_env_counts=np.zeros(N, np.int32), env_bootstrap=np.zeros(N, f),
            env_bootstrap_valid=np.zeros(N, np.uint8))

    def astype(self, fdtype) -> "HostView":
        d = {k: getattr(self, k) for k in self.__dataclass_fields__}
        for k in ("obs", "act_cont", "log_prob", "value", "reward", "latency", "advantage",
                  "returns", "h0", "env_bootstrap"):
            d[k] = np.ascontiguousarray(d[k], dtype=fdtype)
        for k in d:
            if isinstance(d[k], np.ndarray):
                d[k] = np.ascontiguousarray(d[k]).copy()
        return HostView(**d)

    def copy(self) -> "HostView":
        return self.astype(self.obs.dtype)


def make_view(lengths, obs_dim=2, hidden_dim=4, T=0, N=0, fdtype=np.float64) -> HostView:
    """The reference tests' synthetic closed view (test_helpers.hpp:13-67).

    One sequence per length, env = seq % N, done at each sequence end,
    obs[i, 0] = global slot index, obs[i, 1] = t, h0[s, 0] = 0.1 * s.
    """
    total = int(sum(lengths))
    T = T if T > 0 else total
    N = N if N > 0 else 1
    v = HostView.empty(T, N, 0, obs_dim, 0, hidden_dim, total, len(lengths), fdtype=fdtype)
    v.version[:] = 1
    off = 0
    for s, L in enumerate(lengths):
        env = s % N
        v.seqs[s] = (s, env, L, off, s, 0, off, 0)
        v.h0[s, 0] = 0.1 * s
        for t in range(L):
            v.obs[off, 0] = off
            if obs_dim > 1:
                v.obs[off, 1] = t
            v.act_disc[off] = off % 2
            v.env_index[off] = env
            v.seq_of_slot[off] = s
            v.step_in_episode[off] = t
            v.done[off] = 1 if t == L - 1 else 0
            off += 1
    return v


def random_lengths(total: int, max_len: int, rng) -> list[int]:
    """test_helpers.hpp:70-80 with a CounterRng-like object (uniform_int)."""
    out = []
    left = total
    while left > 0:
        L = 1 + int(rng.uniform_int(max_len))
        L = min(L, left)
        out.append(L)
        left -= L
    return out
