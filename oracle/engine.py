"""CPU restatement of the reference's collection-side inference engine.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of the device
InferenceEngine (paper_2210_05064_b200/csrc/engine.cu), never as a product path.

Restates, in double precision:
* the counter RNG (include/ver/rng.hpp:16-73): splitmix64, mix, CounterRng
  streams, uniform = (u >> 11) * 2^-53, Box-Muller normal;
* action sampling (src/nn.cpp:134-183): sample_categorical, sample_gaussian,
  gaussian_log_prob (categorical_log_prob is the C++ oracle's);
* InferenceEngine (src/runtime.cpp:60-229, include/ver/runtime.hpp:96-160):
  begin_rollout, process_batch, complete_pending, compute_actions,
  finalize_bootstraps, close, over the oracle's act (vo_act, nn.cpp:118-126)
  and rollout store (vo_rollout_*, rollout.cpp).

Parity pin: mix() is checked against the C++ oracle's rng::mix, and the RNG and
sampler against the reference's property tests (test_rng.cpp, test_nn.cpp:
237-278), in tests/test_oracle_engine.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import oracle as O

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:  # rng.hpp:16-21
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix(a: int, b: int) -> int:  # rng.hpp:23-25
    return splitmix64(a ^ ((0x9E3779B97F4A7C15 + ((b << 6) & M64) + (b >> 2) + splitmix64(b)) & M64))


class CounterRng:  # rng.hpp:30-73
    def __init__(self, seed: int | None = None):
        self.key = 0 if seed is None else splitmix64(seed & M64)
        self.counter = 0

    def stream(self, *ids: int) -> "CounterRng":
        r = CounterRng()
        k = self.key
        for i in ids:
            k = mix(k, i & M64)
        r.key = k
        return r

    def next_u64(self) -> int:
        v = mix(self.key, self.counter)
        self.counter += 1
        return v

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 <= 0:
            u1 = 2.0 ** -53
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def sample_categorical(logits, rng: CounterRng) -> tuple[int, float]:
    """nn.cpp:134-146; also returns the draw's distance to the nearest
    cumulative boundary (how far a perturbed logit may move before the
    sampled index changes)."""
    z = np.asarray(logits, np.float64)
    p = np.exp(z - z.max())
    p = p / p.sum()
    u = rng.uniform()
    acc = 0.0
    margin = math.inf
    pick = len(p) - 1
    for i in range(len(p)):
        acc += p[i]
        margin = min(margin, abs(u - acc))
        if u < acc:
            pick = i
            break
    return pick, margin


def sample_gaussian(mean, log_std, rng: CounterRng) -> np.ndarray:  # nn.cpp:167-173
    return np.array([mean[i] + math.exp(log_std[i]) * rng.normal() for i in range(len(mean))])


def gaussian_log_prob(mean, log_std, a) -> float:  # nn.cpp:175-183
    lp = -0.5 * math.log(2.0 * math.pi) * len(mean)
    for i in range(len(mean)):
        s = math.exp(log_std[i])
        z = (a[i] - mean[i]) / s
        lp += -0.5 * z * z - log_std[i]
    return lp


@dataclass
class Request:  # runtime.hpp:30-42
    env_index: int
    observation: np.ndarray
    reward: float = 0.0
    done: bool = False
    first: bool = False
    latency: float = 0.0
    obs_episode: int = 0
    obs_step: int = 0


@dataclass
class _Pending:  # runtime.hpp:135-144
    obs: np.ndarray
    action: object
    log_prob: float
    value: float
    h_before: np.ndarray
    episode: int
    t: int
    version: int


@dataclass
class _Slot:  # runtime.hpp:145-150
    h: np.ndarray
    pending: _Pending | None = None
    parked: Request | None = None
    paused: bool = False


@dataclass
class _Records:  # one EnvStepRecord in the oracle store's append_steps layout
    env_index: np.ndarray
    episode_index: np.ndarray
    step_in_episode: np.ndarray
    obs: np.ndarray
    act_disc: np.ndarray | None
    act_cont: np.ndarray | None
    log_prob: np.ndarray
    value: np.ndarray
    reward: np.ndarray
    done: np.ndarray
    latency: np.ndarray
    h_before: np.ndarray
    h_before_valid: np.ndarray | None = None
    snapshot_version: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))

    def __len__(self):
        return 1


@dataclass
class Result:  # runtime.hpp:102-106
    dispatches: list
    new_commits: int = 0
    closed_now: bool = False
    margins: dict = field(default_factory=dict)  # env -> categorical boundary margin of its draw


class Engine:
    """InferenceEngine (runtime.cpp:76-234) over the oracle's act and store."""

    def __init__(self, cfg, T: int, N: int, params, version: int = 0, mode: int = 1, seed: int = 0):
        self.cfg = cfg
        self.N = N
        self.cont = cfg.action_kind == 1
        self.A = cfg.act_dim if self.cont else cfg.num_actions
        self.params = np.asarray(params, np.float64)
        self.version = version
        self.seed = seed
        self.mode = mode
        self.T = T
        self.buf = O.Rollout(T, N, mode, cfg.action_kind, cfg.obs_dim, self.A if self.cont else 0, cfg.hidden_dim)
        self.envs = [_Slot(np.zeros(cfg.hidden_dim)) for _ in range(N)]
        # committed steps per env for the Fixed-mode cap (rollout.hpp:113-117); the oracle
        # store does not expose its counts, and carryovers (committed by begin_rollout)
        # exist only in Variable mode, where caps do not apply
        self.counts = np.zeros(N, np.int64)
        self.bootstrap_set = np.zeros(N, bool)

    # store state helpers (rollout.hpp:109-119)
    def _open(self) -> bool:
        return bool(self.buf.state()[0])

    def _at_cap(self, e: int) -> bool:
        return self.mode == 0 and self.counts[e] >= self.T

    def set_snapshot(self, params, version: int):  # runtime.cpp:82
        self.params = np.asarray(params, np.float64)
        self.version = version

    def begin_rollout(self) -> Result:  # runtime.cpp:84-113
        out = Result([])
        self.buf.begin_rollout(self.version)
        self.counts[:] = 0
        self.bootstrap_set[:] = False
        out.new_commits = self.buf.state()[1]  # consumed carryover
        for es in self.envs:
            es.paused = False
        parked = []
        for es in self.envs:
            if es.parked is not None:
                parked.append(es.parked)
                es.parked = None
        needs = []
        for req in parked:
            if self._open() and not self._at_cap(req.env_index):
                needs.append(req)
            else:
                self.envs[req.env_index].parked = req
        self._compute_actions(needs, out)
        if not self._open():
            out.closed_now = True
        return out

    def _complete_pending(self, req: Request, out: Result):  # runtime.cpp:116-147
        es = self.envs[req.env_index]
        if es.pending is None:
            raise O.OracleProtocolError(
                f"inference: completion for env {req.env_index} without an outstanding action")
        p = es.pending
        es.pending = None
        rec = _Records(
            env_index=np.array([req.env_index], np.int32), episode_index=np.array([p.episode], np.int64),
            step_in_episode=np.array([p.t], np.int32), obs=p.obs.reshape(1, -1),
            act_disc=None if self.cont else np.array([p.action], np.int32),
            act_cont=np.asarray(p.action, np.float64).reshape(1, -1) if self.cont else None,
            log_prob=np.array([p.log_prob]), value=np.array([p.value]), reward=np.array([req.reward]),
            done=np.array([1 if req.done else 0], np.uint8), latency=np.array([req.latency]),
            h_before=p.h_before.reshape(1, -1), snapshot_version=np.array([p.version], np.uint64))
        oc = int(self.buf.append_steps(rec)[0])
        if oc == 0:
            self.counts[req.env_index] += 1
            out.new_commits += 1
            if not self._open():
                out.closed_now = True
        elif p.t > 0:
            self.buf.set_bootstrap(req.env_index, p.value)
            self.bootstrap_set[req.env_index] = True

    def process_batch(self, reqs) -> Result:  # runtime.cpp:192-215
        out = Result([])
        needs = []
        for req in reqs:
            es = self.envs[req.env_index]
            if es.parked is not None:
                raise O.OracleProtocolError(f"inference: request for env {req.env_index} which is already parked")
            if not req.first:
                self._complete_pending(req, out)
            if req.done:
                es.h = np.zeros_like(es.h)
            capped = self.mode == 0 and self._at_cap(req.env_index)
            if self._open() and not capped:
                needs.append(req)
            else:
                es.parked = req
                if capped:
                    es.paused = True
        self._compute_actions(needs, out)
        return out

    def _compute_actions(self, needs, out: Result):  # runtime.cpp:149-190
        if not needs:
            return
        obs = np.stack([np.asarray(r.observation, np.float64).reshape(-1) for r in needs])
        h = np.stack([self.envs[r.env_index].h for r in needs])
        dist, value, h_new = O.act(self.cfg, self.params, obs, h)
        log_std = self.params[-self.A:] if self.cont else None
        for i, req in enumerate(needs):
            es = self.envs[req.env_index]
            rng = CounterRng(self.seed).stream(0xAC7101, req.env_index).stream(req.obs_episode, req.obs_step)
            if not self.cont:
                a, margin = sample_categorical(dist[i], rng)
                lp = O.categorical_log_prob(dist[i], a)
                out.margins[req.env_index] = margin
            else:
                a = sample_gaussian(dist[i], log_std, rng)
                lp = gaussian_log_prob(dist[i], log_std, a)
            es.pending = _Pending(obs[i].copy(), a, lp, float(value[i]), es.h.copy(), req.obs_episode,
                                  req.obs_step, self.version)
            out.dispatches.append((req.env_index, a))
            es.h = h_new[i].copy()

    def finalize_bootstraps(self):  # runtime.cpp:217-229
        for e in range(self.N):
            es = self.envs[e]
            if self.bootstrap_set[e]:
                continue
            if es.pending is not None:
                if es.pending.t > 0:
                    self.buf.set_bootstrap(e, es.pending.value)
                    self.bootstrap_set[e] = True
            elif es.parked is not None and es.parked.obs_step > 0:
                obs = np.asarray(es.parked.observation, np.float64).reshape(1, -1)
                _, v, _ = O.act(self.cfg, self.params, obs, es.h.reshape(1, -1))
                self.buf.set_bootstrap(e, float(v[0]))
                self.bootstrap_set[e] = True

    def force_close(self):
        self.buf.force_close()

    def close(self):  # runtime.cpp:231-234
        return self.buf.close_rollout()
