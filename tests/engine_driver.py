"""Scripted collection stream for the inference-engine tests (device engine vs
the oracle engine, oracle/engine.py): N envs arrive in a seeded random order
and subset per tick; episode lengths, observations and rewards are pure
functions of (env, episode, step), so both engines see identical requests as
long as they dispatch the same envs."""
import numpy as np


def ep_len(e: int, ep: int) -> int:
    return 3 + (7 * e + 13 * ep) % 17


def obs_of(e: int, ep: int, t: int, D: int) -> np.ndarray:
    k = np.arange(D)
    return (np.sin(0.7 * e + 0.31 * t + 1.3 * ep + 0.9 * k) * (1.0 + 0.1 * k)).astype(np.float32)


def reward_of(e: int, ep: int, t: int) -> float:
    return float(np.float32(np.cos(0.37 * e + 0.11 * t - 0.5 * ep)))


class Driver:
    """Env-side state: per env (episode, step, first?); envs with an outstanding
    action step on the next tick when chosen; envs the engine parked wait for
    begin_rollout's dispatch."""

    def __init__(self, N: int, D: int, seed: int):
        self.N, self.D = N, D
        self.rng = np.random.default_rng(seed)
        self.ep = np.zeros(N, np.int64)
        self.t = np.zeros(N, np.int32)
        self.first = np.ones(N, bool)
        self.has_action = np.zeros(N, bool)
        self.parked = np.zeros(N, bool)

    def requests(self, make, p: float = 0.6):
        """One tick: a random subset of the non-parked envs, in random order."""
        order = self.rng.permutation(self.N)
        pick = [int(e) for e in order if not self.parked[e] and self.rng.random() < p]
        reqs = []
        for e in pick:
            if self.first[e]:
                reqs.append(make(env_index=e, observation=obs_of(e, self.ep[e], self.t[e], self.D), first=True,
                                 obs_episode=int(self.ep[e]), obs_step=int(self.t[e])))
                continue
            if not self.has_action[e]:
                continue
            r = reward_of(e, self.ep[e], self.t[e])
            done = self.t[e] + 1 >= ep_len(e, self.ep[e])
            if done:
                self.ep[e] += 1
                self.t[e] = 0
            else:
                self.t[e] += 1
            reqs.append(make(env_index=e, observation=obs_of(e, self.ep[e], self.t[e], self.D), reward=r,
                             done=bool(done), latency=0.01 * (e % 5), obs_episode=int(self.ep[e]),
                             obs_step=int(self.t[e])))
        return reqs

    def after(self, reqs, dispatched_envs):
        got = set(dispatched_envs)
        for q in reqs:
            e = q.env_index
            self.first[e] = False
            self.has_action[e] = e in got
            self.parked[e] = e not in got

    def unpark(self, dispatched_envs):
        for e in dispatched_envs:
            self.parked[e] = False
            self.has_action[e] = True
