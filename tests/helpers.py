"""Shared fixtures mirroring the reference's tests/test_helpers.hpp and record builders."""
from __future__ import annotations

import numpy as np

from paper_2210_05064_b200.api import StepRecords
from paper_2210_05064_b200.hostview import make_view, random_lengths  # noqa: F401


def rec(env, episode, t, done, reward=0.0, hidden=3, obs_dim=2):
    """test_rollout.cpp:25-40: obs = (env, t), action t % 2, log_prob -0.5,
    value 0.1 t, h_before = 0.01 env."""
    return dict(env=env, episode=episode, t=t, done=done, reward=reward, hidden=hidden,
                obs_dim=obs_dim)


def records(rs: list[dict]) -> StepRecords:
    n = len(rs)
    H = rs[0]["hidden"] if rs else 3
    D = rs[0]["obs_dim"] if rs else 2
    obs = np.zeros((n, D))
    for i, r in enumerate(rs):
        obs[i, 0] = r["env"]
        if D > 1:
            obs[i, 1] = r["t"]
    return StepRecords(
        env_index=np.array([r["env"] for r in rs], np.int32),
        obs=obs,
        log_prob=np.full(n, -0.5),
        value=np.array([0.1 * r["t"] for r in rs]),
        reward=np.array([r["reward"] for r in rs]),
        done=np.array([1 if r["done"] else 0 for r in rs], np.uint8),
        act_disc=np.array([r["t"] % 2 for r in rs], np.int32),
        episode_index=np.array([r["episode"] for r in rs], np.int64),
        step_in_episode=np.array([r["t"] for r in rs], np.int32),
        latency=np.zeros(n),
        h_before=np.array([[0.01 * r["env"]] * H for r in rs]).reshape(n, H),
        h_before_valid=np.ones(n, np.uint8),
        snapshot_version=np.ones(n, np.uint64))
