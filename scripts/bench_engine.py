"""Device inference engine throughput: N envs, every env
requests each batch (one env step per batch), E = H = 512, D = 2, A = 2
discrete; one process_batch = H2D of the requests, act + sampling on the GPU,
D2H of the actions, host protocol bookkeeping, store appends.
  python scripts/bench_engine.py [N] [batches]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V  # noqa: E402


def run(N=4096, batches=40, E=512, H=512, T=128):
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=2)
    rng = np.random.default_rng(0)
    p = (rng.standard_normal(V.param_count(cfg)) * 0.05).astype(np.float32)
    g = V.InferenceEngine(cfg, T, N, p, version=1, mode=V.VARIABLE, seed=1)
    g.begin_rollout()
    env = np.arange(N, dtype=np.int32)
    step = np.zeros(N, np.int32)
    ep = np.zeros(N, np.int64)
    obs = rng.standard_normal((N, 2)).astype(np.float32)
    g.process_arrays(env, obs, first=np.ones(N, np.uint8), obs_episode=ep, obs_step=step)
    times = []
    for b in range(batches):
        step += 1
        obs = rng.standard_normal((N, 2)).astype(np.float32)
        t0 = time.perf_counter()
        r, de, act = g.process_arrays(env, obs, reward=np.ones(N, np.float32), done=np.zeros(N, np.uint8),
                                      obs_episode=ep, obs_step=step)
        times.append(time.perf_counter() - t0)
        if g.rollout_done():
            g.close()
            g.begin_rollout()
    ms = 1000 * float(np.median(times[3:]))
    return {"envs": N, "E": E, "H": H, "ms_per_batch": ms, "actions_per_s": N / (ms / 1000.0)}


if __name__ == "__main__":
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    print(json.dumps(run(N, nb)))
