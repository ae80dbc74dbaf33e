"""Small workloads over every production kernel family for compute-sanitizer
(memcheck / racecheck / synccheck):  python scripts/sanitize.py

  * close_rollout compaction, backfill, GAE (look-back scan), split / pack /
    tiled gather on a ragged view;
  * one learner update at E = H = 512 (tcgen05 GEMMs incl. CTA pairs, the
    persistent step kernel forced from 6 rows, K-split kernels, cluster tail,
    fused loss, Adam), and one with the CTA-pair step kernels from 6 rows and
    every forward pair step fused (gate epilogue + row-tile dataflow);
  * one C1-shaped update (H = 64: register recurrence kernels);
  * the inference engine (act + on-device sampling) for a few batches.
Prints one line per stage; any sanitizer report goes to its own output."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix


def update(H, T, N, epochs=1, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
    wl = synth.make_workload(T, N, hidden_dim=H, seed=5)
    buf = V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H)
    synth.fill_buffer(buf, wl)
    view = buf.close_rollout()
    L = V.Learner(cfg, V.params_init(cfg, mix(1, 0x9A9A)), V.PPOConfig(epochs=epochs, minibatches=2),
                  V.EntropyController(), V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D))
    st = L.update(view)
    print(f"update H={H} T={T} N={N}: loss {st.loss:.6f}", flush=True)
    return view


if "--pair-only" in sys.argv:  # just the fused CTA-pair update (for a full racecheck listing)
    update(512, 16, 48, env={"VER_REC_BIG_FWD": "6", "VER_REC_BIG_BWD": "6", "VER_REC_PAIR_ROWS": "6",
                             "VER_REC_FUSE_ALL": "1"})
    sys.exit(0)
v = update(512, 16, 24, env={"VER_REC_BIG_FWD": "6", "VER_REC_BIG_BWD": "6", "VER_REC_PAIR_ROWS": "200"})
# CTA-pair step kernels with the fused forward epilogue and row-tile dataflow
update(512, 16, 48, env={"VER_REC_BIG_FWD": "6", "VER_REC_BIG_BWD": "6", "VER_REC_PAIR_ROWS": "6",
                         "VER_REC_FUSE_ALL": "1"})
for k in ("VER_REC_BIG_FWD", "VER_REC_BIG_BWD", "VER_REC_PAIR_ROWS", "VER_REC_FUSE_ALL"):
    os.environ.pop(k, None)
update(64, 16, 16)
lens = synth.ragged_lengths(1 << 16, seed=3)
v5 = V.view_synth(lens, obs_dim=2, hidden_dim=4, seed=4)
V.compute_gae(v5, 0.99, 0.95)
for grp in V.split_minibatches(v5, 2, 7):
    p = V.pack(v5, grp)
print("gae / split / pack / gather on", int(lens.sum()), "ragged steps", flush=True)
cfg = V.ModelConfig(obs_dim=2, encoder_dim=512, hidden_dim=512, action_kind=0, num_actions=2)
eng = V.InferenceEngine(cfg, 8, 64, V.params_init(cfg, mix(1, 0x9A9A)), version=1, mode=V.VARIABLE, seed=3)
eng.begin_rollout()
rng = np.random.default_rng(0)
env = np.arange(64, dtype=np.int32)
st = np.zeros(64, np.int32)
ep = np.zeros(64, np.int64)
eng.process_arrays(env, rng.standard_normal((64, 2)).astype(np.float32), first=np.ones(64, np.uint8),
                   obs_episode=ep, obs_step=st)
for _ in range(3):
    st += 1
    eng.process_arrays(env, rng.standard_normal((64, 2)).astype(np.float32), reward=np.ones(64, np.float32),
                       done=np.zeros(64, np.uint8), obs_episode=ep, obs_step=st)
print("inference engine: 4 batches of 64 envs", flush=True)
