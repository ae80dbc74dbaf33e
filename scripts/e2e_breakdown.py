"""Where the end-to-end C3 step's host time goes: append (host protocol + staging),
close_rollout (H2D + compaction), update, stats read.  python scripts/e2e_breakdown.py"""
import statistics
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = V.ModelConfig(obs_dim=2, encoder_dim=512, hidden_dim=512, action_kind=0, num_actions=2)
wl = synth.make_workload(128, N, hidden_dim=512, seed=1)
L = V.Learner(cfg, V.params_init(cfg, mix(1, 0x9A9A)), V.PPOConfig(epochs=3, minibatches=2), V.EntropyController(),
              V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D))
buf = V.RolloutBuffer(128, N, V.VARIABLE, 0, 2, 0, 512, ctx=L.ctx)
rows = []
for i in range(6):
    t0 = time.perf_counter()
    buf.begin_rollout(2 + i)
    buf.append_steps(wl.records)
    t1 = time.perf_counter()
    import numpy as np
    envs = np.flatnonzero(wl.bootstrap_valid)
    buf.set_bootstraps(envs, np.asarray(wl.bootstrap, np.float32)[envs])
    t2 = time.perf_counter()
    v = buf.close_rollout()
    L.ctx.synchronize()
    t3 = time.perf_counter()
    st = L.update(v)
    t4 = time.perf_counter()
    dev = sum(x for k, x in L.last_timing().items() if k in ("gae", "replay", "forward", "loss", "backward", "adam"))
    rows.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), dev, 1e3 * (t4 - t0)))
    del v
for r in rows[2:]:
    print("append %.2f  bootstraps %.2f  close %.2f  update(wall) %.2f  update(device phases) %.2f  total %.2f ms" % r)
