"""A/B of a library environment knob on B200: bit-identity of one minibatch's
loss + gradients between the settings, then the device time of full updates.

  python scripts/ab_env.py --N 4096 --epochs 3 VER_REC_FUSE=0 VER_REC_FUSE=1
Each positional argument is one setting: NAME=VALUE[,NAME=VALUE...]."""
import argparse
import os
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--T", type=int, default=128)
ap.add_argument("--H", type=int, default=512)
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--updates", type=int, default=4)
ap.add_argument("settings", nargs="+")
a = ap.parse_args()


def apply(setting):
    for kv in setting.split(","):
        k, v = kv.split("=", 1)
        if v == "":
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


cfg = V.ModelConfig(obs_dim=2, encoder_dim=a.H, hidden_dim=a.H, action_kind=0, num_actions=2)
wl = synth.make_workload(a.T, a.N, hidden_dim=a.H, seed=1)
buf = V.RolloutBuffer(a.T, a.N, V.VARIABLE, 0, 2, 0, a.H)
synth.fill_buffer(buf, wl)
view = buf.close_rollout()
p = V.params_init(cfg, mix(1, 0x9A9A))
V.compute_gae(view, 0.99, 0.95)
groups = V.split_minibatches(view, 2, 12345)
batch = V.pack(view, groups[0])
h0 = np.zeros((len(groups[0].seqs), a.H), np.float32)
ref = None
for s in a.settings:
    apply(s)
    r = V.ppo_loss(cfg, p, view, batch, V.PPOConfig(), 1e-3, h0, True)
    g = np.asarray(r.grads)
    if ref is None:
        ref = (r.loss, g)
        print(f"{s}: loss {r.loss!r}", flush=True)
    else:
        same = r.loss == ref[0] and np.array_equal(g, ref[1])
        d = float(np.max(np.abs(g - ref[1]))) if not same else 0.0
        print(f"{s}: loss {r.loss!r} bit-identical={same} max|dgrad|={d:.3e}", flush=True)
for s in a.settings:
    apply(s)
    L = V.Learner(cfg, p, V.PPOConfig(epochs=a.epochs, minibatches=2), V.EntropyController(),
                  V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D))
    L.update(view, read_stats=False)
    L.ctx.synchronize()
    tot, rf, rb, gf, gb = [], [], [], [], []
    for _ in range(a.updates):
        L.update(view, read_stats=False)
        L.ctx.synchronize()
        t = L.last_timing()
        tot.append(sum(v for k, v in t.items() if k in ("gae", "replay", "forward", "loss", "backward",
                                                         "allreduce", "adam")))
        rf.append(t["rec_fwd"])
        rb.append(t["rec_bwd"])
        gf.append(t["gemm_fwd"])
        gb.append(t["gemm_bwd"])
    print(f"{s}: phases {statistics.median(tot):.2f} ms  rec_fwd {statistics.median(rf):.2f}  "
          f"rec_bwd {statistics.median(rb):.2f}  gemm_fwd {statistics.median(gf):.2f}  "
          f"gemm_bwd {statistics.median(gb):.2f}  forward {t['forward']:.2f}", flush=True)
