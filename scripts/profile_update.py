"""One C2-shaped learner update (after one warm-up update) for ncu launch lists."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=256)
ap.add_argument("--T", type=int, default=128)
ap.add_argument("--H", type=int, default=512)
ap.add_argument("--epochs", type=int, default=4)
ap.add_argument("--updates", type=int, default=2)
a = ap.parse_args()
cfg = V.ModelConfig(obs_dim=2, encoder_dim=a.H, hidden_dim=a.H, action_kind=0, num_actions=2)
wl = synth.make_workload(a.T, a.N, hidden_dim=a.H, seed=1)
buf = V.RolloutBuffer(a.T, a.N, V.VARIABLE, 0, 2, 0, a.H)
synth.fill_buffer(buf, wl)
view = buf.close_rollout()
L = V.Learner(cfg, V.params_init(cfg, mix(1, 0x9A9A)), V.PPOConfig(epochs=a.epochs, minibatches=2),
              V.EntropyController(), V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D))
for i in range(a.updates):
    st = L.update(view)
    print(i, L.ctx.launch_count(reset=True), L.last_timing(), flush=True)
