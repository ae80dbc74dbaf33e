"""Print every PPO loss statistic and the gradient error per parameter tensor,
GPU vs oracle, for group 0 of epoch 0 at N envs (the test_gpu_parity_scale setup)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
import numpy as np
import paper_2210_05064_b200 as V
from oracle import oracle as O
from test_gpu_parity import close_both

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
T, H = 128, 512
O.set_threads(16)
O.set_sparse_rows(True)
cfg = V.ModelConfig(obs_dim=2, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
p = O.params_init(cfg, O.mix(1, 0x9A9A)).astype(np.float32).astype(np.float64)
vg, vo, _ = close_both(T, N, H, seed=1)
O.compute_gae(vo, 0.99, 0.95)
hv = vo.to_host().astype(np.float32).astype(np.float64)
vo2, vg2 = O.View.from_host(hv), V.RolloutView.from_host(hv)
lo = O.Learner(cfg, p, V.PPOConfig(), V.EntropyController(), 2.5e-4, 2_000_000, O.mix(1, 0xF00D))
seed = O.mix(O.mix(O.mix(1, 0xF00D), 0), 0)
seqs, tot = O.split_minibatches(vo2, 2, seed).groups()[0]
bo = O.pack(seqs)
bg = V.pack(vg2, V.SequenceGroup(seqs, tot))
ga = bg.gathered(2)
s = bo.slots
for f, src in (("obs", hv.obs), ("old_logp", hv.log_prob), ("adv", hv.advantage), ("ret", hv.returns)):
    d = np.abs(ga[f].astype(np.float64) - src[s].astype(np.float32).astype(np.float64)).max()
    print("gather", f, d)
h0 = lo.batch_h0(vo2, bo)
ro = O.ppo_loss(cfg, p, vo2, bo, V.PPOConfig(), 1e-3, h0, True)
rg = V.ppo_loss(cfg, p, vg2, bg, V.PPOConfig(), 1e-3, h0, True)
for k in ("loss", "policy_loss", "value_loss", "mean_entropy", "ratio_sum", "clip_count", "w_sum", "w_max", "steps"):
    print(k, getattr(rg, k), ro[k], getattr(rg, k) - ro[k])
err = np.abs(rg.grads - ro["grads"]) / np.maximum(1, np.abs(ro["grads"]))
for name, r, c_, off in V.param_tensors(cfg):
    n = r * c_
    e = err[off:off + n]
    print(f"grad {name:8s} max {e.max():.3e} at {int(np.argmax(e))} |g| max {np.abs(ro['grads'][off:off+n]).max():.3e}")
w = np.abs(rg.is_weights - ro["is_weights"])
print("isw max", w.max())
lg, eg, vgv = V.forward_packed(cfg, p, ga["obs"], ga["act_disc"], None, bo.batch_sizes, bo.offsets, h0)
lo_, eo, vv = O.forward_packed(cfg, p, ga["obs"], ga["act_disc"], None, bo.batch_sizes, bo.offsets, h0)
print("fwd value err", np.abs(vgv - vv).max(), "logp", np.abs(lg - lo_).max())
R = ga["ret"].astype(np.float64)
print("value loss from oracle fwd", 0.5 * np.mean((vv - R) ** 2), "from gpu fwd", 0.5 * np.mean((vgv.astype(np.float64) - R) ** 2))
