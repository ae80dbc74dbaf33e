"""Localise a forward-parity gap: ver_forward_packed vs the oracle per packed
row on one minibatch of the C2/C3-scale workload; prints the worst rows per
timestep range."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import paper_2210_05064_b200 as V
from oracle import oracle as O
from paper_2210_05064_b200 import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
T, H = 128, 512
O.set_threads(16)
O.set_sparse_rows(True)
cfg = V.ModelConfig(obs_dim=2, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
p = O.params_init(cfg, O.mix(1, 0x9A9A)).astype(np.float32).astype(np.float64)
wl = synth.make_workload(T, N, hidden_dim=H, seed=1)
o = O.Rollout(T, N, 1, 0, 2, 0, H)
synth.fill_buffer(o, wl)
vo = o.close_rollout()
hv = vo.to_host()
seed = O.mix(O.mix(O.mix(1, 0xF00D), 0), 0)
seqs, tot = O.split_minibatches(vo, 2, seed).groups()[0]
bo = O.pack(seqs)
s = bo.slots
obs = hv.obs[s].astype(np.float32)
act = hv.act_disc[s]
h0 = np.stack([hv.h0[q[4]] for q in bo.seqs]).astype(np.float32)
lg, eg, vg = V.forward_packed(cfg, p, obs, act, None, bo.batch_sizes, bo.offsets, h0)
lo, eo, vv = O.forward_packed(cfg, p, obs, act, None, bo.batch_sizes, bo.offsets, h0)
print("rows", s.size, "L", bo.max_len, "bs[0..4]", bo.batch_sizes[:5], "bs[-5:]", bo.batch_sizes[-5:])
for name, a, b in (("logp", lg, lo), ("ent", eg, eo), ("value", vg, vv)):
    err = np.abs(a - b) / np.maximum(1, np.abs(b))
    t_of = np.searchsorted(bo.offsets, np.arange(s.size), side="right") - 1
    worst = np.argsort(-err)[:8]
    print(name, "max", err.max(), "mean", err.mean(), "worst rows", [(int(i), int(t_of[i]), float(err[i])) for i in worst])
    # per-timestep max error profile
    prof = np.zeros(bo.max_len)
    np.maximum.at(prof, t_of, err)
    bad = np.flatnonzero(prof > 1e-6)
    print("  steps with err > 1e-6:", bad[:20], "... count", bad.size, "bs there", bo.batch_sizes[bad[:10]])
