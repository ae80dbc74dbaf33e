"""GAE / gather device time at the C5 point for a list of L2-prefetch distances (env knobs)."""
import json, os, subprocess, sys
log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 26
code = f"""
import sys; sys.path.insert(0, '.')
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
lens = synth.ragged_lengths(1 << {log2}, seed=11)
v = V.view_synth(lens, obs_dim=2, hidden_dim=4, seed=12)
g, t = V.bench_gae_gather(v, B=2, seed=13, reps=5)
S = 1 << {log2}
print(g, t, 17 * S / g / 1e6, 52 * S / t / 1e6)
"""
for gpf in (0, 296, 592, 1184):
    for tpf in (0, 148, 296, 592):
        if gpf and tpf and (gpf, tpf) not in ((592, 296), (1184, 592), (296, 148)):
            continue
        env = dict(os.environ, VER_GAE_PF=str(gpf), VER_GATHER_PF=str(tpf))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.split()
        print(json.dumps({"gae_pf": gpf, "gather_pf": tpf, "gae_ms": float(out[0]), "gather_ms": float(out[1]),
                          "gae_gbs": round(float(out[2])), "gather_gbs": round(float(out[3]))}), flush=True)
