"""C5 sweep: GAE + gather on the heavy-tailed ragged view at
S = 2^20 .. 2^28 (or the sizes given), device-synthesized.  One JSON line per
size: call and kernel times, algorithmic GB/s (17 B/step GAE + 9 B/env,
8D+36 B/step gather), fraction of the measured HBM peak."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
sizes = [int(a) for a in sys.argv[1:]] or [20, 22, 24, 26, 28]
D = 2
for lg in sizes:
    S = 1 << lg
    lens = synth.ragged_lengths(S, seed=11)
    view = V.view_synth(lens, obs_dim=D, hidden_dim=4, seed=12)
    g_call, t_call, g_k, t_k = V.bench_gae_gather(view, B=2, seed=13, reps=10, kernels=True)
    gb = 17.0 * S + 9.0 * len(lens)
    tb = (8.0 * D + 36.0) * S
    print(json.dumps({"log2_steps": lg, "envs": len(lens), "gae_ms": g_k, "gather_ms": t_k,
                      "gae_call_ms": g_call, "gather_call_ms": t_call,
                      "gae_gbs": gb / g_k / 1e6, "gather_gbs": tb / t_k / 1e6,
                      "gae_gather_gbs": (gb + tb) / (g_k + t_k) / 1e6,
                      "gae_frac": gb / g_k / 1e6 / peak, "gather_frac": tb / t_k / 1e6 / peak,
                      "gae_gather_frac": (gb + tb) / (g_k + t_k) / 1e6 / peak}), flush=True)
    del view
