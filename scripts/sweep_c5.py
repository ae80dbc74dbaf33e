"""C5 sweep: GAE + gather on the heavy-tailed ragged view at
S = 2^20 .. 2^28 (or the sizes given), device-synthesized.  One JSON line per
size: kernel and call times, algorithmic GB/s (17 B/step GAE + 9 B/env,
8D+36 B/step gather), fraction of the measured HBM peak, and the CPU GAE
baseline on the box's host (one thread): the reference's O(N S) loop
(learner.cpp:11-41) where it finishes within the cap (S <= 2^20), the O(S)
restatement at every size; the GPU advantages are checked against the O(S)
restatement (|gpu - cpu| <= 1e-5 max(1, |cpu|)).

  python scripts/sweep_c5.py [log2 sizes...] [--no-cpu]"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
args = [a for a in sys.argv[1:] if not a.startswith("--")]
sizes = [int(a) for a in args] or [20, 22, 24, 26, 28]
cpu = "--no-cpu" not in sys.argv
D = 2
G, LAM = 0.99, 0.95
for lg in sizes:
    S = 1 << lg
    lens = synth.ragged_lengths(S, seed=11)
    view = V.view_synth(lens, obs_dim=D, hidden_dim=4, seed=12)
    g_call, t_call, g_k, t_k = V.bench_gae_gather(view, B=2, seed=13, reps=10, gamma=G, lam=LAM, kernels=True)
    gb = 17.0 * S + 9.0 * len(lens)
    tb = (8.0 * D + 36.0) * S
    line = {"log2_steps": lg, "envs": len(lens), "gae_ms": g_k, "gather_ms": t_k,
            "gae_call_ms": g_call, "gather_call_ms": t_call,
            "gae_gbs": gb / g_k / 1e6, "gather_gbs": tb / t_k / 1e6,
            "gae_gather_gbs": (gb + tb) / (g_k + t_k) / 1e6,
            "gae_frac": gb / g_k / 1e6 / peak, "gather_frac": tb / t_k / 1e6 / peak,
            "gae_gather_frac": (gb + tb) / (g_k + t_k) / 1e6 / peak}
    if cpu:
        from oracle import oracle as O  # CPU baseline leg only
        f = view.fields("reward", "value", "done", "env_index", "replayed", "env_bootstrap", "env_bootstrap_valid",
                        "advantage")
        argv = (f["reward"], f["value"], f["done"], f["env_index"], f["replayed"], len(lens), f["env_bootstrap"],
                f["env_bootstrap_valid"], G, LAM)
        t0 = time.perf_counter()
        a_cpu, _ = O.gae_arrays(*argv, reference_loop=False)
        line["cpu_gae_os_ms"] = 1000 * (time.perf_counter() - t0)
        if lg <= 20:
            t0 = time.perf_counter()
            O.gae_arrays(*argv, reference_loop=True)
            line["cpu_gae_reference_loop_ms"] = 1000 * (time.perf_counter() - t0)
        err = np.abs(f["advantage"].astype(np.float64) - a_cpu) / np.maximum(1.0, np.abs(a_cpu.astype(np.float64)))
        line["gpu_vs_cpu_max_scaled_err"] = float(err.max())
        line["cpu_cores"] = 1
        del f, a_cpu
    print(json.dumps(line), flush=True)
    del view
