"""GAE + gather on the device-generated ragged view (C5 point) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 26
lens = synth.ragged_lengths(1 << log2, seed=11)
view = V.view_synth(lens, obs_dim=2, hidden_dim=4, seed=12)
print(V.bench_gae_gather(view, B=2, seed=13, reps=1))
