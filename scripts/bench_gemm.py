"""Device time of the learner's GEMM shapes at C2 (S_mb = 16384, E = H = 512)
through the library GEMM: 3xTF32 tcgen05 (engine 1), 1xTF32 (engine 2), SIMT (0)."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V

S, E, H3 = 16384, 512, 1536
SHAPES = [  # name, M, N, K, transA, transB, splitk
    ("enc2 fwd", S, E, E, False, False, 1),
    ("xp fwd", S, H3, E, False, False, 1),
    ("dpre2 = dpre Wx^T", S, E, H3, False, True, 1),
    ("dpre1 = dpre2 W2^T", S, E, E, False, True, 1),
    ("dUx = hprev^T dhu", E, H3, S, True, False, 8),
    ("dW2 = e1^T dpre2", E, E, S, True, False, 8),
]
out = []
for name, M, N, K, ta, tb, sk in SHAPES:
    row = {"gemm": name, "M": M, "N": N, "K": K}
    for eng in (1, 2, 0):
        ms = V.debug_gemm_time(M, N, K, ta, tb, engine=eng, splitk=sk, reps=10)
        row[f"ms_e{eng}"] = round(ms, 4)
        row[f"tflops_e{eng}"] = round(2.0 * M * N * K / ms / 1e9, 1)
    out.append(row)
    print(json.dumps(row), flush=True)
