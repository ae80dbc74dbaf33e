"""Wait-cycle breakdown of the tcgen05 GEMM roles (ver_debug_gemm_prof) for the
learner's GEMMs at C3 (S_mb = 262,144) and one full C3 update, per env setting."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2210_05064_b200 as V

S, E, H3 = 262144, 512, 1536
SHAPES = [("xp fwd", S, H3, E, False, False, 1), ("enc2 fwd", S, E, E, False, False, 1),
          ("dX = dpre Wx^T", S, E, H3, False, True, 1), ("dX2", S, E, E, False, True, 1),
          ("dU = hprev^T dhu", E, H3, S, True, False, 3), ("xp fwd, L2-resident A", 8192, H3, E, False, False, 1),
          ("xp fwd, M=32768", 32768, H3, E, False, False, 1)]
NAMES = ["mma_wait_acc", "mma_wait_split", "mma_total", "split_wait_full", "split_wait_aslot",
         "epi_wait_acc", "epi_final", "tma_wait_empty", "stages", "drains"]
for name, M, N, K, ta, tb, sk in SHAPES:
    V.debug_gemm_time(M, N, K, ta, tb, engine=1, splitk=sk, reps=2)
    V.debug_gemm_prof(True)
    ms = V.debug_gemm_time(M, N, K, ta, tb, engine=1, splitk=sk, reps=3)
    p = V.debug_gemm_prof(False)
    tot = max(1, p[2])
    row = {"gemm": name, "ms": round(ms, 3), "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}
    row.update({k: round(p[i] / tot, 3) for i, k in enumerate(NAMES) if i not in (2, 8, 9)})
    row["stages"] = p[8]
    row["mma_cycles_per_stage"] = round(p[2] / max(1, p[8]), 1)
    row["drains"] = p[9]
    print(json.dumps(row), flush=True)
