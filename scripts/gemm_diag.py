import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, paper_2210_05064_b200 as V
rng = np.random.default_rng(0)
out = {}
M = N = K = 128
I = np.eye(128, dtype=np.float32)
R = rng.standard_normal((128, 128)).astype(np.float32)
for ta in (0, 1):
    for tb in (0, 1):
        for eng in (2, 1):
            out[f"AI_{ta}{tb}_{eng}"] = V.debug_gemm(I, R, bool(ta), bool(tb), engine=eng)
            out[f"BI_{ta}{tb}_{eng}"] = V.debug_gemm(R, I, bool(ta), bool(tb), engine=eng)
out["R"] = R
np.savez("gpurun_out/gemm_diag.npz", **out)
print("saved")
