"""GPU learner update and the CPU oracle (double, the
reference's algorithmic structure) at configs[0] (C1) and configs[1] (C2) on
the box's host, same synthetic workload.  C3 / C5 come from
bench.py and scripts/sweep_c5.py.  One JSON line per config.

  python scripts/configs_table.py [--cpu-threads K]"""
import json
import os
import statistics
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix
from oracle import oracle as O  # CPU baseline leg only

args = sys.argv[1:]
thr_c2 = int(args[args.index("--cpu-threads") + 1]) if "--cpu-threads" in args else (os.cpu_count() or 1)
T = 128
for name, N, EH, epochs, cpu_thr in (("configs[0] C1", 16, 64, 1, 1), ("configs[1] C2", 256, 512, 4, thr_c2)):
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=EH, hidden_dim=EH, action_kind=0, num_actions=2)
    ctx = V.Context(0)
    wl = synth.make_workload(T, N, hidden_dim=EH, seed=1)
    buf = V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, EH, ctx=ctx)
    synth.fill_buffer(buf, wl)
    view = buf.close_rollout()
    L = V.Learner(cfg, V.params_init(cfg, mix(1, 0x9A9A)), V.PPOConfig(epochs=epochs, minibatches=2),
                  V.EntropyController(), V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D), ctx=ctx)
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        L.update(view, read_stats=False)
    ctx.synchronize()
    ms = []
    for _ in range(10):
        with torch.cuda.stream(stream):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
        L.update(view, read_stats=False)
        with torch.cuda.stream(stream):
            b.record(stream)
        ctx.synchronize()
        ms.append(a.elapsed_time(b))
    fresh = view.fresh_steps()
    gpu_ms = statistics.median(ms)
    # CPU: the oracle's full update on the same workload
    O.set_threads(cpu_thr)
    O.set_sparse_rows(False)
    r = O.Rollout(T, N, 1, 0, 2, 0, EH)
    synth.fill_buffer(r, wl)
    ov = r.close_rollout()
    OL = O.Learner(cfg, O.params_init(cfg, O.mix(1, 0x9A9A)), V.PPOConfig(epochs=epochs, minibatches=2),
                   V.EntropyController(), 2.5e-4, 2_000_000, O.mix(1, 0xF00D))
    t0 = time.perf_counter()
    OL.update(ov)
    cpu_s = time.perf_counter() - t0
    print(json.dumps({"config": name, "N": N, "E=H": EH, "epochs": epochs, "fresh_steps": fresh,
                      "gpu_update_ms": gpu_ms, "gpu_env_steps_per_s": fresh / (gpu_ms / 1000.0),
                      "cpu_update_s": cpu_s, "cpu_env_steps_per_s": fresh / cpu_s, "cpu_threads": cpu_thr,
                      "cpu_kind": "oracle port (double), full update"}), flush=True)
