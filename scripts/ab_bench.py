"""A/B of env knobs on the headline learner update (C3 by default; --c2 for configs[1]),
interleaved so clock / power drift hits every variant alike:
  python scripts/ab_bench.py [--c2] [--rounds R] 'VAR=a,VAR2=b' 'VAR=c' ..."""
import json, os, subprocess, sys
args = sys.argv[1:]
c2 = "--c2" in args
rounds = 2
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    del args[i:i + 2]
specs = [a for a in args if a != "--c2"] or [""]
code = r'''
import json, sys, statistics, torch
sys.argv = ["bench.py"]
import bench
C2 = %d
import paper_2210_05064_b200 as V
from paper_2210_05064_b200 import synth
from paper_2210_05064_b200.rng import mix
N, EP = (bench.N2, bench.EPOCHS2) if C2 else (bench.N_, bench.EPOCHS)
cfg = V.ModelConfig(obs_dim=2, encoder_dim=512, hidden_dim=512, action_kind=0, num_actions=2)
ctx = V.Context(0)
wl = synth.make_workload(128, N, hidden_dim=512, seed=1)
buf = V.RolloutBuffer(128, N, V.VARIABLE, 0, 2, 0, 512, ctx=ctx)
synth.fill_buffer(buf, wl)
view = buf.close_rollout()
L = V.Learner(cfg, V.params_init(cfg, mix(1, 0x9A9A)), V.PPOConfig(epochs=EP, minibatches=2), V.EntropyController(),
              V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D), ctx=ctx)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(2):
    L.update(view, read_stats=False)
ctx.synchronize()
ms = []
for _ in range(5):
    with torch.cuda.stream(stream):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True); a.record(stream)
    L.update(view, read_stats=False)
    with torch.cuda.stream(stream):
        b.record(stream)
    ctx.synchronize(); ms.append(a.elapsed_time(b))
print(json.dumps({"ms": statistics.median(ms), "phases": L.last_timing()}))
''' % (1 if c2 else 0)
for r in range(rounds):
    for spec in specs:
        env = dict(os.environ)
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(spec, "FAILED", out.stderr[-2000:], flush=True)
            continue
        print(r, spec or "default", round(d["ms"], 3),
              {k: round(v, 2) for k, v in d["phases"].items() if v}, flush=True)
