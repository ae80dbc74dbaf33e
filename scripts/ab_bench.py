"""A/B of env knobs on the C2 learner update: python scripts/ab_bench.py 'VAR=a,VAR2=b' 'VAR=c' ..."""
import json, os, subprocess, sys
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu", "--no-c5", "--no-c3", "--no-collect", "--steps", "5"], env=env,
                         capture_output=True, text=True).stdout.strip().splitlines()
    d = json.loads(out[-1])
    print(spec or "default", round(d["ms_per_step"], 3),
          {k: round(v, 2) for k, v in d["phases_ms"].items() if v}, flush=True)
