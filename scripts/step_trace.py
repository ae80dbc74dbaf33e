"""Summarise the persistent step kernel's VER_REC_TRACE lines (csrc/stepgemm.cu):
per row bucket, the mean time (us, CTA 0) from step start to each phase point."""
import sys
from collections import defaultdict

NAMES = ["landed", "acc_ready", "stored", "bar1", "gate_done", "next"]
FUSED = ["landed", "acc_ready", "pushed", "received", "gate_done", "next"]
acc = defaultdict(lambda: defaultdict(list))
for line in open(sys.argv[1]):
    tag, n, *rest = line.split()
    if not tag.startswith(("persist", "fused", "pair")):
        continue
    for x in rest:
        v = list(map(int, x.split(":")))
        rows, z, pts = v[0], v[1], v[2:]
        b = (tag, min(rows // 100 * 100, 600) if rows < 1000 else min(rows // 1000 * 1000, 12000), z)
        for k, p in enumerate(pts):
            if p >= 0:
                acc[b][(FUSED if tag.startswith("fused") else NAMES)[k]].append(p / 1000.0)
for b in sorted(acc):
    d = acc[b]
    print(f"{b[0]} rows~{b[1]:>5} Z={b[2]} n={len(d['next']):>4} " +
          " ".join(f"{k}={sum(v) / len(v):.2f}" for k, v in d.items() if v))
