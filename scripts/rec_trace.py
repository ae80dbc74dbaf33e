"""Summarise VER_REC_TRACE output: per-step time (us) vs rows bs_t, per launch."""
import sys
for line in open(sys.argv[1]):
    tag, L, *rest = line.split()
    pts = [tuple(map(int, x.split(":"))) for x in rest]
    bs = [p[0] for p in pts]
    ts = [p[1] for p in pts]
    steps = range(len(ts)) if tag.startswith("fwd") else range(len(ts) - 1, -1, -1)
    order = [t for t in steps if ts[t] > 0]
    d = {}
    for a, b in zip(order, order[1:]):
        d[a] = (ts[b] - ts[a]) / 1000.0
    tot = (ts[order[-1]] - ts[order[0]]) / 1000.0
    big = sum(v for t, v in d.items() if bs[t] > 64)
    small = sum(v for t, v in d.items() if bs[t] <= 16)
    print(f"{tag} L={L} span={tot:.0f}us  steps(bs>64)={sum(1 for t in d if bs[t] > 64)} {big:.0f}us  "
          f"steps(bs<=16)={sum(1 for t in d if bs[t] <= 16)} {small:.0f}us  "
          f"first: " + " ".join(f"{bs[t]}:{d[t]:.1f}" for t in order[:6] if t in d) +
          "  last: " + " ".join(f"{bs[t]}:{d[t]:.1f}" for t in order[-6:-1] if t in d))
