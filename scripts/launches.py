"""Summarise an ncu --metrics gpu__time_duration.sum launch list (last `frac` of launches)."""
import collections, csv, sys
path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
sel = data[int(len(data) * (1 - frac)):]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in sel:
    agg[r[ki].split('(')[0][:70]][0] += 1
    agg[r[ki].split('(')[0][:70]][1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(f"{v[1]/1e6:9.3f} ms {100*v[1]/tot:5.1f}% n={v[0]:5d} avg={v[1]/v[0]/1e3:8.1f}us  {k}")
print(f"total {tot/1e6:.3f} ms over {len(sel)} launches")
