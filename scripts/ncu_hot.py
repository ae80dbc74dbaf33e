"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` (needs --import-source).

  python scripts/ncu_hot.py report.ncu-rep [top] [kernel-substring]
"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sections, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line, []]; sections.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in sections:
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]; data = [r for r in rows[1:] if len(r) == len(h)]
    si, ai, ni = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(int(r[ai] or 0) for r in data) or 1
    byop = collections.Counter()
    for r in data:
        byop[r[si].split()[0] if r[si].split() else "?"] += int(r[ai] or 0)
    print(name[:150]); print("total samples", tot)
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(12)))
    for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][ai] or 0))[:top]:
        print(f"{i:5d} {100*int(r[ai])/tot:5.1f}%  exec={r[ni]:>8}  {r[si].strip()[:90]}")
    break
