"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` (needs --import-source)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]; data = rows[1:]
si, ai, ni = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[ai] or 0) for r in data)
byop = collections.Counter()
for r in data:
    byop[r[si].split()[0] if r[si].split() else "?"] += int(r[ai] or 0)
print("total samples", tot)
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(12)))
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][ai] or 0))[:top]:
    print(f"{i:5d} {100*int(r[ai])/tot:5.1f}%  exec={r[ni]:>8}  {r[si].strip()[:90]}")
