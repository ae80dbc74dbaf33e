"""profiles/traffic.json: DRAM bytes and duration per launch of the profiled kernels
from `ncu --set full` reports (the `traffic` of bench.py's roofline).

  python scripts/traffic_json.py name=report.ncu-rep [...]
"""
import csv, io, json, subprocess, sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
path = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
out = json.loads(path.read_text()) if path.exists() else {}
for arg in sys.argv[1:]:
    k, rep = arg.split("=", 1)
    o = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(o)))
    h, units, r = rows[0], rows[1], rows[2]
    val = lambda m: float(r[h.index(m)]) * SCALE[units[h.index(m)]]  # noqa: E731
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    out[k] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
              "duration_us": val("gpu__time_duration.sum"), "source": Path(rep).name}
path.write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
