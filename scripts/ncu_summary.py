"""Markdown summary of an `ncu --set full` report (one row block per kernel launch).

  python scripts/ncu_summary.py report.ncu-rep [title] > profiles/rNN_<name>.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak (active)"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % of elapsed"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory (TMEM) active % of elapsed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {title}\n")
    print(f"Source: `{path}` (`ncu --set full --clock-control none`), read with `ncu -i --page raw --csv`.\n")
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"## {d['Kernel Name'][:120]}\n")
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d and d[k] != "":
                print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v)))
                except ValueError:
                    pass
        if st:
            st.sort(key=lambda x: -x[1])
            print("\nTop warp stall reasons (cycles per issued instruction): " +
                  ", ".join(f"{k} {v:.2f}" for k, v in st[:6]))
        print()


if __name__ == "__main__":
    main()
