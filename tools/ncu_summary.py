"""Summarise an ncu report: per kernel time, DRAM bytes, issue activity and top stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        print(r[h.index("Kernel Name")][:70])
        print("   " + "  ".join(f"{w.split('.')[0].split('__')[-1]}={r[h.index(w)]}" for w in WANT if w in h))
        st = []
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), name.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
