#!/usr/bin/env python
"""Summarize an ncu report (.ncu-rep) into a small markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/r01_prof8.ncu-rep > profiles/r01_ncu_summary.md

Per kernel launch: duration, DRAM read+write bytes, L2 traffic, instructions, IPC,
occupancy, shared-memory wavefronts/bank conflicts and the top stall reasons (source page).
"""
import csv
import io
import subprocess
import sys
from collections import Counter

RAW = [
    ("gpu__time_duration.sum", "dur_us"),
    ("dram__bytes_read.sum", "dram_rd_MB"),
    ("dram__bytes_write.sum", "dram_wr_MB"),
    ("lts__t_bytes.sum", "l2_MB"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(path):
    rows = list(csv.reader(io.StringIO(ncu(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"ncu report `{path.split('/')[-1]}` (`--set full --clock-control none`; one launch per row)\n")
    print("| kernel | " + " | ".join(n for _, n in RAW) + " | top stalls |")
    print("|---" * (len(RAW) + 2) + "|")
    for r in data:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        vals = []
        for key, _ in RAW:
            v = d.get(key, "")
            u = units[hdr.index(key)] if key in hdr else ""
            try:
                x = float(v.replace(",", ""))
                if key == "gpu__time_duration.sum" and u == "ns":
                    x /= 1000.0
                if key.startswith(("dram__", "lts__")):
                    x = x / 1e6 if u in ("byte", "") else (x / 1e3 if u == "Kbyte" else (x * 1e3 if u == "Gbyte" else x))
                vals.append(f"{x:.4g}")
            except ValueError:
                vals.append(v)
        src = list(csv.reader(io.StringIO(ncu(["-i", path, "--page", "source", "--csv", "-k", f"regex:{name.split('<')[0]}",
                                               "--print-source=sass"]))))
        stalls = Counter()
        if len(src) > 2:
            sh = src[1]
            cols = [h for h in sh if h.startswith("stall_") and "Not Issued" not in h]
            for s in src[2:]:
                for h in cols:
                    try:
                        stalls[h[6:]] += float(s[sh.index(h)] or 0)
                    except (ValueError, IndexError):
                        pass
        tot = sum(stalls.values()) or 1
        top = ", ".join(f"{k} {v / tot:.0%}" for k, v in stalls.most_common(3))
        print(f"| {name} | " + " | ".join(vals) + f" | {top} |")


if __name__ == "__main__":
    main(sys.argv[1])
