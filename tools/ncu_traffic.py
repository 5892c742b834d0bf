#!/usr/bin/env python
"""DRAM traffic per launch of the query kernels, from an `ncu --set full` report of
`bench.py --chunks 1` (one launch per stage per step), into profiles/traffic.json, which
bench.py reports as roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum).

    python tools/ncu_traffic.py gpurun_out/q5_full.ncu-rep gist1m 1000 > profiles/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

STAGE = {"traverse": "traverse", "binsel": "binsel", "rerank": "rerank", "exact": "exact"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, workload, queries):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {}
    for r in data:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        stage = next((v for k, v in STAGE.items() if k in name), None)
        if stage is None:
            continue
        b = sum(float(d[m].replace(",", "")) * UNIT.get(units[hdr.index(m)], 1)
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res.setdefault(stage, []).append((b, name.split("(")[0]))
    traffic = {s: {"kernel": v[0][1], "dram_bytes_per_launch": sum(x for x, _ in v) / len(v), "launches": len(v)}
               for s, v in res.items()}
    print(json.dumps({"report": path.split("/")[-1], "workload": workload, "queries_per_launch": int(queries),
                      "kernels": traffic}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
