"""Phase clocks of the re-rank kernel at a small batch (run with PQTG_PHASES=1; PQTG_SPLIT=1 for
the split variant): start → prologue (tables) → range map → candidates scored → selected →
written (→ merged by the last slice), microseconds from the kernel's first CTA.

    PQTG_PHASES=1 python tools/phase_probe.py [workload] [batch]"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    import bench
    from paper_1702_05911_b200 import DeviceIndex
    from paper_1702_05911_b200._abi import check, lib

    name = sys.argv[1] if len(sys.argv) > 1 else "sift1m"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    hix, Q = bench.make_workload(name, 7, 0, 1)
    dev = DeviceIndex(hix, max_batch=max(B, 1))
    rows = []
    for r in range(20):
        dev.search(Q[r * B:(r + 1) * B], 100)
        ph = (C.c_uint64 * 7)()
        check(lib().pqtg_debug_rerank_phases(ph))
        t = np.array(list(ph), np.float64)
        rows.append(np.diff(t[[0, 1, 2, 3, 4, 5]]) / 1e3)
        if t[6] > t[5]:
            rows[-1] = np.append(rows[-1], (t[6] - t[5]) / 1e3)
    med = np.median(np.array([r[:5] for r in rows]), axis=0)
    out = {"workload": name, "batch": B, "us": dict(zip(["prologue", "range_map", "score", "select", "write"],
                                                        [round(float(x), 2) for x in med]))}
    if len(rows[-1]) > 5:
        out["us"]["last_slice_merge"] = round(float(np.median([r[5] for r in rows if len(r) > 5])), 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
