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
    dev.enable_query_times(True)
    import torch

    k = 100
    dq = torch.empty((B, Q.shape[1]), dtype=torch.float32, device="cuda")
    ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
    d = torch.empty((B, k), dtype=torch.float32, device="cuda")
    c = torch.empty(B, dtype=torch.int32, device="cuda")
    st = torch.empty((B, 3), dtype=torch.int64, device="cuda")
    rows, qts, sms, merge_steps, gaps = [], [], [], [], []
    for r in range(20):
        dq.copy_(torch.from_numpy(Q[r * B:(r + 1) * B]))
        dev.search_device(dq.data_ptr(), B, k, ids.data_ptr(), d.data_ptr(), c.data_ptr(), st.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
        qts.append(dev.query_times(B).max(axis=0))
        raw = np.zeros((B, 3, 2), np.uint64)
        check(lib().pqtg_debug_query_clocks(dev.workspace, B, raw.ctypes.data))
        st0 = raw[:, :, 0].min(axis=0).astype(np.int64)
        en0 = raw[:, :, 1].max(axis=0).astype(np.int64)
        sms.append(dev.stage_ms())
        ph = (C.c_uint64 * 16)()
        check(lib().pqtg_debug_rerank_phases(ph))
        t = np.array(list(ph), np.float64)
        gaps.append([(st0[1] - en0[0]) / 1e3, (t[0] - st0[1]) / 1e3, (st0[2] - en0[1]) / 1e3])
        rows.append(np.diff(t[[0, 1, 2, 3, 4, 5]]) / 1e3)
        if t[6] > t[7] > t[5]:
            merge_steps.append(np.diff(t[[7, 8, 9, 10, 6]]) / 1e3)
            rows[-1] = np.append(rows[-1], [(t[7] - t[5]) / 1e3, (t[6] - t[7]) / 1e3])
    med = np.median(np.array([r[:5] for r in rows]), axis=0)
    out = {"workload": name, "batch": B, "us": dict(zip(["prologue", "range_map", "score", "select", "write"],
                                                        [round(float(x), 2) for x in med]))}
    if len(rows[-1]) > 5:
        out["us"]["last_slice_arrival"] = round(float(np.median([r[5] for r in rows if len(r) > 5])), 2)
        out["us"]["last_slice_merge"] = round(float(np.median([r[6] for r in rows if len(r) > 6])), 2)
    out["in_kernel_us"] = [round(float(x), 2) for x in np.median(np.array(qts), axis=0)]
    out["events_us"] = [round(1e3 * float(x), 2) for x in np.median(np.array(sms), axis=0)]
    out["gaps_us"] = dict(zip(["traverse_end_to_binsel_start", "binsel_start_to_rerank_entry",
                               "binsel_end_to_rerank_start"], [round(float(x), 2) for x in np.median(np.array(gaps), axis=0)]))
    if len(rows[-1]) > 5:
        out["merge_steps_us"] = dict(zip(["lists", "lengths_threshold", "compact", "rank_write"],
                                         [round(float(x), 2) for x in np.median(np.array(merge_steps), axis=0)]))
    out["merge_kept_keys"] = int(t[12])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
