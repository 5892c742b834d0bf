#!/usr/bin/env python
"""GPU probe: where the end-to-end (host-buffer) search time goes, per chunk count.

    python tools/e2e_probe.py [--workload gist1m] [--nq 1000]

Prints, per chunk setting: device-resident ms/step (CUDA events), host-call ms/step
(pqtg_search on pinned buffers), plus the bare H2D/D2H copy times of one step's bytes.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
from paper_1702_05911_b200 import DeviceIndex  # noqa: E402
from paper_1702_05911_b200._abi import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gist1m")
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--reps", type=int, default=100)
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    nq = a.nq or wl["nq"]
    k = wl["k"]
    hix, Qpool = bench.make_workload(a.workload, 7, 0, max(1, (4 * nq + wl["nq"] - 1) // wl["nq"]))
    dim = hix.config.dim
    batches = [Qpool[i * nq:(i + 1) * nq] for i in range(4)]
    dev = DeviceIndex(hix, max_batch=max(nq, 1))
    hq = [torch.from_numpy(np.ascontiguousarray(b)).pin_memory() for b in batches]
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    h_c = torch.empty(nq, dtype=torch.int32).pin_memory()
    h_s = torch.empty((nq, 3), dtype=torch.int64).pin_memory()
    d_q = [b.cuda() for b in hq]
    d_ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d_d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    d_c = torch.empty(nq, dtype=torch.int32, device="cuda")
    d_s = torch.empty((nq, 3), dtype=torch.int64, device="cuda")
    L = lib()
    st = torch.cuda.current_stream()

    # bare copies of one step's bytes
    t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn in [("h2d", lambda: d_q[0].copy_(hq[0], non_blocking=True)),
                     ("d2h", lambda: (h_ids.copy_(d_ids, non_blocking=True), h_d.copy_(d_d, non_blocking=True)))]:
        fn()
        torch.cuda.synchronize()
        t[0].record()
        for _ in range(a.reps):
            fn()
        t[1].record()
        torch.cuda.synchronize()
        print(f"{name}: {t[0].elapsed_time(t[1]) / a.reps * 1000:.1f} us/step")

    import os

    plans = [(c, "") for c in (1, 2, 4, 0)]
    for chunks, plan in plans:
        os.environ["PQTG_CHUNK_PLAN"] = plan
        if not plan:
            del os.environ["PQTG_CHUNK_PLAN"]
        dev.set_chunks(chunks)
        for b in range(4):
            dev.search_device(d_q[b].data_ptr(), nq, k, d_ids.data_ptr(), d_d.data_ptr(), d_c.data_ptr(),
                              d_s.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        t[0].record()
        for r in range(a.reps):
            dev.search_device(d_q[r % 4].data_ptr(), nq, k, d_ids.data_ptr(), d_d.data_ptr(), d_c.data_ptr(),
                              d_s.data_ptr(), st.cuda_stream)
        t[1].record()
        torch.cuda.synchronize()
        dms = t[0].elapsed_time(t[1]) / a.reps

        def host(b):
            rc = L.pqtg_search(dev.handle, dev.workspace, hq[b].data_ptr(), nq, dim, k, h_ids.data_ptr(),
                               h_d.data_ptr(), h_c.data_ptr(), h_s.data_ptr())
            assert rc == 0

        for b in range(4):
            host(b)
        ts = []
        for r in range(a.reps):
            t0 = time.perf_counter()
            host(r % 4)
            ts.append(time.perf_counter() - t0)
        # the bench's e2e loop: a 256 MiB L2 flush (+ sync) outside each timed call
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        tf = []
        for r in range(a.reps):
            flush.fill_(r & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host(r % 4)
            tf.append(time.perf_counter() - t0)
        del flush
        print(f"   after L2 flush: host call median {np.median(tf) * 1e6:.1f} us mean {np.mean(tf) * 1e6:.1f} us "
              f"p90 {np.percentile(tf, 90) * 1e6:.1f} max {np.max(tf) * 1e6:.1f}")
        # back-to-back host calls with no sync between (the CPU cost of one call)
        t0 = time.perf_counter()
        for r in range(a.reps):
            host(r % 4)
        bb = (time.perf_counter() - t0) / a.reps
        print(f"chunks={chunks} plan={plan or '-'}: device {dms * 1000:.1f} us/step ({nq / dms * 1000 / 1e6:.2f} Mq/s); "
              f"host call median {np.median(ts) * 1e6:.1f} us min {np.min(ts) * 1e6:.1f} us "
              f"({nq / np.median(ts) / 1e6:.2f} Mq/s); back-to-back {bb * 1e6:.1f} us")


if __name__ == "__main__":
    main()
