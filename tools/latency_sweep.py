#!/usr/bin/env python
"""BASELINE.json configs[4]: single-query latency sweep on the SIFT1M shape (batch 1 -> 100k).

    python tools/latency_sweep.py [--workload sift1m] [--out gpurun_out/latency_sweep.json]

Per batch size B (queries tiled from the workload's query pool): device latency of one
search with the queries resident in HBM (CUDA events on the launching stream, median over
repetitions) and end-to-end latency of pqtg_search on page-locked host buffers (host clock,
H2D + kernels + D2H, a replayed CUDA graph). The CPU reference's per-query latency on all host
cores is given for the batch of 1 and the batch of 1000. One JSON object per line.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
from paper_1702_05911_b200 import DeviceIndex  # noqa: E402
from paper_1702_05911_b200._abi import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="sift1m")
    ap.add_argument("--sizes", default="1,10,100,1000,10000,100000")
    ap.add_argument("--out", default="")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    k = wl["k"]
    hix, Qpool = bench.make_workload(a.workload, 7, 0, 1)
    # the sweep goes to 100k queries: tile the pool
    sizes = [int(x) for x in a.sizes.split(",")]
    dev = DeviceIndex(hix, max_batch=max(sizes))
    dim = hix.config.dim
    L = lib()
    st = torch.cuda.current_stream()
    lines = []
    for B in sizes:
        reps = int(min(200, max(5, 2e5 / max(B, 1))))
        Q = np.ascontiguousarray(np.resize(Qpool, (B, dim)))
        dq = torch.from_numpy(Q).cuda()
        d_ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
        d_d = torch.empty((B, k), dtype=torch.float32, device="cuda")
        d_c = torch.empty(B, dtype=torch.int32, device="cuda")
        d_s = torch.empty((B, 3), dtype=torch.int64, device="cuda")
        for _ in range(3):
            dev.search_device(dq.data_ptr(), B, k, d_ids.data_ptr(), d_d.data_ptr(), d_c.data_ptr(), d_s.data_ptr(),
                              st.cuda_stream)
        torch.cuda.synchronize()
        ms = []
        sampler = bench.ClockSampler(0, period=0.001)
        sampler.__enter__()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            dev.search_device(dq.data_ptr(), B, k, d_ids.data_ptr(), d_d.data_ptr(), d_c.data_ptr(), d_s.data_ptr(),
                              st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        sampler.__exit__(None, None, None)
        stage = dev.stage_ms()  # [traverse, bin selection, re-rank + top-k, whole] of the last call
        hq = torch.from_numpy(Q).pin_memory()
        h_ids = torch.empty((B, k), dtype=torch.int32).pin_memory()
        h_d = torch.empty((B, k), dtype=torch.float32).pin_memory()
        h_c = torch.empty(B, dtype=torch.int32).pin_memory()
        h_s = torch.empty((B, 3), dtype=torch.int64).pin_memory()

        def host():
            check(L.pqtg_search(dev.handle, dev.workspace, hq.data_ptr(), B, dim, k, h_ids.data_ptr(),
                                h_d.data_ptr(), h_c.data_ptr(), h_s.data_ptr()))

        for _ in range(3):
            host()
        hs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            host()
            hs.append(time.perf_counter() - t0)
        dmed, hmed = float(np.median(ms)), float(np.median(hs)) * 1e3
        line = {"workload": a.workload, "batch": B, "k": k, "reps": reps,
                "device_ms": dmed, "device_p90_ms": float(np.percentile(ms, 90)),
                "device_qps": B / dmed * 1e3, "e2e_ms": hmed, "e2e_p90_ms": float(np.percentile(hs, 90) * 1e3),
                "e2e_qps": B / hmed * 1e3,
                "stage_ms_last_call": {"traverse": stage[0], "binsel": stage[1], "rerank": stage[2], "total": stage[3]},
                "clocks": sampler.summary()}
        if not a.no_cpu and B in (1, 1000):
            from oracle.bindings import Ref

            if Ref.available():
                ref = getattr(main, "_ref", None) or Ref.from_host(hix)
                main._ref = ref
                threads = os.cpu_count() or 1
                ref.knn(Q[:min(B, 16)], k, threads=threads)
                n_rep = 50 if B == 1 else 3
                t0 = time.perf_counter()
                for _ in range(n_rep):
                    ref.knn(Q, k, threads=threads)
                t = (time.perf_counter() - t0) / n_rep
                line["cpu_reference_ms"] = t * 1e3
                line["cpu_reference_cores"] = threads
        print(json.dumps(line), flush=True)
        lines.append(line)
        del dq, d_ids, d_d, d_c, d_s
    if a.out:
        Path(a.out).write_text("\n".join(json.dumps(x) for x in lines) + "\n")


if __name__ == "__main__":
    main()
