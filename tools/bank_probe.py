"""Shared-memory bank-conflict model of the re-rank's per-part table lookups on real candidate
lists (a GPU-built index of the named workload; candidates from the GPU's own bin selection).

For every warp of 32 consecutive candidates of a query and every line part f, counts the
wavefronts of each lookup under candidate table layouts:
  T64      the current float2 T[f][t], t = i << 4 | ((i + j) & 15)        (LDS.64)
  E32/t    split E[f][t], c2[f][t] float tables, same t                   (2 x LDS.32)
  b2       fine[f][i]                                                      (LDS.32)
  P3/<s>   three pid-indexed tables E, c2, b2 [f][slot(pid)] (128 slots)  (3 x LDS.32, one address)
Usage: python tools/bank_probe.py [workload] [queries]"""
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def _uniq_rows(a):
    """a [rows, lanes] -> (sorted a, mask of first occurrences per row)."""
    a = np.sort(a, axis=1)
    first = np.ones_like(a, dtype=bool)
    first[:, 1:] = a[:, 1:] != a[:, :-1]
    return a, first


def _max_bank(a, first, banks_of):
    rows = a.shape[0]
    cnt = np.zeros((rows, 32), np.int64)
    r = np.repeat(np.arange(rows), a.shape[1]).reshape(a.shape)
    for b in banks_of(a):
        np.add.at(cnt, (r[first], b[first]), 1)
    return cnt.max(axis=1)


def wf32(addr):
    """wavefronts of LDS.32 warp accesses (rows of 32 lanes): max over banks of distinct words."""
    a, f = _uniq_rows(addr)
    return _max_bank(a, f, lambda x: [x % 32])


def wf64_half(addr):
    """LDS.64 modelled as two half-warps, each over 32 banks (an 8-byte entry spans 2)."""
    tot = 0
    for h in (addr[:, :16], addr[:, 16:]):
        a, f = _uniq_rows(h)
        tot = tot + _max_bank(a, f, lambda x: [(2 * x) % 32, (2 * x + 1) % 32])
    return tot


def wf64_full(addr):
    a, f = _uniq_rows(addr)
    return np.maximum(2, _max_bank(a, f, lambda x: [(2 * x) % 32, (2 * x + 1) % 32]))


def slot_spread(k1):
    """pid -> slot (0..127): pairs sharing an endpoint in distinct banks where possible
    (greedy: each pair takes the lowest-conflict bank, then the next free row in it)."""
    pairs = [(i, j) for i in range(k1) for j in range(i + 1, k1)]
    used = {}  # bank -> rows used
    ends = {}  # (endpoint, bank) -> count
    slot = {}
    for (i, j) in pairs:
        best = None
        for b in range(32):
            if used.get(b, 0) >= 4:
                continue
            cost = ends.get((i, b), 0) + ends.get((j, b), 0)
            key = (cost, used.get(b, 0), b)
            if best is None or key < best:
                best = key
        b = best[2]
        slot[(i, j)] = used.get(b, 0) * 32 + b
        used[b] = used.get(b, 0) + 1
        ends[(i, b)] = ends.get((i, b), 0) + 1
        ends[(j, b)] = ends.get((j, b), 0) + 1
    return slot


def main():
    import torch

    import bench
    from paper_1702_05911_b200 import DeviceIndex

    name = sys.argv[1] if len(sys.argv) > 1 else "deep100m"
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    hix, Q = bench.make_workload(name, 7, 0, 1)
    c = hix.config
    k1, L = c.k1, c.p_line
    dev = DeviceIndex(hix, max_batch=nq)
    dev.search(Q[:nq], 100)
    inter = dev.intermediates(nq)
    lam = hix.lambda_q.reshape(hix.n, L)
    pid = hix.pair_id.reshape(hix.n, L).astype(np.int64)
    pairs = [(0, 0)] if k1 <= 1 else [(i, j) for i in range(k1) for j in range(i + 1, k1)]
    pi = np.array([p[0] for p in pairs])
    pj = np.array([p[1] for p in pairs])
    sl = slot_spread(k1)
    slot = np.array([sl[p] for p in pairs]) if k1 > 1 else np.zeros(1, np.int64)
    acc = {k: 0.0 for k in ["T64_half", "T64_full", "E32_t", "b2", "P3_spread", "P3_pid"]}
    n = 0
    for q in range(nq):
        pos = inter["positions"][q]
        nw = len(pos) // 32
        if nw == 0:
            continue
        ids = hix.ids[pos[: nw * 32]]
        Pq = pid[ids].reshape(nw, 32, L).transpose(0, 2, 1).reshape(nw * L, 32)  # [warp*part][lane]
        f = np.tile(np.arange(L), nw)[:, None]
        i, j = pi[Pq], pj[Pq]
        t = (i << 4) | ((i + j) & 15)
        acc["T64_half"] += float(wf64_half(f * 256 + t).sum())
        acc["T64_full"] += float(wf64_full(f * 256 + t).sum())
        acc["E32_t"] += 2.0 * float(wf32(f * 256 + t).sum())
        acc["b2"] += float(wf32(f * 16 + i).sum())
        acc["P3_spread"] += 3.0 * float(wf32(f * 128 + slot[Pq]).sum())
        acc["P3_pid"] += 3.0 * float(wf32(f * 128 + Pq).sum())
        n += nw * L
    out = {k: v / n for k, v in acc.items()}
    out["warp_parts"] = n
    out["note"] = "wavefronts per warp-part; measured T64 LDS.64 on DEEP100M (ncu r02a): 4.67, ideal 2"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
