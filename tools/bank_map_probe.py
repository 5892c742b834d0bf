"""CPU model of the re-rank's T-table gathers under slot maps (no GPU): builds (or reuses) a
DEEP-shaped index with the reference builder, samples half-warps of 16 consecutive positions and
counts LDS.64 wavefronts per half-warp-part (max over the 16 bank pairs of the distinct slots in
it) for the fixed slots t = i << 4 | ((i + j) & 15) and for per-part maps.

    python tools/bank_map_probe.py [n] [path]

A 1M-vector index is not DEEP100M: its cells hold ~60 vectors (DEEP100M ~6100, one bin fills the
budget), so its half-warps see fewer distinct pairs (1M: fixed 2.36 -> greedy 2.17 wavefronts per
warp-part; the GPU measured 4.67 on DEEP100M). The GPU numbers (ncu bank conflicts, re-rank time)
are the ones to trust; this is for checking a map's construction without a GPU."""
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def index(n, path):
    from oracle.bindings import Ref
    from paper_1702_05911_b200.index import HostIndex, PqtConfig

    p = Path(path)
    if not p.exists():
        cfg = PqtConfig(dim=96, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=4096, train_iters=10, seed=7)
        X = Ref.synth(n, 96, max(n // 1000, 16), 20.0, 7)
        t0 = time.time()
        Ref.build(X[: min(n, 100_000)], X, cfg).save(str(p))
        print(f"built {n} in {time.time() - t0:.0f}s", flush=True)
    return HostIndex.load(str(p))


def groups(hix, ng, rng):
    n = hix.n
    starts = np.sort(rng.integers(0, n - 16, ng))
    pos = starts[:, None] + np.arange(16)[None, :]
    return hix.pair_id[hix.ids[pos].astype(np.int64)]  # [ng, 16, L] pair ids


def wavefronts(slots):
    """slots [ng, 16] -> wavefronts per half-warp (distinct slots per bank pair, max)."""
    s = np.sort(slots, axis=1)
    first = np.ones_like(s, bool)
    first[:, 1:] = s[:, 1:] != s[:, :-1]
    bank = s & 15
    cnt = np.zeros((s.shape[0], 16), np.int64)
    r = np.repeat(np.arange(s.shape[0]), 16).reshape(s.shape)
    np.add.at(cnt, (r[first], bank[first]), 1)
    return cnt.max(axis=1)


def pairs_of(k1):
    return [(i, j) for i in range(k1) for j in range(i + 1, k1)]


def greedy(G, pr, passes=4):
    """pairwise co-occurrence greedy + move/swap passes (index_prep.cpp bank_map)."""
    np_ = len(pr)
    W = np.zeros((np_, np_), np.int64)
    for g in G:
        u = np.unique(g)
        W[np.ix_(u, u)] += 1
    np.fill_diagonal(W, 0)
    first = np.array([i for i, _ in pr])
    nib = np.full(np_, 16)
    used = np.zeros(16, np.int64)
    order = np.argsort(-W.sum(1), kind="stable")

    def cost(a, n):
        m = (nib == n) & (first != first[a])
        m[a] = False
        return W[a, m].sum()

    for a in order:
        i, j = pr[a]
        best, bc = 16, None
        for k in range(16):
            n = (i + j + k) & 15
            if used[i] >> n & 1:
                continue
            c = cost(a, n)
            if bc is None or c < bc:
                bc, best = c, n
        nib[a] = best
        used[i] |= 1 << best
    for _ in range(passes):
        moved = False
        for a in range(np_):
            i, na = first[a], nib[a]
            for n in range(16):
                if n == na:
                    continue
                r = next((b for b in range(np_) if first[b] == i and nib[b] == n), None)
                before = cost(a, na) + (cost(r, n) if r is not None else 0)
                nib[a] = n
                if r is not None:
                    nib[r] = na
                after = cost(a, n) + (cost(r, na) if r is not None else 0)
                if after < before:
                    if r is None:
                        used[i] = (used[i] & ~(1 << na)) | (1 << n)
                    moved = True
                    break
                nib[a] = na
                if r is not None:
                    nib[r] = n
        if not moved:
            break
    return np.array([(pr[a][0] << 4) | nib[a] for a in range(np_)])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    path = sys.argv[2] if len(sys.argv) > 2 else f"/tmp/bm/deep_{n}.pqt"
    hix = index(n, path)
    rng = np.random.default_rng(1)
    train = groups(hix, 16384, rng)
    test = groups(hix, 8192, np.random.default_rng(2))
    pr = pairs_of(hix.config.k1)
    fixed = np.array([(i << 4) | ((i + j) & 15) for i, j in pr])
    L = hix.config.p_line
    tot = {"fixed": 0.0, "greedy": 0.0, "distinct": 0.0}
    for f in range(L):
        tot["fixed"] += wavefronts(fixed[test[:, :, f]]).mean()
        m = greedy(train[:, :, f], pr)
        tot["greedy"] += wavefronts(m[test[:, :, f]]).mean()
        s = np.sort(test[:, :, f], axis=1)
        tot["distinct"] += (1 + (s[:, 1:] != s[:, :-1]).sum(1)).mean()
    for k, v in tot.items():
        print(k, round(2 * v / L, 3), "wavefronts per warp-part (two half-warps)" if k != "distinct" else "distinct pairs per warp-part (two half-warps)")


if __name__ == "__main__":
    main()
