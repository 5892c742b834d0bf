"""The C oracle's position-shard view (pqto_from_shard_view: whole-index offsets, the shard's
ids and its line codes in position order, as a sharded GPU deployment holds them) is the
checker of the SIFT1B-scale shard in bench.py. Pinned here: its local top-k equals the
whole-index oracle restricted to the same positions, and merging the shards' lists by
(dist, id) (candidate_less, search.cpp:39-41) gives the unsharded answer."""
import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle.bindings import Oracle
from paper_1702_05911_b200.builder import ShardIndex
from paper_1702_05911_b200.index import HostIndex


def shard_of(hix: HostIndex, lo: int, hi: int) -> ShardIndex:
    ids = np.ascontiguousarray(hix.ids[lo:hi])
    return ShardIndex(hix.config, hix.n, hix.level1, hix.level2, hix.d2, hix.slopes, hix.entries, hix.offsets,
                      lo, hi, ids, np.ascontiguousarray(hix.lambda_q.reshape(hix.n, -1)[ids]),
                      np.ascontiguousarray(hix.pair_id.reshape(hix.n, -1)[ids]))


def merge(parts, k):
    nq = parts[0][0].shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dists = np.zeros((nq, k), np.float32)
    counts = np.zeros(nq, np.uint32)
    for q in range(nq):
        c = [(float(p[1][q, j]), int(p[0][q, j])) for p in parts for j in range(p[2][q])]
        c.sort()
        c = c[:k]
        counts[q] = len(c)
        for j, (d, i) in enumerate(c):
            ids[q, j], dists[q, j] = i, d
    return ids, dists, counts


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p2_wide"])
@pytest.mark.parametrize("shards", [2, 3])
def test_oracle_shard_view(name, shards):
    hix = HostIndex.load(str(GOLDEN / f"{name}.pqt"))
    g = load_golden(name)
    Q, k = g["queries"][:32], int(g["k"])
    whole = Oracle(hix)
    parts = []
    for r in range(shards):
        lo, hi = hix.n * r // shards, hix.n * (r + 1) // shards
        got = Oracle(shard_of(hix, lo, hi)).knn(Q, k)
        want = whole.knn(Q, k, shard=(lo, hi))
        for a, b in zip(got, want):
            assert np.array_equal(a, b), f"{name} shard {r}"
        parts.append(got)
    mi, md, mc = merge(parts, k)
    ref = (g["ids"][:32], g["dists"][:32], g["counts"][:32])
    assert np.array_equal(mc, ref[2])
    for q in range(len(mc)):
        c = mc[q]
        assert np.array_equal(mi[q, :c], ref[0][q, :c]) and np.array_equal(md[q, :c], ref[1][q, :c])
