"""Generate the golden fixtures under tests/golden/ from the REFERENCE ITSELF.

Runs only in the build container (needs oracle/_ref/libpqtref.so, i.e. the reference sources
compiled in place by oracle/Makefile). For each case it:
  1. draws data with the reference's synth_clustered (bench.cpp:66-95),
  2. builds the index with the reference's IndexBuilder (search.cpp:52-117),
  3. saves it with the reference's save_index (index_io.cpp:94-146) -> <name>.pqt,
  4. records the reference's knn_query_batch outputs (ids, dists, counts, stats), its
     traverse() outputs for the first queries and heuristic_order() prefixes -> <name>.npz.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle.bindings import Ref  # noqa: E402
from paper_1702_05911_b200.index import PqtConfig  # noqa: E402

# name: (config, n, nq, k, blobs, seed)
CASES = {
    "p2_small": (dict(dim=32, p_tree=2, k1=8, k2=4, w=2, p_line=8, hash_size=2048, candidate_budget=256), 4000, 64, 20, 48, 11),
    "p4_small": (dict(dim=32, p_tree=4, k1=8, k2=4, w=2, p_line=8, hash_size=4096, candidate_budget=256), 4000, 64, 20, 48, 12),
    "p1_small": (dict(dim=16, p_tree=1, k1=16, k2=4, w=4, p_line=4, hash_size=1024, candidate_budget=200), 3000, 48, 10, 32, 13),
    "p2_resort": (dict(dim=32, p_tree=2, k1=8, k2=4, w=3, p_line=8, hash_size=1500, candidate_budget=200, resort_bins=True), 4000, 64, 20, 48, 14),
    "p2_wide": (dict(dim=32, p_tree=2, k1=24, k2=4, w=3, p_line=8, hash_size=4096, candidate_budget=256), 4000, 48, 20, 48, 15),
    "p2_sift": (dict(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=512), 5000, 48, 100, 64, 16),
    "p4_gist": (dict(dim=96, p_tree=4, k1=16, k2=8, w=4, p_line=32, candidate_budget=512), 5000, 32, 50, 64, 17),
}
# raw vectors attached (keep_raw build): the exact re-rank stage (search.cpp:229-249) for two k,
# one below rerank_exact and one above it
EXACT_CASES = {
    "p2_exact": (dict(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=512, rerank_exact=48),
                 5000, 40, (20, 80), 64, 18),
}


def make(name: str) -> None:
    cfgd, n, nq, k, blobs, seed = CASES[name]
    cfg = PqtConfig(train_iters=10, seed=seed, **cfgd)
    X = Ref.synth(n + nq, cfg.dim, blobs, 20.0, seed)
    db, Q = X[:n], X[n:]
    ref = Ref.build(db, db, cfg, threads=8)
    path = HERE / f"{name}.pqt"
    ref.save(str(path))
    ref = Ref.load(str(path))  # everything below runs on the loaded index, as in the GPU path
    ids, dists, counts, stats = ref.knn(Q, k, threads=4)
    ntrav = min(nq, 8)
    trav = [ref.traverse(Q[i]) for i in range(ntrav)]
    W = cfg.w * cfg.k2
    orders = [ref.heuristic_order(t["l2_dist"], 4096) for t in trav]
    np.savez_compressed(
        HERE / f"{name}.npz",
        queries=Q, k=np.array(k), ids=ids, dists=dists, counts=counts, stats=stats,
        fine=np.stack([t["fine"] for t in trav]),
        l1_id=np.stack([t["l1_id"] for t in trav]), l1_dist=np.stack([t["l1_dist"] for t in trav]),
        l2_parent=np.stack([t["l2_parent"] for t in trav]), l2_child=np.stack([t["l2_child"] for t in trav]),
        l2_dist=np.stack([t["l2_dist"] for t in trav]),
        order_len=np.array([len(o) for o in orders]),
        orders=np.concatenate(orders, axis=0) if orders else np.zeros((0, cfg.p_tree), np.uint32),
        list_len=np.array(W),
    )
    print(name, "n", n, "bytes", path.stat().st_size, "mean C", stats[:, 1].mean(), "bins", stats[:, 0].mean())


# part counts without a precomputed heuristic (P = 3), or an index stripped of its slope
# tables (P = 2): the reference's exact Dijkstra bin order (binorder.cpp:114-167, :242-244)
ORDER_CASES = {
    "p3_order": (dict(dim=96, p_tree=3, k1=16, k2=8, w=4, p_line=24, hash_size=20000, candidate_budget=512,
                      rerank_exact=0), 6000, 40, 50, 48, 19),
    "p3_order_resort": (dict(dim=48, p_tree=3, k1=8, k2=4, w=3, p_line=12, hash_size=4000, candidate_budget=300,
                             rerank_exact=0, resort_bins=True), 4000, 40, 20, 48, 20),
    "p2_notables": (dict(dim=32, p_tree=2, k1=8, k2=4, w=3, p_line=8, hash_size=2048, candidate_budget=256,
                         rerank_exact=0), 4000, 48, 20, 48, 22),
}


def make_order(name: str) -> None:
    cfgd, n, nq, k, blobs, seed = ORDER_CASES[name]
    cfg = PqtConfig(train_iters=10, seed=seed, **cfgd)
    X = Ref.synth(n + nq, cfg.dim, blobs, 20.0, seed)
    db, Q = X[:n], X[n:]
    ref = Ref.build(db, db, cfg, threads=8)
    if name.endswith("notables"):  # no slope tables in the container: BinStream falls back to exact
        hix = ref.host_index()
        hix.slopes = np.zeros(0, np.float64)
        hix.entries = np.zeros((0, 0, 2), np.uint32)
        hix.__post_init__()
        ref = Ref.from_host(hix)
    path = HERE / f"{name}.pqt"
    ref.save(str(path))
    ref = Ref.load(str(path))
    ids, dists, counts, stats = ref.knn(Q, k, threads=4)
    np.savez_compressed(HERE / f"{name}.npz", queries=Q, k=np.array(k), ids=ids, dists=dists, counts=counts,
                        stats=stats)
    print(name, "n", n, "bytes", path.stat().st_size, "mean C", stats[:, 1].mean(), "bins", stats[:, 0].mean())


def make_exact(name: str) -> None:
    cfgd, n, nq, ks, blobs, seed = EXACT_CASES[name]
    cfg = PqtConfig(train_iters=10, seed=seed, **cfgd)
    X = Ref.synth(n + nq, cfg.dim, blobs, 20.0, seed)
    db, Q = X[:n], X[n:]
    ref = Ref.build(db, db, cfg, threads=8, keep_raw=True)
    path = HERE / f"{name}.pqt"
    ref.save(str(path))  # the container never holds raw vectors (index_io.hpp:9-11)
    out = dict(queries=Q, db=db, ks=np.array(ks))
    for k in ks:
        ids, dists, counts, stats = ref.knn(Q, k, threads=4)
        assert (stats[:, 2] > 0).all(), "exact re-rank did not run"
        out.update({f"ids_k{k}": ids, f"dists_k{k}": dists, f"counts_k{k}": counts, f"stats_k{k}": stats})
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "n", n, "exact_evals", [int(out[f"stats_k{k}"][0, 2]) for k in ks])


def main() -> None:
    names = sys.argv[1:] or list(CASES) + list(EXACT_CASES) + list(ORDER_CASES)
    for name in names:
        (make_exact if name in EXACT_CASES else make_order if name in ORDER_CASES else make)(name)
    (HERE / "CASES.json").write_text(json.dumps({k: dict(config=v[0], n=v[1], nq=v[2], k=v[3], blobs=v[4], seed=v[5])
                                                 for k, v in {**CASES, **EXACT_CASES, **ORDER_CASES}.items()},
                                                indent=1))


if __name__ == "__main__":
    main()
