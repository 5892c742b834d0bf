"""The query-partitioned sharded search (include/pqtg.h "sharded search", csrc/sharded.cpp)
against the unsharded answer, bit for bit.

* LocalShardedIndex: G position shards driven by one process on one GPU (the local transport:
  the same protocol -- block traversal + bin selection, range-list all-gather, per-shard
  re-rank, all-to-all, merge, result all-gather -- with device copies), G in {2, 3, 8}, batches
  not divisible by G and smaller than G, device and host entry points;
* ShardedIndex over a one-rank NCCL communicator (libpqtg's own, id from pqtg_nccl_unique_id);
* the SIFT1B tree (P = 4, k1 = 32, W = 128, 2-byte pair codes) over 8 shards.
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_golden
from oracle.bindings import Oracle
from paper_1702_05911_b200 import DeviceIndex, PqtConfig, builder
from paper_1702_05911_b200.sharded import LocalShardedIndex, ShardedIndex
from test_gpu_parity import assert_same_results

pytestmark = pytest.mark.gpu


def run_local(lsi: LocalShardedIndex, Q: np.ndarray, k: int, broadcast: bool):
    nq = Q.shape[0]
    G = lsi.world
    dq = [torch.from_numpy(Q).cuda() if (g == 0 or not broadcast) else None for g in range(G)]
    ids = [torch.full((nq, max(k, 1)), -7, dtype=torch.int32, device="cuda") for _ in range(G)]
    d = [torch.full((nq, max(k, 1)), -7.0, dtype=torch.float32, device="cuda") for _ in range(G)]
    c = [torch.full((nq,), -7, dtype=torch.int32, device="cuda") for _ in range(G)]
    st = [torch.full((nq, 3), -7, dtype=torch.int64, device="cuda") for _ in range(G)]
    lsi.search(dq, k, ids, d, c, st, broadcast=broadcast)
    torch.cuda.synchronize()
    return [(ids[g].cpu().numpy().view(np.uint32)[:, :k], d[g].cpu().numpy()[:, :k],
             c[g].cpu().numpy().view(np.uint32), st[g].cpu().numpy().view(np.uint64)) for g in range(G)]


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p2_wide", "p2_small"])
@pytest.mark.parametrize("shards", [2, 3, 8])
def test_local_sharded_equals_unsharded(name, shards):
    g = load_golden(name)
    path = str(GOLDEN / f"{name}.pqt")
    k = int(g["k"])
    want = (g["ids"], g["dists"], g["counts"], g["stats"])
    lsi = LocalShardedIndex(path, shards, max_batch=64)
    for bcast in (False, True):
        for r, got in enumerate(run_local(lsi, g["queries"], k, bcast)):
            assert_same_results(got, want, f"{name} G={shards} rank {r} bcast={bcast}")
    # a batch smaller than G (empty query blocks) and a different k
    Q = g["queries"][:5]
    w5 = DeviceIndex(path).search(Q, 7)
    for got in run_local(lsi, Q, 7, False):
        assert_same_results(got, w5, f"{name} G={shards} nq=5")
    # the host entry point (pqtg_sharded_search)
    assert_same_results(lsi.search_host(g["queries"], k), want, f"{name} G={shards} host")
    # k = 0: empty results, zero stats (search.cpp:130-132)
    got = lsi.search_host(g["queries"], 0)
    assert (got[2] == 0).all() and (got[3] == 0).all()


def test_nccl_one_rank():
    """ShardedIndex over libpqtg's own NCCL communicator of one rank (no torch process group
    needed): every collective of the protocol runs, with the rank as its own peer."""
    g = load_golden("p4_gist")
    path = str(GOLDEN / "p4_gist.pqt")
    k = int(g["k"])
    sh = ShardedIndex(path, device=0, max_batch=64)
    dq = torch.from_numpy(g["queries"]).cuda()
    nq = dq.shape[0]
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    c = torch.empty(nq, dtype=torch.int32, device="cuda")
    st = torch.empty((nq, 3), dtype=torch.int64, device="cuda")
    sh.search(dq, k, ids, d, c, st)
    torch.cuda.synchronize()
    got = (ids.cpu().numpy().view(np.uint32), d.cpu().numpy(), c.cpu().numpy().view(np.uint32),
           st.cpu().numpy().view(np.uint64))
    assert_same_results(got, (g["ids"], g["dists"], g["counts"], g["stats"]), "nccl x1")
    assert len(sh.stage_ms()) == 4


def test_local_sharded_sift1b_tree():
    """The SIFT1B tree on a GPU-built 80k index over 8 shards (K1M = 32 re-rank, DIRECT on
    shards holding <= 1/4 of the lists) against the C oracle on the whole index."""
    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, train_iters=4, seed=81, candidate_budget=2048,
                    hash_size=1 << 20, rerank_exact=0)
    X = builder.synth_clustered(80_000 + 40, cfg.dim, 400, 20.0, 81, device=dev)
    db, Q = X[:80_000], X[80_000:].cpu().numpy()
    hix = builder.build_index(db, db[:30_000], cfg)
    want = Oracle(hix).knn(Q, 100)
    lsi = LocalShardedIndex(hix, 8, max_batch=64)
    for r, got in enumerate(run_local(lsi, Q, 100, True)):
        assert_same_results(got, want, f"sift1b tree G=8 rank {r}")


@pytest.mark.parametrize("split,cluster", [("0", "1"), ("1", "1"), ("1", "0")])
def test_gpu_split_rerank_switch(split, cluster):
    """The small-batch split re-rank (default; PQTG_SPLIT=0 turns it off: each query's candidates
    over up to 16 CTAs whose sorted lists meet in one slice -- through distributed shared memory
    when the slices form a cluster, through global memory and an arrival counter with
    PQTG_SPLIT_CLUSTER=0) and the one-CTA-per-query re-rank against the golden fixtures, in a fresh
    process (the switches are read once)."""
    import subprocess
    import sys

    code = (
        "import numpy as np\n"
        "from conftest import GOLDEN, load_golden\n"
        "from test_gpu_parity import assert_same_results\n"
        "from paper_1702_05911_b200 import DeviceIndex\n"
        "for name in ['p2_sift', 'p4_gist', 'p2_wide']:\n"
        "    g = load_golden(name)\n"
        "    dev = DeviceIndex(str(GOLDEN / f'{name}.pqt'))\n"
        "    for nq in (1, 5, len(g['queries'])):\n"
        "        got = dev.search(g['queries'][:nq], int(g['k']))\n"
        "        assert_same_results(got, tuple(x[:nq] for x in (g['ids'], g['dists'], g['counts'], g['stats'])), name)\n"
        "print('ok')\n")
    import os
    from conftest import REPO

    env = dict(os.environ, PQTG_SPLIT=split, PQTG_SPLIT_CLUSTER=cluster, PYTHONPATH=f"{REPO}:{REPO / 'tests'}")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=str(REPO / "tests"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("shards", [2, 3, 8])
@pytest.mark.parametrize("k", [20, 80])
def test_local_sharded_exact_rerank(shards, k):
    """The exact stage across position shards (search.cpp:229-249): each shard re-ranks its own
    line prefix with its own raw rows and ships (id, line, exact) triples; the merge cuts the
    global prefix min(max(rerank_exact, k), C) by (line, id) and ranks it by (exact, id) --
    bit-exact against the reference's keep_raw build (golden p2_exact), exact_evals included."""
    from paper_1702_05911_b200 import HostIndex

    g = load_golden("p2_exact")
    path = str(GOLDEN / "p2_exact.pqt")
    hix = HostIndex.load(path)
    lsi = LocalShardedIndex(path, shards, max_batch=64)
    lsi.attach_database(g["db"], hix.ids)
    want = (g[f"ids_k{k}"], g[f"dists_k{k}"], g[f"counts_k{k}"], g[f"stats_k{k}"])
    for r, got in enumerate(run_local(lsi, g["queries"], k, True)):
        assert_same_results(got, want, f"exact G={shards} k={k} rank {r}")
    assert_same_results(lsi.search_host(g["queries"], k), want, f"exact G={shards} k={k} host")


def test_shard_exact_outside_the_sharded_search_is_refused():
    from paper_1702_05911_b200 import HostIndex, shard_range

    g = load_golden("p2_exact")
    path = str(GOLDEN / "p2_exact.pqt")
    hix = HostIndex.load(path)
    lo, hi = shard_range(hix.n, 2, 1)
    dev = DeviceIndex(path, shard=(lo, hi))
    dev.attach_database(g["db"][hix.ids[lo:hi].astype(np.int64)])
    with pytest.raises(Exception, match="sharded search"):
        dev.search(g["queries"], 20)


def test_gpu_fixed_slots_without_bank_map():
    """PQTG_BANK_MAP=0: the 1-byte line codes keep the fixed slots t = i << 4 | ((i + j) & 15)
    instead of the per-part bank map learned at upload; same results (fresh process: the switch
    is read once)."""
    import os
    import subprocess
    import sys

    from conftest import REPO

    code = (
        "from conftest import GOLDEN, load_golden\n"
        "from test_gpu_parity import assert_same_results\n"
        "from paper_1702_05911_b200 import DeviceIndex\n"
        "for name in ['p2_sift', 'p4_gist', 'p2_wide', 'p2_small']:\n"
        "    g = load_golden(name)\n"
        "    dev = DeviceIndex(str(GOLDEN / f'{name}.pqt'))\n"
        "    for nq in (1, len(g['queries'])):\n"
        "        got = dev.search(g['queries'][:nq], int(g['k']))\n"
        "        assert_same_results(got, tuple(x[:nq] for x in (g['ids'], g['dists'], g['counts'], g['stats'])), name)\n"
        "print('ok')\n")
    env = dict(os.environ, PQTG_BANK_MAP="0", PYTHONPATH=f"{REPO}:{REPO / 'tests'}")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=str(REPO / "tests"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_local_sharded_bank_mapped_codes():
    """k1 = 16 shards large enough for the per-part bank map (index_prep.cpp bank_map, learned
    from each shard's own positions) against the unsharded index, bit for bit."""
    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=96, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=4, seed=5, candidate_budget=2048,
                    rerank_exact=0)
    X = builder.synth_clustered(60_000 + 64, cfg.dim, 60, 20.0, 5, device=dev)
    db, Q = X[:60_000], X[60_000:].cpu().numpy()
    hix = builder.build_index(db, db[:20_000], cfg)
    want = DeviceIndex(hix).search(Q, 50)
    assert_same_results(want, Oracle(hix).knn(Q, 50), "unsharded vs oracle")
    lsi = LocalShardedIndex(hix, 2, max_batch=64)
    for r, got in enumerate(run_local(lsi, Q, 50, True)):
        assert_same_results(got, want, f"bank-mapped shards rank {r}")
