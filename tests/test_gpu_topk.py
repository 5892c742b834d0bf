"""Top-k selection edge cases of the re-rank kernels (search.cpp:229-257) against the C oracle.

* k from 1 to beyond the 512-key wide-select capacity and beyond the block size (bitonic
  fallback), on the golden indexes whose shapes take the fast (i, j)-code re-rank;
* a database of repeated vectors, so thousands of candidates share one distance and the
  wide select's bin overflows (exact 8-bit select fallback); ties resolve by id.
"""
import numpy as np
import pytest

from conftest import GOLDEN, ORDER_CASES, load_golden
from oracle.bindings import Oracle
from paper_1702_05911_b200 import DeviceIndex, PqtConfig, builder
from test_gpu_parity import VARIANTS, assert_same_results

pytestmark = pytest.mark.gpu


@pytest.fixture(params=list(VARIANTS), autouse=True)
def kernel_variant(request):
    from paper_1702_05911_b200._abi import lib

    lib().pqtg_set_kernel_variant(VARIANTS[request.param])
    yield request.param
    lib().pqtg_set_kernel_variant(0)


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist"])
@pytest.mark.parametrize("k", [1, 3, 511, 1500])
def test_gpu_topk_sizes(name, k):
    path = str(GOLDEN / f"{name}.pqt")
    Q = load_golden(name)["queries"][:24]
    got = DeviceIndex(path).search(Q, k)
    want = Oracle(path).knn(Q, k)
    assert_same_results(got, want, f"{name} k={k}")


def test_gpu_topk_repeated_vectors():
    import torch

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=4, seed=9,
                    candidate_budget=4096)
    base = builder.synth_clustered(300, cfg.dim, 8, 20.0, 9, device=dev)
    db = base.repeat(100, 1).contiguous()  # every vector 100 times: equal codes, equal distances
    hix = builder.build_index(db, db[:3000], cfg)
    Q = builder.synth_clustered(16, cfg.dim, 8, 20.0, 10, device=dev).cpu().numpy()
    o = Oracle(hix)
    for k in (100, 700):
        got = DeviceIndex(hix).search(Q, k)
        want = o.knn(Q, k)
        assert_same_results(got, want, f"repeated k={k}")


@pytest.mark.parametrize("budget", [2048, 4096])
def test_gpu_many_small_bins(budget):
    """P = 4 with (k1·k2)^4 > H (the visited set is needed) and bins of about one vector:
    ~2000 / ~4000 bins per query overflow the shared visited sets (binsel_fast: 512 slots,
    binsel_par: 1536) into the global tables."""
    import torch

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=64, p_tree=4, k1=8, k2=8, w=4, p_line=16, train_iters=4, seed=12,
                    hash_size=1 << 17, candidate_budget=budget)
    db = builder.synth_clustered(60_000, cfg.dim, 60_000, 20.0, 12, device=dev)  # ~uniform
    hix = builder.build_index(db, db[:20_000], cfg)
    Q = builder.synth_clustered(24, cfg.dim, 64, 20.0, 13, device=dev).cpu().numpy()
    got = DeviceIndex(hix).search(Q, 50)
    want = Oracle(hix).knn(Q, 50)
    assert_same_results(got, want, "small bins")
    assert (got[3][:, 0] > (600 if budget == 2048 else 1600)).any()  # bins_visited past the shared sets


@pytest.mark.parametrize("k", [10, 100])
def test_gpu_exact_rerank_built_index(k):
    """A GPU-built 200k × 128 index with its raw vectors attached, rerank_exact = 64: the
    exact stage against the C oracle with the same vectors attached."""
    import torch

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=6, seed=21,
                    candidate_budget=2048, rerank_exact=64)
    X = builder.synth_clustered(200_000 + 64, cfg.dim, 256, 20.0, 21, device=dev)
    db, Q = X[:200_000], X[200_000:].cpu().numpy()
    hix = builder.build_index(db, db[:40_000], cfg)
    rows = db.cpu().numpy()
    g = DeviceIndex(hix)
    g.attach_database(rows)
    got = g.search(Q, k)
    o = Oracle(hix)
    o.attach_database(rows)
    want = o.knn(Q, k)
    assert_same_results(got, want, f"exact k={k}")
    assert (got[3][:, 2] == np.minimum(max(64, k), got[3][:, 1])).all()


@pytest.mark.parametrize("k1,p_tree,p_line", [(24, 2, 16), (32, 4, 32)])
def test_gpu_two_byte_pair_codes(k1, p_tree, p_line):
    """16 < k1 <= 32: 2-byte pair ids whose device codes also carry the first centroid
    (v = pid | i << 9, index_prep.cpp) — the fast re-rank (K1M = 32) and the generic one
    against the C oracle on a GPU-built index."""
    import torch

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=p_tree, k1=k1, k2=8, w=4, p_line=p_line, train_iters=4, seed=31 + k1,
                    candidate_budget=1024)
    X = builder.synth_clustered(80_000 + 48, cfg.dim, 128, 20.0, 31, device=dev)
    db, Q = X[:80_000], X[80_000:].cpu().numpy()
    hix = builder.build_index(db, db[:20_000], cfg)
    assert hix.pair_width == 2
    got = DeviceIndex(hix).search(Q, 100)
    want = Oracle(hix).knn(Q, 100)
    assert_same_results(got, want, f"k1={k1}")


@pytest.mark.parametrize("k1,p_tree,p_line,shards", [(24, 2, 16, 4), (32, 4, 32, 8), (32, 4, 32, 3)])
def test_gpu_two_byte_pair_codes_sharded(k1, p_tree, p_line, shards):
    """Position shards of a 2-byte-pair index: with at most a quarter of the lists per shard
    the re-rank computes E per part (rerank_ij DIRECT, no per-query table); merged, the shards
    equal the oracle's unsharded search."""
    import torch

    from paper_1702_05911_b200 import merge_topk_host, shard_range

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=p_tree, k1=k1, k2=8, w=4, p_line=p_line, train_iters=4, seed=61 + k1,
                    candidate_budget=2048)
    X = builder.synth_clustered(90_000 + 40, cfg.dim, 160, 20.0, 61, device=dev)
    db, Q = X[:90_000], X[90_000:].cpu().numpy()
    hix = builder.build_index(db, db[:20_000], cfg)
    want = Oracle(hix).knn(Q, 100)
    parts = [DeviceIndex(hix, shard=shard_range(hix.n, shards, r)).search(Q, 100) for r in range(shards)]
    for part in parts:
        assert np.array_equal(part[3], want[3])
    mi, md, mc = merge_topk_host(np.stack([x[0] for x in parts]), np.stack([x[1] for x in parts]),
                                 np.stack([x[2] for x in parts]))
    assert_same_results((mi, md, mc, want[3]), want, f"k1={k1} shards={shards}")


@pytest.mark.parametrize("p_line", [16, 64])
def test_gpu_line_counts(p_line):
    """The (i, j)-code re-rank at L = 16 and L = 64 (L = 32 is covered by the golden cases)."""
    import torch

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=p_line, train_iters=4, seed=40 + p_line,
                    candidate_budget=1500)
    X = builder.synth_clustered(60_000 + 40, cfg.dim, 96, 20.0, 41, device=dev)
    db, Q = X[:60_000], X[60_000:].cpu().numpy()
    hix = builder.build_index(db, db[:20_000], cfg)
    got = DeviceIndex(hix).search(Q, 64)
    want = Oracle(hix).knn(Q, 64)
    assert_same_results(got, want, f"L={p_line}")


def test_gpu_sharded_index_raw_vectors_are_the_shards_rows():
    """A position shard's attach_database takes its own rows (db[ids[lo:hi]], position order):
    the full set is refused like a mismatched set in the reference (search.cpp:46-48)."""
    from paper_1702_05911_b200 import HostIndex

    path = str(GOLDEN / "p2_exact.pqt")
    g = load_golden("p2_exact")
    hix = HostIndex.load(path)
    shard = DeviceIndex(hix, shard=(0, hix.n // 2))
    with pytest.raises(ValueError):
        shard.attach_database(g["db"])
    shard.attach_database(g["db"][hix.ids[: hix.n // 2].astype(np.int64)])


def test_gpu_sharded_build_equals_full_build():
    """builder.build_index_sharded (two streaming passes, only one shard's ids and codes kept)
    gives, shard by shard, exactly the device index of the full build restricted to the same
    position range; the shards' merged top-k equals the unsharded search."""
    import torch

    from paper_1702_05911_b200 import merge_topk_host

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, train_iters=4, seed=51,
                    candidate_budget=2048, hash_size=1 << 20)
    n, blobs, ntrain, chunk = 300_000, 300, 50_000, 1 << 16
    X = builder.synth_clustered(n, cfg.dim, blobs, 20.0, 51, device=dev, chunk=chunk)
    full = builder.build_index(X, X[:ntrain], cfg)
    Q = builder.synth_queries(40, cfg.dim, blobs, 20.0, 51, 52, device=dev).cpu().numpy()
    k = 50
    want = DeviceIndex(full).search(Q, k)
    parts = []
    for rank in range(3):
        sh = builder.build_index_sharded(n, blobs, 20.0, 51, cfg, 3, rank, ntrain, device=dev, chunk=chunk,
                                         tree=(full.level1, full.level2))
        got = DeviceIndex(sh).search(Q, k)
        ref = DeviceIndex(full, shard=(sh.shard_lo, sh.shard_hi)).search(Q, k)
        assert_same_results(got, ref, f"shard {rank}")
        parts.append(got)
    mi, md, mc = merge_topk_host(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]),
                                 np.stack([p[2] for p in parts]))
    assert_same_results((mi, md, mc, want[3]), want, "merged")


@pytest.mark.parametrize("name", ORDER_CASES)
def test_gpu_exact_bin_order_golden(name):
    """Indexes the reference walks in its exact Dijkstra order (binorder.cpp:114-167): P = 3
    (with and without resort_bins) and a P = 2 container without slope tables. The GPU's heap
    of canonical-parent pushes (kernels.cu exact_fill) against the reference's own outputs."""
    g = load_golden(name)
    dev = DeviceIndex(str(GOLDEN / f"{name}.pqt"))
    got = dev.search(g["queries"], int(g["k"]))
    assert_same_results(got, (g["ids"], g["dists"], g["counts"], g["stats"]), name)


def test_gpu_exact_bin_order_built_index():
    """A GPU-built P = 3 index at budget 4096 (a deep heap) against the reference compiled in
    place, run on the same index."""
    import torch

    from oracle.bindings import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=96, p_tree=3, k1=16, k2=8, w=4, p_line=24, train_iters=4, seed=71, candidate_budget=4096,
                    rerank_exact=0)
    X = builder.synth_clustered(60_000 + 64, cfg.dim, 256, 20.0, 71, device=dev)
    db, Q = X[:60_000], X[60_000:].cpu().numpy()
    hix = builder.build_index(db, db[:20_000], cfg)
    got = DeviceIndex(hix).search(Q, 100)
    want = Ref.from_host(hix).knn(Q, 100)
    assert_same_results(got, want, "p3 built")
    assert (got[3][:, 1] == 4096).all()


@pytest.mark.parametrize("n,dim,k", [(5000, 128, 100), (3000, 30, 20), (50, 16, 100), (4000, 96, 0)])
def test_gpu_brute_force_knn(n, dim, k):
    """pqt::brute_force_knn (search.cpp:276-299) on the GPU against the reference's own, bit for
    bit: unaligned dim, n < k, k = 0, and repeated rows (ties broken by id)."""
    from oracle.bindings import Ref

    from paper_1702_05911_b200 import brute_force_knn

    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(n + dim)
    db = (rng.standard_normal((n, dim)) * 10).astype(np.float32)
    db[n // 2:n // 2 + 7] = db[3]  # duplicates: equal distances, order by id
    Q = (rng.standard_normal((24, dim)) * 10).astype(np.float32)
    Q[0] = db[3]
    ids, dists, counts, stats = brute_force_knn(db, Q, k)
    assert (counts == min(k, n)).all()
    if k and n:
        assert (stats[:, 1] == n).all() and (stats[:, 2] == n).all()
        r_ids, r_d = Ref.brute_force(db, Q, k)
        c = min(k, n)
        assert np.array_equal(ids[:, :c], r_ids[:, :c])
        assert np.array_equal(dists[:, :c].view(np.uint32), r_d[:, :c].view(np.uint32))
        assert ids[0, 0] == 3 and dists[0, 0] == 0.0


def test_gpu_brute_force_device_entry_point():
    """pqtg_brute_force_knn_device (device buffers, caller stream; what bench.py's recall uses)
    equals the host entry point."""
    import torch

    from paper_1702_05911_b200 import brute_force_knn
    from paper_1702_05911_b200._abi import check, lib

    rng = np.random.default_rng(5)
    db = rng.standard_normal((7000, 96)).astype(np.float32)
    Q = rng.standard_normal((33, 96)).astype(np.float32)
    k = 17
    ids, dists, counts, _ = brute_force_knn(db, Q, k)
    d_db, d_q = torch.from_numpy(db).cuda(), torch.from_numpy(Q).cuda()
    d_i = torch.empty((33, k), dtype=torch.int32, device="cuda")
    d_d = torch.empty((33, k), dtype=torch.float32, device="cuda")
    d_c = torch.empty(33, dtype=torch.int32, device="cuda")
    check(lib().pqtg_brute_force_knn_device(d_db.data_ptr(), 7000, 96, d_q.data_ptr(), 33, k, d_i.data_ptr(),
                                            d_d.data_ptr(), d_c.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(d_i.cpu().numpy().view(np.uint32), ids)
    assert np.array_equal(d_d.cpu().numpy().view(np.uint32), dists.view(np.uint32))
    assert np.array_equal(d_c.cpu().numpy().view(np.uint32), counts)


def test_gpu_sift1b_tree_small():
    """The SIFT1B tree (P = 4, k1 = 32, k2 = 16, w = 8: W = 128, 2-byte pair codes, H = 2^20) on a
    GPU-built 80k index: the wide warp-per-part traversal, the partial pair-stream fold and the
    K1M = 32 re-rank against the C oracle, unsharded and as 8 position shards merged."""
    import torch

    from paper_1702_05911_b200 import merge_topk_host, shard_range

    dev = torch.device("cuda", 0)
    cfg = PqtConfig(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, train_iters=4, seed=81, candidate_budget=2048,
                    hash_size=1 << 20, rerank_exact=0)
    X = builder.synth_clustered(80_000 + 40, cfg.dim, 400, 20.0, 81, device=dev)
    db, Q = X[:80_000], X[80_000:].cpu().numpy()
    hix = builder.build_index(db, db[:30_000], cfg)
    want = Oracle(hix).knn(Q, 100)
    assert_same_results(DeviceIndex(hix).search(Q, 100), want, "sift1b tree")
    parts = [DeviceIndex(hix, shard=shard_range(hix.n, 8, r)).search(Q, 100) for r in range(8)]
    mi, md, mc = merge_topk_host(np.stack([x[0] for x in parts]), np.stack([x[1] for x in parts]),
                                 np.stack([x[2] for x in parts]))
    assert_same_results((mi, md, mc, want[3]), want, "sift1b tree, 8 shards")

