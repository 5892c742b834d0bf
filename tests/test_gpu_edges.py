"""Edge cases of the query path on the GPU against the REFERENCE itself (oracle/_ref), on
indexes the reference builds (pqtref IndexBuilder, search.cpp:52-117) and writes
(save_index, index_io.cpp:94-146), read by the GPU through pqtg_index_load:

* k1 = 1: the single pair (0, 0) and lambda = 0 (linequant.cpp:72-74, 96-100);
* W = w·k2 = 1 (one child per part list);
* an empty index, n = 0 (search.cpp:130-132);
* candidate budgets above 4096 (8192, 16384; search.cpp:153, 166-217), also with resort_bins,
  whose budget-sized batches (search.cpp:153, 179-190) are then longer than one 4096-tuple chunk
  (heuristic P = 2 and the exact order at P = 3);
* SPEC.md acceptance criterion 2, "full-coverage degeneracy": w = k1, budget >= n,
  rerank_exact >= k  =>  knn_query equals brute_force_knn id for id (n = 5000, D in {16, 64, 128});
* a 1M-vector SIFT-shaped index built by the reference.
"""
import numpy as np
import pytest

from conftest import needs_ref
from paper_1702_05911_b200 import DeviceIndex, PqtConfig, brute_force_knn
from test_gpu_parity import assert_same_results

pytestmark = [pytest.mark.gpu, needs_ref]


def clustered(n, dim, blobs, seed, sigma=20.0):
    rng = np.random.default_rng(seed)
    means = rng.random((blobs, dim), dtype=np.float32) * 255.0
    x = means[rng.integers(0, blobs, n)] + sigma * rng.standard_normal((n, dim), dtype=np.float32)
    return np.ascontiguousarray(x, np.float32)


def ref_index(tmp_path, name, cfg, db, ntrain, keep_raw=False):
    """(path, pqtref handle) of an index the reference builds and saves."""
    from oracle.bindings import Ref

    ref = Ref.build(db[:ntrain] if len(db) else clustered(max(ntrain, 64), cfg.dim, 16, 1), db, cfg,
                    keep_raw=keep_raw)
    path = str(tmp_path / f"{name}.pqt")
    ref.save(path)
    return path, ref


@pytest.mark.parametrize("k1,k2,w", [(1, 8, 1), (4, 1, 1), (1, 1, 1)])
def test_gpu_degenerate_trees(tmp_path, k1, k2, w):
    cfg = PqtConfig(dim=32, p_tree=2, k1=k1, k2=k2, w=w, p_line=8, train_iters=4, seed=3, candidate_budget=512,
                    rerank_exact=0)
    db = clustered(4000, 32, 64, 5)
    Q = clustered(40, 32, 64, 6)
    path, ref = ref_index(tmp_path, f"deg{k1}_{k2}_{w}", cfg, db, 2000)
    dev = DeviceIndex(path)
    for k in (1, 10, 100):
        assert_same_results(dev.search(Q, k), ref.knn(Q, k), f"k1={k1} k2={k2} w={w} k={k}")


def test_gpu_empty_index(tmp_path):
    cfg = PqtConfig(dim=16, p_tree=2, k1=4, k2=2, w=2, p_line=4, train_iters=2, seed=1, candidate_budget=64,
                    rerank_exact=0)
    path, ref = ref_index(tmp_path, "empty", cfg, np.zeros((0, 16), np.float32), 64)
    dev = DeviceIndex(path)
    assert dev.n == 0
    Q = clustered(5, 16, 4, 2)
    ids, dists, counts, stats = dev.search(Q, 10)
    r = ref.knn(Q, 10)
    assert (counts == 0).all() and (r[2] == 0).all()
    assert np.array_equal(stats, r[3])


@pytest.mark.parametrize("budget", [8192, 16384])
def test_gpu_large_budget(tmp_path, budget):
    cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=6, seed=11, candidate_budget=budget,
                    rerank_exact=0)
    db = clustered(60_000, 128, 128, 12)
    Q = clustered(64, 128, 128, 13)
    path, ref = ref_index(tmp_path, f"b{budget}", cfg, db, 20_000)
    dev = DeviceIndex(path)
    for k in (100, 600):
        got = dev.search(Q, k)
        want = ref.knn(Q, k)
        assert_same_results(got, want, f"budget {budget} k={k}")
    assert want[3][:, 1].max() > budget // 2  # the large-budget path (keys in the workspace at 16384) ran


@pytest.mark.parametrize("p_tree,k2,w,budget,resort", [(2, 16, 8, 8192, True), (2, 16, 8, 16384, True),
                                                      (3, 8, 4, 8192, True), (3, 8, 4, 16384, False),
                                                      (2, 32, 8, 65535, True)])
def test_gpu_resort_large_budget(tmp_path, p_tree, k2, w, budget, resort):
    """resort_bins with a batch of `budget` tuples (W^P > budget > 4096): the batch is sorted
    through the workspace (binsel_kernel's merge of 4096-tuple runs) and gathered chunk by chunk.
    The exact order without resort at 16384: the visited set lives in the workspace."""
    dim = 96 if p_tree == 3 else 128
    cfg = PqtConfig(dim=dim, p_tree=p_tree, k1=16, k2=k2, w=w, p_line=dim // 4, train_iters=6, seed=budget + p_tree,
                    candidate_budget=budget, resort_bins=resort, rerank_exact=0)
    db = clustered(max(60_000, budget + 20_000), dim, 128, 21)
    Q = clustered(48, dim, 128, 22)
    path, ref = ref_index(tmp_path, f"rs{p_tree}_{budget}_{resort}", cfg, db, 20_000)
    dev = DeviceIndex(path)
    assert (w * k2) ** p_tree >= budget  # a whole budget-sized batch, several 4096-tuple chunks
    for k in (10, 300):
        got = dev.search(Q, k)
        want = ref.knn(Q, k)
        assert_same_results(got, want, f"resort P={p_tree} budget {budget} k={k}")
    assert want[3][:, 1].max() > 4096  # candidates beyond the first chunk


@pytest.mark.parametrize("dim", [16, 64, 128])
def test_gpu_full_coverage_equals_brute_force(tmp_path, dim):
    """SPEC.md acceptance criterion 2 on the GPU path: w = k1 (every parent), budget >= n (every
    candidate), rerank_exact >= k with the raw vectors attached (the exact stage)."""
    from oracle.bindings import Ref

    n, k = 5000, 10
    cfg = PqtConfig(dim=dim, p_tree=2, k1=8, k2=4, w=8, p_line=8, train_iters=6, seed=dim, candidate_budget=8192,
                    rerank_exact=5000)
    db = clustered(n, dim, 32, dim + 1)
    Q = clustered(20, dim, 32, dim + 2)
    path, ref = ref_index(tmp_path, f"cov{dim}", cfg, db, n, keep_raw=True)
    dev = DeviceIndex(path)
    dev.attach_database(db)
    got = dev.search(Q, k)
    assert_same_results(got, ref.knn(Q, k), f"full coverage D={dim}")
    assert (got[3][:, 1] == n).all() and (got[3][:, 2] == n).all()  # every vector, all exact
    b_ids, b_d, b_c, _ = brute_force_knn(db, Q, k)
    r_ids, r_d = Ref.brute_force(db, Q, k)
    assert np.array_equal(b_ids, r_ids.astype(b_ids.dtype))
    assert np.array_equal(got[0], b_ids)
    assert np.array_equal(got[1].view(np.uint32), b_d.view(np.uint32))


def test_gpu_reference_built_sift1m(tmp_path):
    """A 1M x 128-D SIFT-shaped index (P = 2, k1 = 16, k2 = 8, w = 4, L = 32, H = 4M) built by
    the reference on the CPU, read through pqtg_index_load, 1000 queries bit for bit."""
    from oracle.bindings import Ref

    cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=15, seed=7, candidate_budget=4096)
    db = clustered(1_000_000, 128, 1024, 7)
    Q = clustered(1000, 128, 1024, 8)
    path = str(tmp_path / "sift1m_ref.pqt")
    ref = Ref.build(db[:100_000], db, cfg)
    ref.save(path)
    del db
    dev = DeviceIndex(path, max_batch=1000)
    got = dev.search(Q, 100)
    want = Ref.load(path).knn(Q, 100)
    assert_same_results(got, want, "reference-built SIFT1M")
    assert_same_results(got, ref.knn(Q, 100), "reference-built SIFT1M (in memory)")
