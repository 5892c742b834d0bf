"""CUDA path vs the reference (golden fixtures) and vs the C oracle, through the C-ABI.

Bar: candidate positions, bins_visited, candidates, neighbour ids and distances all
bit-exact (the kernels follow the reference's fp32 operation order; the only documented
near-tie class is pick_slope_table's fp64 log rounding, never hit at these shapes)."""
import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, load_golden
from oracle.bindings import Oracle
from paper_1702_05911_b200 import DeviceIndex, HostIndex, knn_query_batch, merge_topk_host, shard_range

pytestmark = pytest.mark.gpu


VARIANTS = {"auto": 0, "generic": 1, "tc_screen": 2, "walker_binsel": 3, "allwarp_binsel": 4}


@pytest.fixture(params=list(VARIANTS), autouse=True)
def kernel_variant(request):
    """Run every GPU parity test through the fast kernels and through the generic ones."""
    from paper_1702_05911_b200._abi import lib

    lib().pqtg_set_kernel_variant(VARIANTS[request.param])
    yield request.param
    lib().pqtg_set_kernel_variant(0)


def assert_same_results(a, b, ctx=""):
    ids_a, d_a, c_a, s_a = a
    ids_b, d_b, c_b, s_b = b
    assert np.array_equal(c_a, c_b), ctx + " counts"
    assert np.array_equal(s_a, s_b), ctx + " stats"
    for q in range(len(c_a)):
        c = c_a[q]
        assert np.array_equal(ids_a[q, :c], ids_b[q, :c]), f"{ctx} ids q={q}"
        assert np.array_equal(d_a[q, :c].view(np.uint32), d_b[q, :c].view(np.uint32)), f"{ctx} dists q={q}"


@pytest.mark.parametrize("name", GOLDEN_CASES)
@pytest.mark.parametrize("source", ["file", "view"])
def test_gpu_matches_reference_golden(name, source):
    g = load_golden(name)
    path = str(GOLDEN / f"{name}.pqt")
    dev = DeviceIndex(path if source == "file" else HostIndex.load(path))
    k = int(g["k"])
    got = dev.search(g["queries"], k)
    assert_same_results(got, (g["ids"], g["dists"], g["counts"], g["stats"]), name)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_gpu_stages_match_reference(name, kernel_variant):
    """Per stage: traversal LUT + level-2 lists, slope pick, gathered candidate positions.

    With the tensor-core screen (variant "tc_screen") the level-2 lists' ORDER and their first two
    distances are the reference's bits (the rest are screened values: bin selection reads only
    ranks and the first two distances); the other variants compute every distance exactly."""
    g = load_golden(name)
    path = str(GOLDEN / f"{name}.pqt")
    dev = DeviceIndex(path)
    o = Oracle(path)
    Q = g["queries"]
    dev.search(Q, int(g["k"]))
    inter = dev.intermediates(len(Q))
    screened = kernel_variant == "tc_screen" and not o.config.resort_bins
    for i in range(len(Q)):
        t = o.traverse(Q[i]) if i >= g["fine"].shape[0] else {k: g[k][i] for k in ("fine", "l2_parent", "l2_child",
                                                                                  "l2_dist")}
        assert np.array_equal(inter["fine"][i].view(np.uint32), t["fine"].view(np.uint32)), f"q={i}"
        assert np.array_equal(inter["l2_parent"][i], t["l2_parent"]), f"q={i}"
        assert np.array_equal(inter["l2_child"][i], t["l2_child"]), f"q={i}"
        got, want = inter["l2_dist"][i], t["l2_dist"]
        if screened:
            assert np.array_equal(got[:, :2].view(np.uint32), want[:, :2].view(np.uint32)), f"q={i}"
            assert np.allclose(got, want, rtol=1e-3, atol=1e-3), f"q={i}"
        else:
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"q={i}"
    for i in range(len(Q)):
        pos, bins = o.candidates(Q[i])
        assert np.array_equal(inter["positions"][i], pos), f"q={i}"
        assert int(g["stats"][i, 0]) == bins


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p2_wide"])
@pytest.mark.parametrize("shards", [2, 3])
def test_gpu_sharded_merge_equals_unsharded(name, shards):
    g = load_golden(name)
    path = str(GOLDEN / f"{name}.pqt")
    k = int(g["k"])
    n = HostIndex.load(path).n
    parts = []
    for r in range(shards):
        lo, hi = shard_range(n, shards, r)
        dev = DeviceIndex(path, shard=(lo, hi))
        parts.append(dev.search(g["queries"], k))
    ids = np.stack([p[0] for p in parts])
    dists = np.stack([p[1] for p in parts])
    counts = np.stack([p[2] for p in parts])
    for p in parts:  # bin selection is global on every shard
        assert np.array_equal(p[3], g["stats"])
    mi, md, mc = merge_topk_host(ids, dists, counts)
    assert_same_results((mi, md, mc, g["stats"]), (g["ids"], g["dists"], g["counts"], g["stats"]), name)


def test_gpu_edge_cases():
    path = str(GOLDEN / "p2_small.pqt")
    g = load_golden("p2_small")
    dev = DeviceIndex(path)
    Q = g["queries"]
    o = Oracle(path)
    # k == 0 -> empty results and zero stats (search.cpp:130-132)
    ids, d, c, s = dev.search(Q, 0)
    assert (c == 0).all() and (s == 0).all()
    # k larger than the candidate count -> short results (search.cpp:251)
    got = dev.search(Q, 1000)
    want = o.knn(Q, 1000)
    assert_same_results(got, want, "k>C")
    assert (got[2] <= got[3][:, 1]).all()
    # dists non-decreasing
    for q in range(len(Q)):
        dd = got[1][q, : got[2][q]]
        assert (np.diff(dd) >= 0).all()
    # empty batch
    ids, d, c, s = dev.search(Q[:0], 10)
    assert c.shape == (0,)
    # dimension mismatch -> ValueError (std::invalid_argument)
    with pytest.raises(ValueError):
        dev.search(np.zeros((2, 31), np.float32), 5)
    # a query equal to a database vector: reference-identical answer
    hix = HostIndex.load(path)
    assert hix.n == 4000


def test_gpu_knn_query_batch_api():
    path = str(GOLDEN / "p4_small.pqt")
    g = load_golden("p4_small")
    dev = DeviceIndex(path)
    res = knn_query_batch(dev, g["queries"], int(g["k"]))
    for q, r in enumerate(res):
        c = g["counts"][q]
        assert np.array_equal(r.ids, g["ids"][q, :c])
        assert r.stats.bins_visited == g["stats"][q, 0]
        assert r.stats.candidates == g["stats"][q, 1]


def test_gpu_batching_is_deterministic():
    """Sub-batching (max_batch) and repeated runs give identical results."""
    path = str(GOLDEN / "p4_gist.pqt")
    g = load_golden("p4_gist")
    Q = np.concatenate([g["queries"]] * 5)
    a = DeviceIndex(path, max_batch=7).search(Q, 50)
    b = DeviceIndex(path, max_batch=4096).search(Q, 50)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("chunks", [1, 2, 3, 0])
def test_gpu_chunked_searches_identical(chunks):
    """Chunked two-stream searches (host and device entry points) return the reference's results."""
    import torch

    g = load_golden("p4_gist")
    Q = np.concatenate([g["queries"]] * 9)  # 288 queries -> auto picks 2 chunks
    k = int(g["k"])
    dev = DeviceIndex(str(GOLDEN / "p4_gist.pqt"), max_batch=300)
    dev.set_chunks(chunks)
    host = dev.search(Q, k)
    n = len(g["queries"])
    for r in range(9):
        sl = slice(r * n, (r + 1) * n)
        assert_same_results(tuple(x[sl] for x in host), (g["ids"], g["dists"], g["counts"], g["stats"]), "host")
    dq = torch.from_numpy(Q).cuda()
    d_ids = torch.empty((len(Q), k), dtype=torch.int32, device="cuda")
    d_d = torch.empty((len(Q), k), dtype=torch.float32, device="cuda")
    d_c = torch.empty(len(Q), dtype=torch.int32, device="cuda")
    d_s = torch.empty((len(Q), 3), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    dev.search_device(dq.data_ptr(), len(Q), k, d_ids.data_ptr(), d_d.data_ptr(), d_c.data_ptr(), d_s.data_ptr(),
                      stream.cuda_stream)
    torch.cuda.synchronize()
    got = (d_ids.cpu().numpy().view(np.uint32), d_d.cpu().numpy(), d_c.cpu().numpy().view(np.uint32),
           d_s.cpu().numpy().view(np.uint64))
    for x, y in zip(got, host):
        assert np.array_equal(x, y)


def test_gpu_exact_rerank_matches_reference_golden():
    """Raw vectors attached (pqtg_index_attach_database): K5 keeps the max(k, rerank_exact)
    line-ranked prefix, K6 re-ranks it by exact l2_sq — bit-exact against the reference's
    keep_raw build (search.cpp:229-249), for k below and above rerank_exact."""
    from test_oracle_golden import _check_exact

    g = load_golden("p2_exact")
    dev = DeviceIndex(str(GOLDEN / "p2_exact.pqt"))
    dev.attach_database(g["db"])
    for k in g["ks"]:
        _check_exact(dev.search(g["queries"], int(k)), g, int(k), f"k={k}")
    with pytest.raises(ValueError):
        dev.attach_database(g["db"][:, :-1])
    dev.attach_database(None)
    ids, d, c, s = dev.search(g["queries"], 20)
    assert (s[:, 2] == 0).all()
    want = Oracle(str(GOLDEN / "p2_exact.pqt")).knn(g["queries"], 20)
    assert_same_results((ids, d, c, s), want, "detached")


def test_gpu_pinned_search_graph_replays():
    """pqtg_search on page-locked buffers runs as a replayed CUDA graph: same results as the
    direct path, also when the buffers' contents change between replays."""
    import torch

    from paper_1702_05911_b200._abi import check, lib

    path = str(GOLDEN / "p4_gist.pqt")
    g = load_golden("p4_gist")
    Q = g["queries"]
    k = int(g["k"])
    dev = DeviceIndex(path)
    nq, dim = Q.shape
    hq = torch.from_numpy(Q.copy()).pin_memory()
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    h_c = torch.empty(nq, dtype=torch.int32).pin_memory()
    h_s = torch.empty((nq, 3), dtype=torch.int64).pin_memory()

    def run():
        check(lib().pqtg_search(dev.handle, dev.workspace, hq.data_ptr(), nq, dim, k, h_ids.data_ptr(),
                                h_d.data_ptr(), h_c.data_ptr(), h_s.data_ptr()))
        return (h_ids.numpy().view(np.uint32).copy(), h_d.numpy().copy(), h_c.numpy().view(np.uint32).copy(),
                h_s.numpy().view(np.uint64).copy())

    want = Oracle(path).knn(Q, k)
    for _ in range(3):  # capture, then replays
        assert_same_results(run(), want, "pinned")
    Q2 = Q[::-1].copy()
    hq.copy_(torch.from_numpy(Q2))
    assert_same_results(run(), Oracle(path).knn(Q2, k), "pinned, new contents")
