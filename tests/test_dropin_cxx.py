"""The C++ drop-in (include/pqt/*.hpp over libpqtg.so) used the way reference callers use
pqt::load_index / save_index / knn_query_batch / knn_query."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, REPO, load_golden
from paper_1702_05911_b200._abi import LIB_PATH


@pytest.fixture(scope="module")
def dropin_bin(tmp_path_factory):
    out = tmp_path_factory.mktemp("cxx") / "dropin_main"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(REPO / "include"), str(REPO / "tests/cxx/dropin_main.cpp"),
                    "-o", str(out), str(LIB_PATH), f"-Wl,-rpath,{LIB_PATH.parent}"], check=True)
    return out


@pytest.mark.parametrize("name", ["p2_small", "p4_gist", "p2_wide"])
def test_cxx_load_save_byte_identical(dropin_bin, name, tmp_path):
    src = GOLDEN / f"{name}.pqt"
    copy = tmp_path / "copy.pqt"
    subprocess.run([str(dropin_bin), "io", str(src), str(copy)], check=True, capture_output=True)
    assert copy.read_bytes() == src.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["query", "sharded"])
@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p1_small", "p2_resort"])
def test_cxx_knn_query_batch_matches_reference(dropin_bin, name, mode, tmp_path):
    """pqt::knn_query_batch, and pqt::ShardedIndex::knn_query_batch over a one-rank NCCL
    communicator (pqtg_sharded_*: the whole protocol with the rank as its own peer)."""
    if mode == "sharded" and name == "p2_resort":
        pytest.skip("resort_bins index: covered by the query mode")
    g = load_golden(name)
    qf = tmp_path / "q.f32"
    g["queries"].astype(np.float32).tofile(qf)
    out = tmp_path / "out.bin"
    k = int(g["k"])
    r = subprocess.run([str(dropin_bin), mode, str(GOLDEN / f"{name}.pqt"), str(qf), str(g["queries"].shape[1]),
                        str(k), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    buf = out.read_bytes()
    pos = 0
    for q in range(g["queries"].shape[0]):
        c = int(np.frombuffer(buf, np.uint32, 1, pos)[0])
        st = np.frombuffer(buf, np.uint64, 3, pos + 4)
        ids = np.frombuffer(buf, np.uint32, c, pos + 28)
        d = np.frombuffer(buf, np.float32, c, pos + 28 + 4 * c)
        pos += 28 + 8 * c
        assert c == g["counts"][q]
        assert np.array_equal(st, g["stats"][q])
        assert np.array_equal(ids, g["ids"][q, :c])
        assert np.array_equal(d.view(np.uint32), g["dists"][q, :c].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [20, 80])
def test_cxx_attach_database_exact_rerank(dropin_bin, k, tmp_path):
    """PqtIndex::attach_database through the C++ drop-in: the exact re-rank stage on the GPU,
    bit-exact against the reference's keep_raw build (golden p2_exact)."""
    g = load_golden("p2_exact")
    qf, dbf, out = tmp_path / "q.f32", tmp_path / "db.f32", tmp_path / "out.bin"
    g["queries"].astype(np.float32).tofile(qf)
    g["db"].astype(np.float32).tofile(dbf)
    r = subprocess.run([str(dropin_bin), "query", str(GOLDEN / "p2_exact.pqt"), str(qf), str(g["queries"].shape[1]),
                        str(k), str(out), str(dbf)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    buf = out.read_bytes()
    pos = 0
    for q in range(g["queries"].shape[0]):
        c = int(np.frombuffer(buf, np.uint32, 1, pos)[0])
        st = np.frombuffer(buf, np.uint64, 3, pos + 4)
        ids = np.frombuffer(buf, np.uint32, c, pos + 28)
        d = np.frombuffer(buf, np.float32, c, pos + 28 + 4 * c)
        pos += 28 + 8 * c
        assert c == g[f"counts_k{k}"][q]
        assert np.array_equal(st, g[f"stats_k{k}"][q])
        assert np.array_equal(ids, g[f"ids_k{k}"][q, :c])
        assert np.array_equal(d.view(np.uint32), g[f"dists_k{k}"][q, :c].view(np.uint32))


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p1_small", "p2_wide", "p3_order"])
def test_cxx_stage_functions_match_reference(dropin_bin, name, tmp_path):
    """The per-stage public functions a reference caller may use directly -- traverse
    (pqtree.hpp:56-79), pick_slope_table / heuristic_order / dijkstra_order / build_slope_tables
    (binorder.hpp), decode_pair / line_distance (linequant.hpp) -- through the C++ drop-in,
    against the reference compiled in place, bit for bit."""
    from oracle.bindings import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    path = str(GOLDEN / f"{name}.pqt")
    g = load_golden(name)
    Q = g["queries"][:6].astype(np.float32)
    qf, out = tmp_path / "q.f32", tmp_path / "stages.bin"
    Q.tofile(qf)
    max_bins = 300
    r = subprocess.run([str(dropin_bin), "stages", path, str(qf), str(Q.shape[1]), str(max_bins), str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    ref = Ref.load(path)
    c = ref.config
    W, P = c.w * c.k2, c.p_tree
    hix = ref.host_index()
    buf, pos = out.read_bytes(), 0

    def take(dtype, n):
        nonlocal pos
        a = np.frombuffer(buf, dtype, n, pos)
        pos += a.nbytes
        return a

    for y in Q:
        want = ref.traverse(y)
        assert np.array_equal(take(np.float32, c.p_line * c.k1), want["fine"].reshape(-1).view(np.float32))
        l1 = take(np.uint32, 2 * P * c.k1).reshape(P, c.k1, 2)
        assert np.array_equal(l1[:, :, 0], want["l1_id"]) and np.array_equal(l1[:, :, 1], want["l1_dist"].view(np.uint32))
        l2 = take(np.uint32, 3 * P * W).reshape(P, W, 3)
        assert np.array_equal(l2[:, :, 0], want["l2_parent"]) and np.array_equal(l2[:, :, 1], want["l2_child"])
        assert np.array_equal(l2[:, :, 2], want["l2_dist"].view(np.uint32))
        slope = int(take(np.uint32, 1)[0])
        if P >= 2:
            assert slope == Ref.pick_slope_table(want["l2_dist"][0], want["l2_dist"][1])
        for fn in (lambda: ref.heuristic_order(want["l2_dist"], max_bins), lambda: Ref.dijkstra_order(want["l2_dist"], max_bins)):
            cnt = int(take(np.uint32, 1)[0])
            assert np.array_equal(take(np.uint32, cnt * P).reshape(cnt, P), fn())
        lam = hix.lambda_q.reshape(hix.n, c.p_line)
        pid = hix.pair_id.reshape(hix.n, c.p_line)
        for v in range(min(8, hix.n)):
            d = take(np.float32, 1)[0]
            assert np.float32(d).view(np.uint32) == np.float32(ref.line_distance(lam[v], pid[v], want["fine"])).view(np.uint32)
    npairs = c.k1 * (c.k1 - 1) // 2 if c.k1 > 1 else 1
    assert np.array_equal(take(np.uint16, 2 * npairs).reshape(npairs, 2), Ref.decode_pairs(c.k1, npairs))
    slopes, entries = Ref.build_slope_tables(4096)
    for t in range(10):
        assert take(np.float64, 1)[0] == slopes[t]
        assert np.array_equal(take(np.uint32, 2 * 4096).reshape(4096, 2), entries[t])
    assert pos == len(buf)
