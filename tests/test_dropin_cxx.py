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
@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p1_small", "p2_resort"])
def test_cxx_knn_query_batch_matches_reference(dropin_bin, name, tmp_path):
    g = load_golden(name)
    qf = tmp_path / "q.f32"
    g["queries"].astype(np.float32).tofile(qf)
    out = tmp_path / "out.bin"
    k = int(g["k"])
    r = subprocess.run([str(dropin_bin), "query", str(GOLDEN / f"{name}.pqt"), str(qf), str(g["queries"].shape[1]),
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
