"""The C restatement (oracle/) against golden vectors produced by the reference itself."""
import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, ORDER_CASES, load_golden
from oracle.bindings import Oracle
from paper_1702_05911_b200.index import HostIndex


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_knn_matches_golden(name):
    g = load_golden(name)
    o = Oracle(str(GOLDEN / f"{name}.pqt"))
    ids, dists, counts, stats = o.knn(g["queries"], int(g["k"]), threads=4)
    assert np.array_equal(counts, g["counts"])
    assert np.array_equal(stats, g["stats"])
    for q in range(len(counts)):
        c = counts[q]
        assert np.array_equal(ids[q, :c], g["ids"][q, :c])
        assert np.array_equal(dists[q, :c].view(np.uint32), g["dists"][q, :c].view(np.uint32))


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_traverse_and_order_match_golden(name):
    g = load_golden(name)
    o = Oracle(str(GOLDEN / f"{name}.pqt"))
    off = 0
    for i in range(g["fine"].shape[0]):
        t = o.traverse(g["queries"][i])
        for key in ("fine", "l1_id", "l1_dist", "l2_parent", "l2_child", "l2_dist"):
            assert np.array_equal(t[key].view(np.uint32), g[key][i].view(np.uint32)), key
        n = int(g["order_len"][i])
        order = o.heuristic_order(t["l2_dist"], 4096)
        assert np.array_equal(order, g["orders"][off:off + n])
        off += n


@pytest.mark.parametrize("name", GOLDEN_CASES + ORDER_CASES)
def test_container_roundtrip_is_byte_identical(name, tmp_path):
    """PQTINDEX v1 reader/writer (index.py) reproduce the reference's save_index bytes."""
    src = GOLDEN / f"{name}.pqt"
    ix = HostIndex.load(str(src))
    out = tmp_path / "rt.pqt"
    ix.save(str(out))
    assert out.read_bytes() == src.read_bytes()
    o = Oracle(str(src))
    out2 = tmp_path / "rt2.pqt"
    o.save(str(out2))
    assert out2.read_bytes() == src.read_bytes()


def test_truncated_container_is_rejected(tmp_path):
    src = (GOLDEN / "p2_small.pqt").read_bytes()
    for cut in (4, 40, 73, 500, len(src) - 1):
        p = tmp_path / f"t{cut}.pqt"
        p.write_bytes(src[:cut])
        with pytest.raises(Exception):
            HostIndex.load(str(p))
        with pytest.raises(RuntimeError):
            Oracle(str(p))
    bad = bytearray(src)
    bad[0:8] = b"NOTINDEX"
    (tmp_path / "m.pqt").write_bytes(bytes(bad))
    with pytest.raises(RuntimeError, match="magic"):
        Oracle(str(tmp_path / "m.pqt"))


def _check_exact(got, g, k, ctx):
    ids, dists, counts, stats = got
    assert np.array_equal(counts, g[f"counts_k{k}"]), ctx
    assert np.array_equal(stats, g[f"stats_k{k}"]), ctx  # exact_evals = min(max(rerank_exact, k), C)
    for q in range(len(counts)):
        c = counts[q]
        assert np.array_equal(ids[q, :c], g[f"ids_k{k}"][q, :c]), f"{ctx} q={q}"
        assert np.array_equal(dists[q, :c].view(np.uint32), g[f"dists_k{k}"][q, :c].view(np.uint32)), f"{ctx} q={q}"


def test_oracle_exact_rerank_matches_golden():
    """Raw vectors attached: the exact re-rank stage (search.cpp:229-249), k below and above
    rerank_exact, against the reference's outputs on its keep_raw build."""
    g = load_golden("p2_exact")
    o = Oracle(str(GOLDEN / "p2_exact.pqt"))
    assert o.config.rerank_exact == 48
    o.attach_database(g["db"])
    for k in g["ks"]:
        _check_exact(o.knn(g["queries"], int(k), threads=4), g, int(k), f"k={k}")
    # detached: the loaded-index path (no exact stage, exact_evals 0)
    o.attach_database(None)
    ids, dists, counts, stats = o.knn(g["queries"], 20, threads=4)
    assert (stats[:, 2] == 0).all()
    with pytest.raises(ValueError):
        o.attach_database(g["db"][:-1])


@pytest.mark.parametrize("name", ORDER_CASES)
def test_exact_order_golden_is_the_reference(name):
    """The exact-order fixtures (P = 3; P = 2 without slope tables) replay on the reference
    compiled in place: its knn_query_batch reproduces them (the C restatement has no exact order,
    so these are pinned by the reference alone)."""
    from oracle.bindings import Ref

    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    g = load_golden(name)
    ids, dists, counts, stats = Ref.load(str(GOLDEN / f"{name}.pqt")).knn(g["queries"], int(g["k"]), threads=4)
    assert np.array_equal(counts, g["counts"]) and np.array_equal(stats, g["stats"])
    for q in range(len(counts)):
        c = counts[q]
        assert np.array_equal(ids[q, :c], g["ids"][q, :c])
        assert np.array_equal(dists[q, :c].view(np.uint32), g["dists"][q, :c].view(np.uint32))
