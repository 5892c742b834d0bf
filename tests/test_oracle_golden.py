"""The C restatement (oracle/) against golden vectors produced by the reference itself."""
import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, load_golden
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


@pytest.mark.parametrize("name", GOLDEN_CASES)
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
