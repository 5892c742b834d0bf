"""Pin the C restatement against the reference compiled in place (oracle/_ref), plus the
SPEC.md known-answer examples for the hot-path functions."""
import numpy as np
import pytest

from conftest import needs_ref
from oracle.bindings import Oracle, Ref
from paper_1702_05911_b200.index import PqtConfig

pytestmark = [needs_ref]

CONFIGS = [
    dict(dim=64, p_tree=2, k1=16, k2=8, w=4, p_line=16, candidate_budget=1024),
    dict(dim=64, p_tree=4, k1=16, k2=8, w=4, p_line=16, candidate_budget=1024),
    dict(dim=48, p_tree=4, k1=8, k2=8, w=8, p_line=16, candidate_budget=600, hash_size=3001),
    dict(dim=32, p_tree=1, k1=8, k2=8, w=3, p_line=8, candidate_budget=300),
    dict(dim=64, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=700, resort_bins=True),
    dict(dim=64, p_tree=4, k1=8, k2=4, w=4, p_line=16, candidate_budget=512, resort_bins=True),
    dict(dim=60, p_tree=2, k1=30, k2=4, w=5, p_line=20, candidate_budget=800),   # pair width 2
    dict(dim=32, p_tree=2, k1=1, k2=4, w=1, p_line=8, candidate_budget=100),    # k1 == 1
    dict(dim=32, p_tree=2, k1=4, k2=1, w=1, p_line=8, candidate_budget=100),    # W == 1
    dict(dim=64, p_tree=2, k1=16, k2=16, w=8, p_line=16, candidate_budget=6000, resort_bins=True),  # resort batch > 4096
]


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_oracle_equals_reference(ci):
    cfg = PqtConfig(train_iters=8, seed=100 + ci, **CONFIGS[ci])
    X = Ref.synth(12000 + 100, cfg.dim, 128, 20.0, 100 + ci)
    db, Q = X[:12000], X[12000:]
    ref = Ref.build(db[:6000], db, cfg, threads=8)
    o = Oracle(ref.host_index())
    for k in (1, 37, 100):
        a = ref.knn(Q, k, threads=8)
        b = o.knn(Q, k, threads=3)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_encode_slot_spec_examples():
    # P=2, k1=4, k2=4: part0=(1,2), part1=(0,0) -> global 6 -> slot 6
    assert Ref.encode_slot([1, 2, 0, 0], 4, 4, 1 << 20) == 6
    assert Oracle.encode_slot([1, 2, 0, 0], 4, 4, 1 << 20) == 6
    # all-zero code -> 0; codes differing by exactly H collide
    assert Oracle.encode_slot([0, 0, 0, 0], 4, 4, 7) == 0
    a = Oracle.encode_slot([1, 2, 0, 0], 4, 4, 6)   # 6 % 6
    b = Oracle.encode_slot([0, 0, 0, 0], 4, 4, 6)
    assert a == b == 0
    rng = np.random.default_rng(0)
    for _ in range(500):
        P = int(rng.choice([1, 2, 4]))
        k1, k2 = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        parts = np.stack([rng.integers(0, k1, P), rng.integers(0, k2, P)], 1).reshape(-1)
        H = int(rng.integers(1, 1 << 40))
        assert Oracle.encode_slot(parts, k1, k2, H) == Ref.encode_slot(parts, k1, k2, H)


def test_pick_slope_table_matches_reference():
    rng = np.random.default_rng(1)
    cases = [([0.0], [0.0, 1.0]), ([1.0, 1.0], [0.0, 2.0]), ([0.0, 2.0], [5.0, 5.0]), ([0.0, 1.0], [0.0, 1.0])]
    for _ in range(2000):
        a = np.sort(rng.exponential(10, 4)).astype(np.float32)
        b = np.sort(rng.exponential(10, 4) * rng.choice([0.5, 1, 2, 3])).astype(np.float32)
        cases.append((a, b))
    for a, b in cases:
        assert Oracle.pick_slope_table(a, b) == Ref.pick_slope_table(a, b)
    assert Oracle.pick_slope_table([0.0, 1.0], [0.0, 1.0]) == 5


def test_slope_table_spec_examples():
    slopes, entries = Ref.build_slope_tables(4096)
    assert np.allclose(slopes, 1.08 ** np.arange(-5, 5))
    t1 = [tuple(e) for e in entries[5][:3]]
    assert t1 == [(0, 0), (0, 1), (1, 0)]          # SPEC.md:281 tie rule
    t9 = [tuple(e) for e in entries[9][:3]]
    assert t9[0] == (0, 0) and t9.index((1, 0)) < t9.index((0, 1))


def test_line_distance_spec_examples():
    # One fine part of 2 dims, centroids c0=(0,0), c1=(4,0): SPEC.md:357-359.
    cfg = PqtConfig(dim=2, p_tree=1, k1=2, k2=1, w=1, p_line=1, candidate_budget=4)
    X = np.array([[0, 0], [4, 0], [0, 0], [4, 0], [1, 0], [3, 0]], np.float32)
    ref = Ref.build(X, X, cfg, threads=1)
    hix = ref.host_index()
    hix.level1[0] = np.array([[0, 0], [4, 0]], np.float32)
    hix.d2[0] = np.array([[0, 16], [16, 0]], np.float32)
    o = Oracle(hix)
    # query y=(2,3): b2 = |y-c0|^2 = 13, a2 = |y-c1|^2 = 13, c2 = 16
    fine = np.array([[13.0, 13.0]], np.float32)
    assert o.line_distance([0], [0], fine) == 13.0               # lambda = 0 -> b^2
    assert o.line_distance([255], [0], fine) == 13.0             # lambda = 1 -> a^2
    lam = np.float32(128) * np.float32(1.0 / 255.0)
    expect = np.float32(13) + lam * lam * np.float32(16) + lam * (np.float32(13 - 13 - 16))
    assert abs(o.line_distance([128], [0], fine) - float(expect)) == 0.0
    assert abs(float(expect) - 9.0) < 0.01                        # ~9 at lambda ~ 0.5
    r = Ref.from_host(hix)
    for lq in range(256):
        assert o.line_distance([lq], [0], fine) == r.line_distance([lq], [0], fine)
