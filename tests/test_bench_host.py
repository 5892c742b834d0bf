"""bench.py's host-side pieces (no GPU): the algorithmic-byte model of DESIGN.md §5, the
launch-count rule mirrored from api.cpp, and the reference arm's answer for a shard workload."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
from paper_1702_05911_b200.index import HostIndex  # noqa: E402


def test_algorithmic_bytes_model():
    hix = HostIndex.load(str(GOLDEN / "p4_gist.pqt"))
    g = load_golden("p4_gist")
    c = hix.config
    nq = len(g["counts"])
    T = np.full(nq, 100, np.uint32)
    C = g["stats"][:, 1].astype(np.uint32)
    ab = bench.algorithmic_bytes(hix, {"ncand": C, "ntuples": T, "nlocal": C}, g["stats"], int(g["k"]))
    pw = hix.pair_width
    bins = g["stats"][:, 0].astype(np.float64)
    want_rerank = float(np.sum(C * (c.p_line * (1 + pw) + 4) + bins * 8 + 4 * c.p_line * c.k1 + 8 * int(g["k"]) + 4))
    assert ab["rerank"] == pytest.approx(want_rerank)
    assert ab["C_q"] == pytest.approx(C.mean())
    assert ab["T_q"] == pytest.approx(100.0)
    # a shard re-ranks only its own candidates: the model follows nlocal
    ab2 = bench.algorithmic_bytes(hix, {"ncand": C, "ntuples": T, "nlocal": C // 2}, g["stats"], int(g["k"]))
    assert ab2["rerank"] < ab["rerank"] and ab2["C_q"] == pytest.approx((C // 2).mean())


class _Shard:
    def __init__(self, lo, hi, n):
        self.shard_lo, self.shard_hi, self.n = lo, hi, n


def test_gpu_launch_rule_matches_api():
    # api.cpp pqtg_search_device: 2 chunks from 256 queries; a position shard only below 4096
    assert bench.gpu_launches(object(), 100, 0) == 3
    assert bench.gpu_launches(object(), 1000, 0) == 6
    assert bench.gpu_launches(object(), 10000, 0) == 6
    assert bench.gpu_launches(_Shard(0, 10, 80), 10000, 0) == 3
    assert bench.gpu_launches(_Shard(0, 10, 80), 1000, 0) == 6
    assert bench.gpu_launches(_Shard(0, 80, 80), 10000, 0) == 6  # the whole range is no shard
    assert bench.gpu_launches(object(), 1000, 4) == 12


def test_reference_arm_on_a_shard_workload_is_unavailable():
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--workload", "sift1b"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and "unavailable" in line
