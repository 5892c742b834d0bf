import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"
GOLDEN_CASES = ["p2_small", "p4_small", "p1_small", "p2_resort", "p2_wide", "p2_sift", "p4_gist"]
# the reference's exact (Dijkstra) bin order: P = 3, and P = 2 without slope tables
ORDER_CASES = ["p3_order", "p3_order_resort", "p2_notables"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference compiled in place)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the test-only oracle (and the reference when its sources are present) once."""
    from oracle import bindings

    bindings.build(ref=Path("/root/reference/proj/src").exists())
    from paper_1702_05911_b200 import build as pbuild

    pbuild.build()


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


def ref_available():
    from oracle.bindings import Ref

    return Ref.available()


needs_ref = pytest.mark.skipif(not (REPO / "oracle" / "_ref" / "libpqtref.so").exists()
                               and not Path("/root/reference/proj/src").exists(),
                               reason="reference not compiled (oracle/_ref)")
