"""Host-side pieces of the GPU index builder reproduce the reference exactly."""
import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, needs_ref
from paper_1702_05911_b200.builder import fine_slices, pair_d2, slope_tables
from paper_1702_05911_b200.index import HostIndex


@needs_ref
def test_slope_tables_equal_reference():
    from oracle.bindings import Ref

    s_ref, e_ref = Ref.build_slope_tables(4096)
    s, e = slope_tables(4096)
    assert np.array_equal(s.view(np.uint64), s_ref.view(np.uint64))
    assert np.array_equal(e, e_ref)
    s_ref, e_ref = Ref.build_slope_tables(100)
    s, e = slope_tables(100)
    assert np.array_equal(e, e_ref)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_pair_table_equals_reference(name):
    """d2 recomputed from the level-1 codebooks equals the reference's stored table bit for bit."""
    ix = HostIndex.load(str(GOLDEN / f"{name}.pqt"))
    d2 = pair_d2(fine_slices(ix.level1, ix.config.p_line))
    assert np.array_equal(d2.view(np.uint32), ix.d2.view(np.uint32))


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden_tables_equal_builder_tables(name):
    ix = HostIndex.load(str(GOLDEN / f"{name}.pqt"))
    s, e = slope_tables(ix.entries.shape[1])
    assert np.array_equal(e, ix.entries)
