"""Host-API behaviour on the GPU that is not a parity question: per-query stage clocks
(QueryStats *_us, search.cpp:134-137,167-216,220,258) and workspace ordering across streams and
entry points."""
import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_golden
from paper_1702_05911_b200 import DeviceIndex, knn_query_batch
from test_gpu_parity import assert_same_results

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist"])
def test_query_stage_times(name):
    g = load_golden(name)
    dev = DeviceIndex(str(GOLDEN / f"{name}.pqt"))
    res = knn_query_batch(dev, g["queries"], int(g["k"]))
    t = np.array([[r.stats.traversal_us, r.stats.bin_selection_us, r.stats.rerank_us] for r in res])
    assert (t > 0).all() and (t < 1e5).all(), t
    assert all(r.stats.vector_proposal_us == 0.0 for r in res)
    # the device entry point: the same clocks for its batch
    dq = torch.from_numpy(g["queries"]).cuda()
    nq, k = dq.shape[0], int(g["k"])
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    c = torch.empty(nq, dtype=torch.int32, device="cuda")
    dev.search_device(dq.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), c.data_ptr(), None,
                      torch.cuda.current_stream().cuda_stream)
    t2 = dev.query_times(nq)
    assert (t2 > 0).all() and (t2 < 1e5).all()


def test_workspace_calls_on_two_streams_and_both_entry_points():
    """One workspace used from two streams and through both entry points in turn: every call
    starts after the previous one (its completion event), so results stay exact."""
    g = load_golden("p2_sift")
    dev = DeviceIndex(str(GOLDEN / "p2_sift.pqt"), max_batch=64)
    want = (g["ids"], g["dists"], g["counts"], g["stats"])
    k = int(g["k"])
    nq = g["queries"].shape[0]
    dq = torch.from_numpy(g["queries"]).cuda()
    outs = []
    for rep in range(4):
        s = torch.cuda.Stream()
        ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        c = torch.empty(nq, dtype=torch.int32, device="cuda")
        st = torch.empty((nq, 3), dtype=torch.int64, device="cuda")
        dev.search_device(dq.data_ptr(), nq, k, ids.data_ptr(), d.data_ptr(), c.data_ptr(), st.data_ptr(), s.cuda_stream)
        outs.append((s, ids, d, c, st))
        assert_same_results(dev.search(g["queries"], k), want, f"host call {rep}")
    torch.cuda.synchronize()
    for s, ids, d, c, st in outs:
        got = (ids.cpu().numpy().view(np.uint32), d.cpu().numpy(), c.cpu().numpy().view(np.uint32),
               st.cpu().numpy().view(np.uint64))
        assert_same_results(got, want, "device call")
