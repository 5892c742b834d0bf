"""GPU-side checks at full workload scale and of the offline build kernels.

* pqtg_build_codes (assign_bin + global_code + encode_line) equals the reference's CPU
  functions on the same codebooks, vector for vector.
* 1M-vector GIST- and SIFT-shaped indexes built on the GPU: a sample of queries matches the C
  oracle bit for bit, and the size-independent properties hold for the whole batch
  (dists non-decreasing, counts = min(k, C), determinism across batchings).
"""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN, needs_ref
from oracle.bindings import Oracle, Ref
from paper_1702_05911_b200 import DeviceIndex, HostIndex, PqtConfig, builder
from paper_1702_05911_b200._abi import check, lib

pytestmark = pytest.mark.gpu


@needs_ref
@pytest.mark.parametrize("name", ["p2_sift", "p4_gist", "p2_wide", "p1_small"])
def test_build_codes_match_reference(name):
    import torch

    hix = HostIndex.load(str(GOLDEN / f"{name}.pqt"))
    ref = Ref.from_host(hix)
    c = hix.config
    X = Ref.synth(3000, c.dim, 40, 25.0, 99)
    codes_ref, lam_ref, pid_ref = ref.assign_encode(X)
    dev = torch.device("cuda", 0)
    sl = builder.fine_slices(hix.level1, c.p_line)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    l1, l2, tsl, tsq, td2, tx = t(hix.level1), t(hix.level2), t(sl), t(builder.seq_sqnorm(sl)), t(hix.d2), t(X)
    n = X.shape[0]
    pc = torch.empty((n, c.p_tree), dtype=torch.int32, device=dev)
    slots = torch.empty(n, dtype=torch.int64, device=dev)
    lam = torch.empty((n, c.p_line), dtype=torch.uint8, device=dev)
    pid = torch.empty((n, c.p_line), dtype=torch.int16, device=dev)
    cfg = c.to_c()
    cfg.hash_size = 0  # raw global code
    check(lib().pqtg_build_codes(C.byref(cfg), l1.data_ptr(), l2.data_ptr(), tsl.data_ptr(), tsq.data_ptr(),
                                 td2.data_ptr(), tx.data_ptr(), n, pc.data_ptr(), slots.data_ptr(), lam.data_ptr(),
                                 pid.data_ptr(), None))
    torch.cuda.synchronize()
    assert np.array_equal(slots.cpu().numpy().view(np.uint64), codes_ref)
    assert np.array_equal(lam.cpu().numpy(), lam_ref)
    assert np.array_equal(pid.cpu().numpy().view(np.uint16), pid_ref)


def _built(shape):
    import torch

    dev = torch.device("cuda", 0)
    if shape == "gist":
        cfg = PqtConfig(dim=960, p_tree=4, k1=16, k2=8, w=4, p_line=32, train_iters=8, seed=3)
        n, blobs = 1_000_000, 1024
    elif shape == "sift":
        cfg = PqtConfig(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, train_iters=8, seed=4)
        n, blobs = 1_000_000, 1024
    else:  # pair width 2 (k1 = 32, 496 pairs), the SIFT1B tree
        cfg = PqtConfig(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, train_iters=6, seed=5,
                        candidate_budget=2048)
        n, blobs = 300_000, 512
    X = builder.synth_clustered(n + 256, cfg.dim, blobs, 20.0, cfg.seed, device=dev)
    db, Q = X[:n], X[n:]
    hix = builder.build_index(db, db[:50_000], cfg)
    return hix, Q.cpu().numpy()


@pytest.mark.parametrize("shape", ["gist", "sift", "wide"])
def test_full_scale_parity_and_properties(shape):
    from paper_1702_05911_b200._abi import lib as L

    hix, Q = _built(shape)
    k = 100
    dev = DeviceIndex(hix)
    ids, dists, counts, stats = dev.search(Q, k)
    o = Oracle(hix)
    sample = np.arange(0, len(Q), 8)
    oi, od, oc, os_ = o.knn(Q[sample], k)
    assert np.array_equal(counts[sample], oc)
    assert np.array_equal(stats[sample], os_)
    for a, q in enumerate(sample):
        c = counts[q]
        assert np.array_equal(ids[q, :c], oi[a, :c])
        assert np.array_equal(dists[q, :c].view(np.uint32), od[a, :c].view(np.uint32))
    # properties over the whole batch
    assert (counts == np.minimum(k, stats[:, 1])).all()
    for q in range(len(Q)):
        d = dists[q, : counts[q]]
        assert (np.diff(d) >= 0).all()
        assert len(set(ids[q, : counts[q]].tolist())) == counts[q]
    # generic kernels and a different batching give identical results
    L().pqtg_set_kernel_variant(1)
    try:
        g = DeviceIndex(hix, max_batch=37).search(Q, k)
    finally:
        L().pqtg_set_kernel_variant(0)
    for x, y in zip((ids, dists, counts, stats), g):
        assert np.array_equal(x, y)
