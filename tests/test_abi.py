"""CPU-only checks of the C-ABI library: it loads, exports every declared symbol, and its
host-side logic (bin-order addressing, shard ranges, top-k merge) is right. No GPU calls."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, REPO, load_golden
from paper_1702_05911_b200 import HostIndex, merge_topk_host, shard_range
from paper_1702_05911_b200._abi import LIB_PATH, SIGNATURES, lib


def declared_symbols():
    text = (REPO / "include" / "pqtg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pqtg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    so = C.CDLL(str(LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(so, name), name
        assert name in SIGNATURES, f"{name} missing from the ctypes mirror"
    assert lib().pqtg_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_host_bin_stream_addressing_matches_reference_order(name):
    """The static-stream materialization + closed-form addressing the kernels use reproduces
    the reference's heuristic_order (golden, from binorder.cpp BinStream)."""
    g = load_golden(name)
    ix = HostIndex.load(str(GOLDEN / f"{name}.pqt"))
    v = ix.view()
    off = 0
    for i in range(g["l2_dist"].shape[0]):
        lists = np.ascontiguousarray(g["l2_dist"][i], np.float32)
        n = int(g["order_len"][i])
        out = np.zeros((n, ix.config.p_tree), np.uint32)
        cnt = lib().pqtg_bin_stream_host(C.byref(v), lists.ctypes.data, n, out.ctypes.data)
        assert cnt == n
        assert np.array_equal(out, g["orders"][off:off + n])
        off += n


def test_host_bin_stream_deep_quad_order_vs_oracle():
    """P=4 far past the slope-1 table prefix (closed-form sweep rows) vs the C restatement."""
    from oracle.bindings import Oracle

    for name, depth in (("p4_small", 10 ** 6), ("p4_gist", 300000)):
        path = str(GOLDEN / f"{name}.pqt")
        ix = HostIndex.load(path)
        o = Oracle(path)
        v = ix.view()
        rng = np.random.default_rng(3)
        W = ix.config.w * ix.config.k2
        for _ in range(3):
            lists = np.sort(rng.exponential(5, (4, W)), axis=1).astype(np.float32)
            want = o.heuristic_order(lists, depth)
            out = np.zeros((len(want), 4), np.uint32)
            cnt = lib().pqtg_bin_stream_host(C.byref(v), lists.ctypes.data, len(want), out.ctypes.data)
            assert cnt == len(want) == min(depth, W ** 4)
            assert np.array_equal(out, want)


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1000, 12345):
        for g in (1, 2, 3, 8):
            r = [shard_range(n, g, i) for i in range(g)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(g - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1


def test_merge_topk_host_orders_by_dist_then_id():
    rng = np.random.default_rng(0)
    G, nq, k = 3, 50, 10
    ids = np.zeros((G, nq, k), np.uint32)
    dists = np.zeros((G, nq, k), np.float32)
    counts = rng.integers(0, k + 1, (G, nq)).astype(np.uint32)
    allv = []
    for q in range(nq):
        pool = rng.permutation(1000)[: G * k]
        dd = rng.integers(0, 5, G * k).astype(np.float32)  # many exact ties
        items = []
        for gg in range(G):
            sl = sorted(zip(dd[gg * k:(gg + 1) * k], pool[gg * k:(gg + 1) * k]))[: counts[gg, q]]
            for j, (d, i) in enumerate(sl):
                ids[gg, q, j], dists[gg, q, j] = i, d
            items += sl
        allv.append(sorted(items)[:k])
    oi, od, oc = merge_topk_host(ids, dists, counts)
    for q in range(nq):
        want = allv[q]
        assert oc[q] == len(want)
        assert [(float(od[q, j]), int(oi[q, j])) for j in range(oc[q])] == [(float(d), int(i)) for d, i in want]


def test_errors_without_gpu_are_reported_not_crashes():
    from paper_1702_05911_b200._abi import PqtgError, check

    ix = HostIndex.load(str(GOLDEN / "p2_small.pqt"))
    v = ix.view()
    h = C.c_void_p()
    rc = lib().pqtg_index_create(C.byref(v), 0, C.byref(h))
    if lib().pqtg_device_ok(0):
        assert rc == 0
        lib().pqtg_index_destroy(h)
    else:
        assert rc < 0 and not h.value
        with pytest.raises(PqtgError):
            check(rc)
    # invalid config -> CONFIG (-2) before touching the device
    bad = ix.view()
    bad.config.w = 100
    assert lib().pqtg_index_create(C.byref(bad), 0, C.byref(h)) == -2
    assert b"w must be in" in lib().pqtg_last_error()


def test_kernel_variant_selector_range():
    """pqtg_set_kernel_variant: 0 auto, 1 generic, 2 tensor-core screen, 3 / 4 walker / all-warp
    bin selection (include/pqtg.h); anything else is an argument error."""
    L = lib()
    try:
        for v in range(5):
            assert L.pqtg_set_kernel_variant(v) == 0
        assert L.pqtg_set_kernel_variant(5) == -7  # PQTG_ERR_ARG
        assert L.pqtg_set_kernel_variant(-1) == -7
        assert b"variant must be" in L.pqtg_last_error()
    finally:
        L.pqtg_set_kernel_variant(0)


def test_brute_force_argument_errors_without_device_work():
    """pqtg_brute_force_knn rejects bad arguments before touching a device."""
    import numpy as np

    L = lib()
    q = np.zeros((2, 8), np.float32)
    out_i = np.zeros((2, 4), np.uint32)
    out_d = np.zeros((2, 4), np.float32)
    out_c = np.zeros(2, np.uint32)
    assert L.pqtg_brute_force_knn(None, 10, 8, q.ctypes.data, 2, 4, 0, out_i.ctypes.data, out_d.ctypes.data,
                                  out_c.ctypes.data, None) == -7  # PQTG_ERR_ARG: null db with n > 0
    db = np.zeros((10, 8), np.float32)
    assert L.pqtg_brute_force_knn(db.ctypes.data, 10, 0, q.ctypes.data, 2, 4, 0, out_i.ctypes.data,
                                  out_d.ctypes.data, out_c.ctypes.data, None) < 0  # dim 0
