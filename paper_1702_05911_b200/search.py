"""Python mirror of the reference query API over the C-ABI (include/pqtg.h).

    index = load_index(path)                       # pqt::load_index        (index_io.hpp:16)
    results = knn_query_batch(index, queries, k)   # pqt::knn_query_batch   (search.hpp:83)
    result = knn_query(index, y, k)                # pqt::knn_query         (search.hpp:80)

Same names, argument meaning and error behaviour as the reference: a query-dimension
mismatch raises ValueError (std::invalid_argument, search.cpp:264-266), a malformed
container raises FormatError (index_io.cpp), k == 0 or an empty index gives empty results,
and fewer than k candidates give short results. Everything runs in libpqtg.so on the GPU;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import PqtgError, PqtgIndexInfo, check, lib
from .index import FormatError, HostIndex, PqtConfig


@dataclass
class QueryStats:
    """pqt::QueryStats (search.hpp:15-23); *_us are the query's per-stage device times."""

    bins_visited: int = 0
    candidates: int = 0
    exact_evals: int = 0
    traversal_us: float = 0.0
    bin_selection_us: float = 0.0
    vector_proposal_us: float = 0.0
    rerank_us: float = 0.0


@dataclass
class QueryResult:
    ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    dists: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    stats: QueryStats = field(default_factory=QueryStats)


_warned_missing_db = False


def _warn_missing_database():
    # search.cpp:25-32: one-time warning when rerank_exact > 0 but no raw vectors are attached
    global _warned_missing_db
    if not _warned_missing_db:
        _warned_missing_db = True
        sys.stderr.write("pqt: rerank_exact > 0 but no raw vectors attached; exact re-ranking disabled\n")


def _raise(e: PqtgError):
    if e.status == -1 or e.status == -2:
        raise ValueError(str(e)) from None
    if e.status == -3:
        raise FormatError(str(e)) from None
    raise e


class DeviceIndex:
    """A PQT index resident in one GPU's HBM (pqtg_index), plus a workspace for searches."""

    def __init__(self, source: "HostIndex | str", device: int = 0, shard: tuple[int, int] = (0, 0),
                 max_batch: int = 4096):
        L = lib()
        h = C.c_void_p()
        try:
            if isinstance(source, HostIndex):
                view = source.view(*shard)
                check(L.pqtg_index_create(C.byref(view), device, C.byref(h)))
            elif hasattr(source, "shard_lo"):  # builder.ShardIndex: one shard, codes by position
                view = source.view()
                check(L.pqtg_index_create_shard(C.byref(view), source.lambda_q.ctypes.data,
                                                source.pair_id.ctypes.data, device, C.byref(h)))
            else:
                check(L.pqtg_index_load(str(source).encode(), device, shard[0], shard[1], C.byref(h)))
        except PqtgError as e:
            _raise(e)
        self._h = h
        info = PqtgIndexInfo()
        check(L.pqtg_index_info_get(h, C.byref(info)))
        self.info = info
        self.config = PqtConfig.from_c(info.config)
        self.n = int(info.n)
        self.device = device
        self.max_batch = int(max_batch)
        ws = C.c_void_p()
        check(L.pqtg_workspace_create(h, self.max_batch, C.byref(ws)))
        self._ws = ws
        self._query_times = False
        self.has_database = False

    def close(self):
        L = _abi._LIB
        if L is not None:
            if getattr(self, "_ws", None):
                L.pqtg_workspace_destroy(self._ws)
                self._ws = None
            if getattr(self, "_h", None):
                L.pqtg_index_destroy(self._h)
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self) -> int:
        return self.n

    @property
    def handle(self):
        return self._h

    def attach_database(self, rows: "np.ndarray | None") -> None:
        """PqtIndex::attach_database (search.cpp:44-49): n × dim raw vectors (id order) for the
        exact re-rank stage (search.cpp:229-249, when rerank_exact > 0); on a position shard the
        shard's rows in position order (db[ids[lo:hi]]), used by the sharded search. None detaches."""
        if rows is None:
            check(lib().pqtg_index_attach_database(self._h, None, 0, 0))
            self.has_database = False
            return
        r = np.ascontiguousarray(rows, np.float32)
        if r.ndim != 2:
            raise ValueError("attach_database: vector set does not match index")
        try:
            check(lib().pqtg_index_attach_database(self._h, r.ctypes.data, r.shape[0], r.shape[1]))
        except _abi.PqtgError as e:
            if e.status == -1:  # BAD_DIM: std::invalid_argument in the reference
                raise ValueError(str(e)) from None
            raise
        self.has_database = True

    @property
    def workspace(self):
        return self._ws

    # ---- host-buffer search (pqtg_search) --------------------------------------------
    def search(self, queries: np.ndarray, k: int):
        """Returns (ids [nq,k] u32, dists [nq,k] f32, counts [nq] u32, stats [nq,3] u64)."""
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        nq, dim = q.shape
        kk = max(int(k), 1)
        ids = np.empty((nq, kk), np.uint32)
        dists = np.empty((nq, kk), np.float32)
        counts = np.zeros(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        try:
            check(lib().pqtg_search(self._h, self._ws, q.ctypes.data if nq else None, nq, dim, int(k),
                                    ids.ctypes.data, dists.ctypes.data, counts.ctypes.data,
                                    stats.ctypes.data))
        except PqtgError as e:
            _raise(e)
        return ids[:, :k], dists[:, :k], counts, stats

    # ---- device-buffer search (pqtg_search_device) -------------------------------------
    def search_device(self, d_queries: int, nq: int, k: int, d_ids: int, d_dists: int, d_counts: int,
                      d_stats: int | None = None, stream: int | None = None) -> None:
        check(lib().pqtg_search_device(self._h, self._ws, d_queries, nq, k, d_ids, d_dists, d_counts,
                                       d_stats, stream))

    def set_chunks(self, chunks: int) -> None:
        """Overlap stages across `chunks` pieces of each batch on two streams (0 = auto, 1 = off)."""
        check(lib().pqtg_workspace_set_chunks(self._ws, int(chunks)))

    def status(self) -> None:
        """Raise what the last search_device call's kernels flagged (pqtg_workspace_status)."""
        try:
            check(lib().pqtg_workspace_status(self._ws))
        except PqtgError as e:
            _raise(e)

    def enable_query_times(self, on: bool = True) -> None:
        """Collect per-query stage clocks (pqtg_workspace_query_times)."""
        check(lib().pqtg_workspace_query_times(self._ws, 1 if on else 0))

    def query_times(self, nq: int) -> np.ndarray:
        """nq × 3 per-query stage device times of the last search, µs: traversal, bin
        selection + gather, re-rank (+ exact) -- QueryStats' *_us (search.cpp:134-137)."""
        us = np.zeros((nq, 3), np.float32)
        check(lib().pqtg_workspace_read_query_times(self._ws, nq, us.ctypes.data))
        return us

    def stage_ms(self) -> list[float]:
        ms = (C.c_float * 4)()
        check(lib().pqtg_workspace_stage_ms(self._ws, ms))
        return list(ms)

    def intermediates(self, nq: int) -> dict:
        """Per-query intermediates of the last searched sub-batch (for per-stage parity)."""
        c = self.config
        W = c.w * c.k2
        budget = min(c.candidate_budget, self.n)
        fine = np.zeros((nq, c.p_line, c.k1), np.float32)
        l2c = np.zeros((nq, c.p_tree, W), np.uint32)
        l2d = np.zeros((nq, c.p_tree, W), np.float32)
        slope = np.zeros((nq, 2), np.uint8)
        pos = np.zeros((nq, max(budget, 1)), np.uint32)
        nc = np.zeros(nq, np.uint32)
        nt = np.zeros(nq, np.uint32)
        check(lib().pqtg_workspace_read(self._ws, nq, fine.ctypes.data, l2c.ctypes.data, l2d.ctypes.data,
                                        slope.ctypes.data, pos.ctypes.data, nc.ctypes.data, nt.ctypes.data))
        return dict(fine=fine, l2_parent=l2c >> 16, l2_child=l2c & 0xFFFF, l2_dist=l2d, slope=slope,
                    positions=[pos[i, : nc[i]] for i in range(nq)], ncand=nc, ntuples=nt)

    def counters(self, nq: int) -> dict:
        """Cheap per-query counters of the last sub-batch: candidates, tuples consumed, and
        (`nlocal`) the candidates inside this index's position shard, which are the ones its
        re-rank scores (all of them when unsharded)."""
        nc = np.zeros(nq, np.uint32)
        nt = np.zeros(nq, np.uint32)
        lo, hi = int(self.info.shard_lo), int(self.info.shard_hi)
        if hi > lo and self.config.candidate_budget:
            pos = np.zeros((nq, self.config.candidate_budget), np.uint32)
            check(lib().pqtg_workspace_read(self._ws, nq, None, None, None, None, pos.ctypes.data,
                                            nc.ctypes.data, nt.ctypes.data))
            valid = np.arange(pos.shape[1])[None, :] < nc[:, None]
            nl = np.count_nonzero(valid & (pos >= lo) & (pos < hi), axis=1).astype(np.uint32)
        else:
            check(lib().pqtg_workspace_read(self._ws, nq, None, None, None, None, None, nc.ctypes.data,
                                            nt.ctypes.data))
            nl = nc
        return dict(ncand=nc, ntuples=nt, nlocal=nl)


def brute_force_knn(db: np.ndarray, queries: np.ndarray, k: int, device: int = 0):
    """pqt::brute_force_knn (search.cpp:276-299) for a batch, on the GPU: exact sequential-fp32
    l2_sq to every row, (dist, id) order. Returns (ids, dists, counts, stats) like
    DeviceIndex.search; stats rows are (bins_visited, candidates, exact_evals) = (0, n, n)."""
    x = np.ascontiguousarray(db, np.float32)
    q = np.ascontiguousarray(queries, np.float32)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if x.ndim != 2 or q.shape[1] != x.shape[1]:
        raise ValueError("brute_force_knn: query dimension mismatch")
    nq = q.shape[0]
    ids = np.zeros((nq, max(k, 1)), np.uint32)
    dists = np.zeros((nq, max(k, 1)), np.float32)
    counts = np.zeros(nq, np.uint32)
    stats = np.zeros((nq, 3), np.uint64)
    check(lib().pqtg_brute_force_knn(x.ctypes.data, x.shape[0], x.shape[1], q.ctypes.data, nq, k, device,
                                     ids.ctypes.data, dists.ctypes.data, counts.ctypes.data, stats.ctypes.data))
    return ids[:, :k], dists[:, :k], counts, stats


def load_index(path: str, device: int = 0, shard: tuple[int, int] = (0, 0)) -> DeviceIndex:
    """pqt::load_index: read a PQTINDEX v1 file straight into GPU memory."""
    return DeviceIndex(path, device=device, shard=shard)


def knn_query_batch(index: DeviceIndex, queries: np.ndarray, k: int, threads: int = 0) -> list[QueryResult]:
    """pqt::knn_query_batch (search.cpp:262-274). `threads` is accepted for API parity."""
    q = np.asarray(queries, np.float32)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.shape[0] > 0 and q.shape[1] != index.config.dim:
        raise ValueError("knn_query_batch: query dimension mismatch")
    if index.config.rerank_exact > 0 and k > 0 and index.n > 0 and q.shape[0] > 0 and not index.has_database:
        _warn_missing_database()
    if not index._query_times:
        index.enable_query_times()
        index._query_times = True
    ids, dists, counts, stats = index.search(q, k)
    # each query's stage device times (search.cpp:134-137,167-216,220,258); bin selection and
    # gathering are one kernel, reported as bin_selection_us
    us = index.query_times(q.shape[0]) if q.shape[0] else np.zeros((0, 3), np.float32)
    out = []
    for i in range(q.shape[0]):
        c = int(counts[i])
        st = QueryStats(int(stats[i, 0]), int(stats[i, 1]), int(stats[i, 2]),
                        float(us[i, 0]), float(us[i, 1]), 0.0, float(us[i, 2]))
        out.append(QueryResult(ids[i, :c].copy(), dists[i, :c].copy(), st))
    return out


def knn_query(index: DeviceIndex, y: np.ndarray, k: int) -> QueryResult:
    """pqt::knn_query (search.cpp:126-260) for one query vector."""
    y = np.asarray(y, np.float32).reshape(1, -1)
    return knn_query_batch(index, y, k)[0]


def merge_topk_host(ids: np.ndarray, dists: np.ndarray, counts: np.ndarray):
    """Merge per-shard top-k lists [G, nq, k] by (dist, id) via pqtg_merge_topk_host."""
    ids = np.ascontiguousarray(ids, np.uint32)
    dists = np.ascontiguousarray(dists, np.float32)
    counts = np.ascontiguousarray(counts, np.uint32)
    G, nq, k = ids.shape
    oi = np.empty((nq, k), np.uint32)
    od = np.empty((nq, k), np.float32)
    oc = np.empty(nq, np.uint32)
    check(lib().pqtg_merge_topk_host(G, nq, k, ids.ctypes.data, dists.ctypes.data, counts.ctypes.data,
                                     oi.ctypes.data, od.ctypes.data, oc.ctypes.data))
    return oi, od, oc


def shard_range(n: int, shards: int, rank: int) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    check(lib().pqtg_shard_range(n, shards, rank, C.byref(lo), C.byref(hi)))
    return int(lo.value), int(hi.value)
