"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the two checkers:

* `Oracle`: oracle/_build/libpqt_oracle.so, the C restatement of the query path.
* `Ref`:    oracle/_ref/libpqtref.so, the reference's own sources compiled in place
            (oracle/Makefile) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs may
import this module. Neither library reads /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_1702_05911_b200._abi import PqtgConfig, PqtgIndexView
from paper_1702_05911_b200.index import HostIndex, PqtConfig

ORACLE_DIR = Path(__file__).resolve().parent
ORACLE_SO = ORACLE_DIR / "_build" / "libpqt_oracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libpqtref.so"

_vp, _u32, _u64 = C.c_void_p, C.c_uint32, C.c_uint64


def build(ref: bool = True) -> None:
    """make the oracle (and, when /root/reference is present, oracle/_ref)."""
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-j8", *targets], cwd=ORACLE_DIR, check=True)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class _Lib:
    _so = None
    _path: Path
    _sigs: dict

    @classmethod
    def so(cls):
        if cls._so is None:
            if not cls._path.exists():
                raise RuntimeError(f"{cls._path} not built (make -C oracle)")
            so = C.CDLL(str(cls._path))
            for name, (res, args) in cls._sigs.items():
                fn = getattr(so, name)
                fn.restype = res
                fn.argtypes = args
            cls._so = so
        return cls._so

    @classmethod
    def available(cls) -> bool:
        return cls._path.exists()


class Oracle(_Lib):
    """C restatement (oracle/pqt_oracle.c) of traverse / BinStream / gather / line_distance / top-k."""

    _path = ORACLE_SO
    _sigs = {
        "pqto_last_error": (C.c_char_p, []),
        "pqto_from_view": (_vp, [C.POINTER(PqtgIndexView)]),
        "pqto_load": (_vp, [C.c_char_p]),
        "pqto_save": (C.c_int, [_vp, C.c_char_p]),
        "pqto_free": (None, [_vp]),
        "pqto_view": (None, [_vp, C.POINTER(PqtgIndexView)]),
        "pqto_traverse": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        "pqto_pick_slope_table": (_u32, [_vp, _u64, _vp, _u64]),
        "pqto_heuristic_order": (C.c_int64, [_vp, _vp, _u32, _u32, _u64, _vp]),
        "pqto_encode_slot": (_u64, [_vp, _u32, _u32, _u32, _u64]),
        "pqto_line_distance": (C.c_float, [_vp, _vp, _vp, _vp]),
        "pqto_candidates": (C.c_int64, [_vp, _vp, _vp, _u64, C.POINTER(_u64)]),
        "pqto_knn_batch": (C.c_int, [_vp, _vp, _u64, _u32, _u32, C.c_int, _u64, _u64, _vp, _vp, _vp, _vp]),
        "pqto_attach_database": (None, [_vp, _vp]),
        "pqto_from_shard_view": (_vp, [_vp, _vp, _vp]),
    }

    def __init__(self, index: HostIndex | str):
        so = self.so()
        if hasattr(index, "shard_lo"):  # builder.ShardIndex: one position shard, codes by position
            v = index.view()
            lam = np.ascontiguousarray(index.lambda_q, np.uint8)
            pid = np.ascontiguousarray(index.pair_id).view(np.uint16)
            self._keep = (index, lam, pid)  # borrowed by the oracle
            h = so.pqto_from_shard_view(C.byref(v), _p(lam), _p(pid))
        elif isinstance(index, (str, os.PathLike)):
            h = so.pqto_load(str(index).encode())
        else:
            v = index.view()
            h = so.pqto_from_view(C.byref(v))
        if not h:
            raise RuntimeError("oracle: " + so.pqto_last_error().decode())
        self.h = h
        v = PqtgIndexView()
        so.pqto_view(h, C.byref(v))
        self.config = PqtConfig.from_c(v.config)
        self.n = int(v.n)

    def __del__(self):
        if getattr(self, "h", None):
            self.so().pqto_free(self.h)
            self.h = None

    def host_index(self) -> HostIndex:
        v = PqtgIndexView()
        self.so().pqto_view(self.h, C.byref(v))
        return HostIndex.from_view(v)

    def save(self, path: str) -> None:
        if self.so().pqto_save(self.h, str(path).encode()) != 0:
            raise RuntimeError(self.so().pqto_last_error().decode())

    def attach_database(self, rows: np.ndarray | None) -> None:
        """PqtIndex::attach_database (search.cpp:44-49); the array is kept alive here."""
        if rows is None:
            self._db = None
            self.so().pqto_attach_database(self.h, None)
            return
        rows = np.ascontiguousarray(rows, np.float32)
        if rows.shape != (self.n, self.config.dim):
            raise ValueError("attach_database: vector set does not match index")
        self._db = rows
        self.so().pqto_attach_database(self.h, _p(rows))

    def knn(self, queries: np.ndarray, k: int, threads: int = 0, shard=(0, 0)):
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float32)
        counts = np.zeros(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        rc = self.so().pqto_knn_batch(self.h, _p(q), nq, q.shape[1] if q.ndim == 2 else 0, k, threads,
                                      shard[0], shard[1], _p(ids), _p(dists), _p(counts), _p(stats))
        if rc != 0:
            raise RuntimeError(f"oracle knn ({rc}): " + self.so().pqto_last_error().decode())
        return ids[:, :k], dists[:, :k], counts, stats

    def traverse(self, y: np.ndarray):
        c = self.config
        W = c.w * c.k2
        y = np.ascontiguousarray(y, np.float32)
        fine = np.zeros((c.p_line, c.k1), np.float32)
        l1i = np.zeros((c.p_tree, c.k1), np.uint32)
        l1d = np.zeros((c.p_tree, c.k1), np.float32)
        l2p = np.zeros((c.p_tree, W), np.uint32)
        l2c = np.zeros((c.p_tree, W), np.uint32)
        l2d = np.zeros((c.p_tree, W), np.float32)
        self.so().pqto_traverse(self.h, _p(y), _p(fine), _p(l1i), _p(l1d), _p(l2p), _p(l2c), _p(l2d))
        return dict(fine=fine, l1_id=l1i, l1_dist=l1d, l2_parent=l2p, l2_child=l2c, l2_dist=l2d)

    def candidates(self, y: np.ndarray, cap: int | None = None):
        cap = cap or max(self.config.candidate_budget, 1)
        y = np.ascontiguousarray(y, np.float32)
        pos = np.zeros(cap, np.uint32)
        bins = _u64(0)
        C_ = self.so().pqto_candidates(self.h, _p(y), _p(pos), cap, C.byref(bins))
        if C_ < 0:
            raise RuntimeError(self.so().pqto_last_error().decode())
        return pos[:C_], int(bins.value)

    def heuristic_order(self, lists: np.ndarray, max_bins: int):
        lists = np.ascontiguousarray(lists, np.float32)
        parts, ln = lists.shape
        out = np.zeros((max_bins, parts), np.uint32)
        cnt = self.so().pqto_heuristic_order(self.h, _p(lists), parts, ln, max_bins, _p(out))
        if cnt < 0:
            raise RuntimeError(self.so().pqto_last_error().decode())
        return out[:cnt]

    def line_distance(self, lam: np.ndarray, pid: np.ndarray, fine: np.ndarray) -> float:
        lam = np.ascontiguousarray(lam, np.uint8)
        pid = np.ascontiguousarray(pid, np.uint16)
        fine = np.ascontiguousarray(fine, np.float32)
        return float(self.so().pqto_line_distance(self.h, _p(lam), _p(pid), _p(fine)))

    @classmethod
    def pick_slope_table(cls, a, b) -> int:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return int(cls.so().pqto_pick_slope_table(_p(a), a.size, _p(b), b.size))

    @classmethod
    def encode_slot(cls, parts_i1i2, k1, k2, H) -> int:
        a = np.ascontiguousarray(parts_i1i2, np.uint32).reshape(-1)
        return int(cls.so().pqto_encode_slot(_p(a), a.size // 2, k1, k2, H))


class Ref(_Lib):
    """The reference itself (compiled in place) behind oracle/ref_shim.cpp."""

    _path = REF_SO
    _sigs = {
        "ref_last_error": (C.c_char_p, []),
        "ref_synth_clustered": (C.c_int, [_u64, _u32, _u32, C.c_float, _u64, _vp]),
        "ref_build_index": (_vp, [_vp, _u64, _vp, _u64, C.POINTER(PqtgConfig), C.c_int, C.c_int]),
        "ref_builder_new": (_vp, [_vp, _u64, _vp, C.c_int]),
        "ref_builder_add": (C.c_int, [_vp, _vp, _u64, _u32]),
        "ref_builder_finalize": (_vp, [_vp]),
        "ref_load_index": (_vp, [C.c_char_p]),
        "ref_save_index": (C.c_int, [_vp, C.c_char_p]),
        "ref_free": (None, [_vp]),
        "ref_from_view": (_vp, [C.POINTER(PqtgIndexView)]),
        "ref_index_view": (C.c_int, [_vp, C.POINTER(PqtgIndexView)]),
        "ref_index_database": (_vp, [_vp]),
        "ref_detach_database": (None, [_vp]),
        "ref_attach_database": (C.c_int, [_vp, _vp, _u64]),
        "ref_knn_batch": (C.c_int, [_vp, _vp, _u64, _u32, C.c_int, _vp, _vp, _vp, _vp, _vp]),
        "ref_traverse": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        "ref_heuristic_order": (C.c_int64, [_vp, _vp, _u32, _u32, _u64, _vp]),
        "ref_dijkstra_order": (C.c_int64, [_vp, _u32, _u32, _u64, _vp]),
        "ref_decode_pairs": (C.c_int, [_u32, _u32, _vp]),
        "ref_pick_slope_table": (_u32, [_vp, _u64, _vp, _u64]),
        "ref_build_slope_tables": (C.c_int, [_u32, _vp, _vp]),
        "ref_encode_slot": (_u64, [_vp, _u32, _u32, _u32, _u64]),
        "ref_line_distance": (C.c_float, [_vp, _vp, _vp, _vp]),
        "ref_assign_encode": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp]),
        "ref_brute_force": (C.c_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp]),
    }

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference: " + self.so().ref_last_error().decode())
        self.h = handle
        v = PqtgIndexView()
        self.so().ref_index_view(self.h, C.byref(v))
        self.config = PqtConfig.from_c(v.config)
        self.n = int(v.n)

    def __del__(self):
        if getattr(self, "h", None):
            self.so().ref_free(self.h)
            self.h = None

    # constructors ------------------------------------------------------------------
    @classmethod
    def synth(cls, n: int, dim: int, blobs: int = 1024, sigma: float = 20.0, seed: int = 7) -> np.ndarray:
        out = np.zeros((n, dim), np.float32)
        if cls.so().ref_synth_clustered(n, dim, blobs, sigma, seed, _p(out)) != 0:
            raise RuntimeError(cls.so().ref_last_error().decode())
        return out

    @classmethod
    def build(cls, train: np.ndarray, db: np.ndarray, cfg: PqtConfig, threads: int = 0,
              keep_raw: bool = False) -> "Ref":
        train = np.ascontiguousarray(train, np.float32)
        db = np.ascontiguousarray(db, np.float32)
        c = cfg.to_c()
        h = cls.so().ref_build_index(_p(train), train.shape[0], _p(db), db.shape[0], C.byref(c),
                                     threads, 1 if keep_raw else 0)
        return cls(h)

    @classmethod
    def build_streamed(cls, train: np.ndarray, chunks, cfg: PqtConfig, threads: int = 0) -> "Ref":
        """pqt::IndexBuilder(train, cfg, threads, keep_raw=false), add(chunk) for every chunk of
        the iterable, finalize() (search.cpp:52-117): the reference's wave build."""
        train = np.ascontiguousarray(train, np.float32)
        c = cfg.to_c()
        so = cls.so()
        b = so.ref_builder_new(_p(train), train.shape[0], C.byref(c), threads)
        if not b:
            raise RuntimeError("reference: " + so.ref_last_error().decode())
        try:
            for x in chunks:
                x = np.ascontiguousarray(x, np.float32)
                if so.ref_builder_add(b, _p(x), x.shape[0], cfg.dim) != 0:
                    raise RuntimeError("reference: " + so.ref_last_error().decode())
        except BaseException:
            so.ref_builder_finalize(b)  # frees the builder
            raise
        return cls(so.ref_builder_finalize(b))

    @classmethod
    def load(cls, path: str) -> "Ref":
        return cls(cls.so().ref_load_index(str(path).encode()))

    @classmethod
    def from_host(cls, ix: HostIndex) -> "Ref":
        v = ix.view()
        return cls(cls.so().ref_from_view(C.byref(v)))

    # accessors ---------------------------------------------------------------------
    def save(self, path: str) -> None:
        if self.so().ref_save_index(self.h, str(path).encode()) != 0:
            raise RuntimeError(self.so().ref_last_error().decode())

    def host_index(self) -> HostIndex:
        v = PqtgIndexView()
        if self.so().ref_index_view(self.h, C.byref(v)) != 0:
            raise RuntimeError(self.so().ref_last_error().decode())
        return HostIndex.from_view(v)

    def detach_database(self) -> None:
        self.so().ref_detach_database(self.h)

    def attach_database(self, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows, np.float32)
        if self.so().ref_attach_database(self.h, _p(rows), rows.shape[0]) != 0:
            raise ValueError("reference: " + self.so().ref_last_error().decode())

    def knn(self, queries: np.ndarray, k: int, threads: int = 0, stage_times: bool = False):
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float32)
        counts = np.zeros(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        us = np.zeros((nq, 4), np.float64) if stage_times else None
        if self.so().ref_knn_batch(self.h, _p(q), nq, k, threads, _p(ids), _p(dists), _p(counts),
                                   _p(stats), _p(us)) != 0:
            raise RuntimeError(self.so().ref_last_error().decode())
        out = (ids[:, :k], dists[:, :k], counts, stats)
        return out + (us,) if stage_times else out

    def traverse(self, y: np.ndarray):
        c = self.config
        W = c.w * c.k2
        y = np.ascontiguousarray(y, np.float32)
        fine = np.zeros((c.p_line, c.k1), np.float32)
        l1i = np.zeros((c.p_tree, c.k1), np.uint32)
        l1d = np.zeros((c.p_tree, c.k1), np.float32)
        l2p = np.zeros((c.p_tree, W), np.uint32)
        l2c = np.zeros((c.p_tree, W), np.uint32)
        l2d = np.zeros((c.p_tree, W), np.float32)
        self.so().ref_traverse(self.h, _p(y), _p(fine), _p(l1i), _p(l1d), _p(l2p), _p(l2c), _p(l2d))
        return dict(fine=fine, l1_id=l1i, l1_dist=l1d, l2_parent=l2p, l2_child=l2c, l2_dist=l2d)

    def heuristic_order(self, lists: np.ndarray, max_bins: int):
        lists = np.ascontiguousarray(lists, np.float32)
        parts, ln = lists.shape
        out = np.zeros((max_bins, parts), np.uint32)
        cnt = self.so().ref_heuristic_order(self.h, _p(lists), parts, ln, max_bins, _p(out))
        if cnt < 0:
            raise RuntimeError(self.so().ref_last_error().decode())
        return out[:cnt]

    def line_distance(self, lam, pid, fine) -> float:
        lam = np.ascontiguousarray(lam, np.uint8)
        pid = np.ascontiguousarray(pid, np.uint16)
        fine = np.ascontiguousarray(fine, np.float32)
        return float(self.so().ref_line_distance(self.h, _p(lam), _p(pid), _p(fine)))

    def assign_encode(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float32)
        n = x.shape[0]
        L = self.config.p_line
        codes = np.zeros(n, np.uint64)
        lam = np.zeros((n, L), np.uint8)
        pid = np.zeros((n, L), np.uint16)
        if self.so().ref_assign_encode(self.h, _p(x), n, _p(codes), _p(lam), _p(pid)) != 0:
            raise RuntimeError(self.so().ref_last_error().decode())
        return codes, lam, pid

    @classmethod
    def pick_slope_table(cls, a, b) -> int:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return int(cls.so().ref_pick_slope_table(_p(a), a.size, _p(b), b.size))

    @classmethod
    def dijkstra_order(cls, lists: np.ndarray, max_bins: int):
        lists = np.ascontiguousarray(lists, np.float32)
        parts, ln = lists.shape
        out = np.zeros((max(max_bins, 1), parts), np.uint32)
        cnt = cls.so().ref_dijkstra_order(_p(lists), parts, ln, max_bins, _p(out))
        if cnt < 0:
            raise RuntimeError(cls.so().ref_last_error().decode())
        return out[:cnt]

    @classmethod
    def decode_pairs(cls, k1: int, count: int):
        out = np.zeros((max(count, 1), 2), np.uint16)
        cls.so().ref_decode_pairs(k1, count, _p(out))
        return out[:count]

    @classmethod
    def build_slope_tables(cls, length: int = 4096):
        slopes = np.zeros(10, np.float64)
        entries = np.zeros((10, length, 2), np.uint32)
        cls.so().ref_build_slope_tables(length, _p(slopes), _p(entries))
        return slopes, entries

    @classmethod
    def encode_slot(cls, parts_i1i2, k1, k2, H) -> int:
        a = np.ascontiguousarray(parts_i1i2, np.uint32).reshape(-1)
        return int(cls.so().ref_encode_slot(_p(a), a.size // 2, k1, k2, H))

    @classmethod
    def brute_force(cls, db: np.ndarray, queries: np.ndarray, k: int):
        db = np.ascontiguousarray(db, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        ids = np.zeros((q.shape[0], k), np.uint32)
        dists = np.zeros((q.shape[0], k), np.float32)
        cls.so().ref_brute_force(_p(db), db.shape[0], db.shape[1], _p(q), q.shape[0], k, _p(ids), _p(dists))
        return ids, dists
