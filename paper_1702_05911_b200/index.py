"""Host-side mirror of the reference's index types (include/pqt/codebook.hpp, search.hpp).

`PqtConfig` mirrors pqt::PqtConfig field for field (codebook.hpp:12-36) with the same
`validate` rules (src/codebook.cpp:15-35) and `resolved_hash_size` (:37-43).
`HostIndex` holds, as numpy arrays, exactly what pqt::PqtIndex holds for the query path
(search.hpp:34-47) in the reference's in-memory layouts; `view()` turns it into the C-ABI
`pqtg_index_view`. `save`/`load` read and write the reference's PQTINDEX v1 container
(src/index_io.cpp:94-229) so indexes move freely between this package and the reference.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import struct
from dataclasses import dataclass, field

import numpy as np

from ._abi import PqtgConfig, PqtgIndexView

MAGIC = b"PQTINDEX"
VERSION = 1


class FormatError(RuntimeError):
    """pqt::FormatError (include/pqt/vecio.hpp:13-16)."""


@dataclass
class PqtConfig:
    dim: int = 128
    p_tree: int = 2
    k1: int = 16
    k2: int = 8
    w: int = 4
    p_line: int = 32
    hash_size: int = 0
    candidate_budget: int = 4096
    rerank_exact: int = 64
    resort_bins: bool = False
    train_iters: int = 25
    seed: int = 42

    def validate(self) -> None:
        def fail(msg: str):
            raise ValueError("config: " + msg)

        if self.dim == 0 or self.p_tree == 0 or self.p_line == 0:
            fail("dim, p_tree and p_line must be positive")
        if self.dim % self.p_tree:
            fail("dim must be divisible by p_tree")
        if self.p_line % self.p_tree:
            fail("p_line must be a multiple of p_tree")
        if self.dim % self.p_line:
            fail("dim must be divisible by p_line")
        if self.k1 < 1 or self.k2 < 1:
            fail("k1 and k2 must be at least 1")
        if self.w < 1 or self.w > self.k1:
            fail("w must be in [1, k1]")

    @property
    def part_dim(self) -> int:
        return self.dim // self.p_tree

    @property
    def fine_dim(self) -> int:
        return self.dim // self.p_line

    @property
    def fine_per_part(self) -> int:
        return self.p_line // self.p_tree

    @property
    def pair_count(self) -> int:
        return 1 if self.k1 <= 1 else self.k1 * (self.k1 - 1) // 2

    def resolved_hash_size(self, n: int) -> int:
        if self.hash_size > 0:
            return self.hash_size
        return max(1, min(1 << 26, 4 * n))

    def to_c(self) -> PqtgConfig:
        c = PqtgConfig()
        for f in dataclasses.fields(self):
            setattr(c, f.name, int(getattr(self, f.name)))
        return c

    @classmethod
    def from_c(cls, c: PqtgConfig) -> "PqtConfig":
        kw = {f.name: getattr(c, f.name) for f in dataclasses.fields(cls)}
        kw["resort_bins"] = bool(kw["resort_bins"])
        return cls(**kw)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


@dataclass
class HostIndex:
    """Arrays of pqt::PqtIndex that the query path reads (config.hash_size resolved)."""

    config: PqtConfig
    n: int
    level1: np.ndarray   # f32 [P, k1, m]
    level2: np.ndarray   # f32 [P, k1, k2, m]
    d2: np.ndarray       # f32 [L, k1, k1]
    slopes: np.ndarray   # f64 [T]
    entries: np.ndarray  # u32 [T, len, 2]
    offsets: np.ndarray  # u64 [H + 1]
    ids: np.ndarray      # u32 [n]
    lambda_q: np.ndarray  # u8 [n, L]
    pair_id: np.ndarray  # u16 [n, L]
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        c = self.config
        P, k1, k2, m, L = c.p_tree, c.k1, c.k2, c.part_dim, c.p_line
        self.level1 = np.ascontiguousarray(self.level1, np.float32).reshape(P, k1, m)
        self.level2 = np.ascontiguousarray(self.level2, np.float32).reshape(P, k1, k2, m)
        self.d2 = np.ascontiguousarray(self.d2, np.float32).reshape(L, k1, k1)
        self.slopes = np.ascontiguousarray(self.slopes, np.float64).reshape(-1)
        self.entries = (np.ascontiguousarray(self.entries, np.uint32).reshape(len(self.slopes), -1, 2)
                        if len(self.slopes) else np.zeros((0, 0, 2), np.uint32))
        self.offsets = np.ascontiguousarray(self.offsets, np.uint64).reshape(-1)
        self.ids = np.ascontiguousarray(self.ids, np.uint32).reshape(-1)
        self.lambda_q = np.ascontiguousarray(self.lambda_q, np.uint8).reshape(self.n, L)
        self.pair_id = np.ascontiguousarray(self.pair_id, np.uint16).reshape(self.n, L)

    # ---- C-ABI view -------------------------------------------------------------------
    def view(self, shard_lo: int = 0, shard_hi: int = 0) -> PqtgIndexView:
        v = PqtgIndexView()
        v.config = self.config.to_c()
        v.n = self.n
        v.level1 = _ptr(self.level1)
        v.level2 = _ptr(self.level2)
        v.d2 = _ptr(self.d2)
        v.table_count = len(self.slopes)
        v.table_len = self.entries.shape[1] if len(self.slopes) else 0
        v.table_slopes = _ptr(self.slopes)
        v.table_entries = _ptr(self.entries)
        v.offsets = _ptr(self.offsets)
        v.ids = _ptr(self.ids)
        v.lambda_q = _ptr(self.lambda_q)
        v.pair_id = _ptr(self.pair_id)
        v.shard_lo = shard_lo
        v.shard_hi = shard_hi
        return v

    @classmethod
    def from_view(cls, v: PqtgIndexView) -> "HostIndex":
        """Deep-copy the arrays a C view points to."""
        cfg = PqtConfig.from_c(v.config)
        P, k1, k2, m, L = cfg.p_tree, cfg.k1, cfg.k2, cfg.part_dim, cfg.p_line
        n = int(v.n)

        def arr(ptr, ctype, count, dtype):
            if count == 0:
                return np.zeros(0, dtype)
            buf = (ctype * count).from_address(ptr)
            return np.frombuffer(buf, dtype=dtype, count=count).copy()

        T, TL = int(v.table_count), int(v.table_len)
        return cls(
            config=cfg,
            n=n,
            level1=arr(v.level1, C.c_float, P * k1 * m, np.float32),
            level2=arr(v.level2, C.c_float, P * k1 * k2 * m, np.float32),
            d2=arr(v.d2, C.c_float, L * k1 * k1, np.float32),
            slopes=arr(v.table_slopes, C.c_double, T, np.float64),
            entries=arr(v.table_entries, C.c_uint32, T * TL * 2, np.uint32).reshape(T, TL, 2),
            offsets=arr(v.offsets, C.c_uint64, cfg.hash_size + 1, np.uint64),
            ids=arr(v.ids, C.c_uint32, n, np.uint32),
            lambda_q=arr(v.lambda_q, C.c_uint8, n * L, np.uint8),
            pair_id=arr(v.pair_id, C.c_uint16, n * L, np.uint16),
        )

    @property
    def pair_width(self) -> int:
        return 1 if self.config.pair_count <= 256 else 2

    # ---- PQTINDEX v1 container (src/index_io.cpp:94-229) -------------------------------
    def save(self, path: str) -> None:
        c = self.config
        hdr = MAGIC + struct.pack(
            "<IIIIIIIQIIBIQ",
            VERSION, c.dim, c.p_tree, c.k1, c.k2, c.w, c.p_line, c.hash_size,
            c.candidate_budget, c.rerank_exact, 1 if c.resort_bins else 0, c.train_iters, c.seed,
        ) + struct.pack("<Q", self.n)
        P, k1, k2, m = c.p_tree, c.k1, c.k2, c.part_dim
        with open(path, "wb") as fp:
            fp.write(hdr)
            for p in range(P):
                fp.write(struct.pack("<II", m, k1))
                fp.write(self.level1[p].tobytes())
            for p in range(P):
                for i in range(k1):
                    fp.write(struct.pack("<II", m, k2))
                    fp.write(self.level2[p, i].tobytes())
            fp.write(self.d2.tobytes())
            fp.write(struct.pack("<II", len(self.slopes), self.entries.shape[1] if len(self.slopes) else 0))
            for t in range(len(self.slopes)):
                fp.write(struct.pack("<d", self.slopes[t]))
                fp.write(self.entries[t].tobytes())
            fp.write(self.offsets.tobytes())
            fp.write(self.ids.tobytes())
            pw = self.pair_width
            fp.write(struct.pack("<B", pw))
            rec = np.empty((self.n * c.p_line, 1 + pw), np.uint8)
            rec[:, 0] = self.lambda_q.reshape(-1)
            if pw == 1:
                rec[:, 1] = self.pair_id.reshape(-1).astype(np.uint8)
            else:
                rec[:, 1:3] = self.pair_id.reshape(-1).astype("<u2").view(np.uint8).reshape(-1, 2)
            fp.write(rec.tobytes())

    @staticmethod
    def read_header(path: str) -> tuple["PqtConfig", int]:
        """(config, n) from a PQTINDEX v1 file's fixed 73-byte header (index_io.cpp:94-106)."""
        with open(path, "rb") as fp:
            buf = fp.read(73)
        if len(buf) < 73 or buf[:8] != MAGIC:
            raise FormatError(f"{path}: bad index magic")
        (version,) = struct.unpack("<I", buf[8:12])
        if version != VERSION:
            raise FormatError(f"{path}: unsupported index version {version}, expected {VERSION}")
        f = struct.unpack("<IIIIIIQIIBIQ", buf[12:65])
        cfg = PqtConfig(dim=f[0], p_tree=f[1], k1=f[2], k2=f[3], w=f[4], p_line=f[5], hash_size=f[6],
                        candidate_budget=f[7], rerank_exact=f[8], resort_bins=bool(f[9]),
                        train_iters=f[10], seed=f[11])
        (n,) = struct.unpack("<Q", buf[65:73])
        return cfg, n

    @classmethod
    def load(cls, path: str) -> "HostIndex":
        with open(path, "rb") as fp:
            buf = fp.read()
        pos = 0

        def take(nbytes: int) -> bytes:
            nonlocal pos
            if pos + nbytes > len(buf):
                raise FormatError(f"{path}: truncated index file")
            out = buf[pos:pos + nbytes]
            pos += nbytes
            return out

        if take(8) != MAGIC:
            raise FormatError(f"{path}: bad index magic")
        (version,) = struct.unpack("<I", take(4))
        if version != VERSION:
            raise FormatError(f"{path}: unsupported index version {version}, expected {VERSION}")
        f = struct.unpack("<IIIIIIQIIBIQ", take(53))
        cfg = PqtConfig(dim=f[0], p_tree=f[1], k1=f[2], k2=f[3], w=f[4], p_line=f[5], hash_size=f[6],
                        candidate_budget=f[7], rerank_exact=f[8], resort_bins=bool(f[9]),
                        train_iters=f[10], seed=f[11])
        cfg.validate()
        (n,) = struct.unpack("<Q", take(8))
        P, k1, k2, m, L = cfg.p_tree, cfg.k1, cfg.k2, cfg.part_dim, cfg.p_line

        def book(k):
            pd, kk = struct.unpack("<II", take(8))
            if pd != m or kk != k:
                raise FormatError(f"{path}: codebook shape does not match config")
            return np.frombuffer(take(4 * pd * kk), np.float32)

        level1 = np.stack([book(k1) for _ in range(P)])
        level2 = np.stack([book(k2) for _ in range(P * k1)])
        d2 = np.frombuffer(take(4 * L * k1 * k1), np.float32)
        T, TL = struct.unpack("<II", take(8))
        slopes = np.zeros(T, np.float64)
        entries = np.zeros((T, TL, 2), np.uint32)
        for t in range(T):
            (slopes[t],) = struct.unpack("<d", take(8))
            entries[t] = np.frombuffer(take(8 * TL), np.uint32).reshape(TL, 2)
        H = cfg.hash_size
        offsets = np.frombuffer(take(8 * (H + 1)), np.uint64)
        ids = np.frombuffer(take(4 * n), np.uint32)
        (pw,) = struct.unpack("<B", take(1))
        if pw not in (1, 2):
            raise FormatError(f"{path}: invalid line-code pair width {pw}")
        rec = np.frombuffer(take(n * L * (1 + pw)), np.uint8).reshape(n * L, 1 + pw)
        lam = rec[:, 0].copy()
        if pw == 1:
            pid = rec[:, 1].astype(np.uint16)
        else:
            pid = np.ascontiguousarray(rec[:, 1:3]).view("<u2").reshape(-1).astype(np.uint16)
        return cls(config=cfg, n=n, level1=level1, level2=level2, d2=d2, slopes=slopes,
                   entries=entries, offsets=offsets, ids=ids, lambda_q=lam, pair_id=pid)
