"""Offline index construction on the GPU, producing the reference's index layout.

This is input preparation for benchmarks and large tests, not the measured query path:

* synthetic data: clustered Gaussian blobs like the reference's synth_clustered
  (bench.cpp:66-95) — means uniform in [0, 255]^D, isotropic noise sigma — drawn with a
  torch generator on the GPU in chunks (the reference's single mt19937 stream is not
  chunkable), so 100M-scale sets are cheap;
* codebook training: Lloyd k-means (k-means++-style seeding) per part and per level-1 parent,
  mirroring train_tree's structure (codebook.cpp:229-300); training is not part of the
  parity contract — the GPU query path and the oracle always read the same trained index;
* fine slices / |slice|^2 / pair distances d2: the reference's exact sequential fp32 order
  (linequant.cpp:13-75), computed with numpy float32;
* slope tables: build_slope_tables (binorder.cpp:13-50) restated exactly;
* per-vector bin codes and line codes: pqtg_build_codes (build_kernels.cu), exact
  assign_bin / global_code / encode_line;
* inverted lists: stable sort of slots, i.e. ascending ids within a slot (pqtree.cpp:40-57).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from ._abi import check, lib
from .index import HostIndex, PqtConfig


# ------------------------------------------------------------------------ exact helpers
def fine_slices(level1: np.ndarray, p_line: int) -> np.ndarray:
    """FineCentroids::slices [L, k1, fd] (linequant.cpp:13-46)."""
    P, k1, m = level1.shape
    per = p_line // P
    fd = m // per
    return np.ascontiguousarray(level1.reshape(P, k1, per, fd).transpose(0, 2, 1, 3).reshape(p_line, k1, fd),
                                np.float32)


def seq_sqnorm(sl: np.ndarray) -> np.ndarray:
    """dot(c, c) accumulated sequentially in fp32 (distance.hpp:20-26)."""
    acc = np.zeros(sl.shape[:-1], np.float32)
    for t in range(sl.shape[-1]):
        acc = acc + sl[..., t] * sl[..., t]
    return acc


def pair_d2(sl: np.ndarray) -> np.ndarray:
    """PairDistanceTable::d2 [L, k1, k1]: l2_sq(c_i, c_j) sequentially (linequant.cpp:60-75)."""
    L, k1, fd = sl.shape
    acc = np.zeros((L, k1, k1), np.float32)
    for t in range(fd):
        d = sl[:, :, None, t] - sl[:, None, :, t]
        acc = acc + d * d
    iu = np.triu_indices(k1, 1)
    out = np.zeros_like(acc)
    out[:, iu[0], iu[1]] = acc[:, iu[0], iu[1]]
    out[:, iu[1], iu[0]] = acc[:, iu[0], iu[1]]
    return out


def slope_tables(table_len: int = 4096):
    """build_slope_tables (binorder.cpp:13-50): 10 tables of the table_len smallest (a, b)
    under a + 1.08^k * b, k in [-5, 4], ties lexicographic."""
    slopes = np.zeros(10, np.float64)
    entries = np.zeros((10, table_len, 2), np.uint32)
    for t, k in enumerate(range(-5, 5)):
        slope = math.pow(1.08, k)
        bound = math.sqrt(2.0 * slope * (table_len + 4.0)) + slope + 2.0
        max_a = int(bound) + 1
        max_b = int(bound / slope) + 1
        a, b = np.meshgrid(np.arange(max_a + 1, dtype=np.float64), np.arange(max_b + 1, dtype=np.float64),
                           indexing="ij")
        a = a.reshape(-1)
        b = b.reshape(-1)
        cost = a + slope * b
        order = np.lexsort((b, a, cost))[:table_len]
        slopes[t] = slope
        entries[t, : len(order), 0] = a[order]
        entries[t, : len(order), 1] = b[order]
    return slopes, entries


# ------------------------------------------------------------------------ data + training
def synth_clustered(n: int, dim: int, blobs: int, sigma: float, seed: int, device="cuda", chunk=1 << 20):
    """Clustered synthetic vectors on the GPU (bench.cpp:66-95 distribution), chunkable."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.rand((blobs, dim), generator=g, device=device) * 255.0
    out = torch.empty((n, dim), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = torch.randint(0, blobs, (e - s,), generator=g, device=device)
        out[s:e] = means[pick] + sigma * torch.randn((e - s, dim), generator=g, device=device)
    return out


def _kmeans(x, k: int, iters: int, seed: int):
    """Lloyd iterations with greedy-farthest-style seeding; deterministic for a seed."""
    import torch

    n = x.shape[0]
    g = torch.Generator(device=x.device)
    g.manual_seed(seed)
    if n == 0:
        raise ValueError("empty training set")
    idx = torch.randint(0, n, (1,), generator=g, device=x.device)
    cent = [x[idx[0]]]
    d2 = ((x - cent[0]) ** 2).sum(1)
    for _ in range(1, k):
        p = d2 / d2.sum() if float(d2.sum()) > 0 else torch.full_like(d2, 1.0 / n)
        j = torch.multinomial(p, 1, generator=g)[0]
        cent.append(x[j])
        d2 = torch.minimum(d2, ((x - x[j]) ** 2).sum(1))
    c = torch.stack(cent).clone()
    xx = (x * x).sum(1, keepdim=True)
    for _ in range(iters):
        dist = xx - 2.0 * (x @ c.T) + (c * c).sum(1)[None, :]
        a = dist.argmin(1)
        cnt = torch.bincount(a, minlength=k).to(x.dtype)
        s = torch.zeros_like(c).index_add_(0, a, x)
        live = cnt > 0
        c[live] = s[live] / cnt[live, None]
        if (~live).any():
            far = dist.min(1).values.topk(int((~live).sum())).indices
            c[~live] = x[far]
    return c


def train_tree(train, cfg: PqtConfig, iters: int | None = None):
    """Level-1 codebooks per part and level-2 codebooks per (part, parent)."""
    import torch

    old_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        iters = cfg.train_iters if iters is None else iters
        P, k1, k2, m = cfg.p_tree, cfg.k1, cfg.k2, cfg.part_dim
        level1 = np.zeros((P, k1, m), np.float32)
        level2 = np.zeros((P, k1, k2, m), np.float32)
        g = torch.Generator(device=train.device)
        g.manual_seed(cfg.seed ^ 0x6A69)
        for p in range(P):
            xs = train[:, p * m:(p + 1) * m].contiguous()
            c1 = _kmeans(xs, k1, iters, cfg.seed * 1000 + p)
            level1[p] = c1.cpu().numpy()
            dist = (xs * xs).sum(1, keepdim=True) - 2.0 * (xs @ c1.T) + (c1 * c1).sum(1)[None, :]
            parent = dist.argmin(1)
            for i in range(k1):
                sub = xs[parent == i]
                if sub.shape[0] == 0:
                    jit = (torch.rand((k2, m), generator=g, device=train.device) * 2 - 1) * 1e-6
                    level2[p, i] = (c1[i][None, :] + jit).cpu().numpy()
                    continue
                level2[p, i] = _kmeans(sub, k2, iters, cfg.seed * 1000 + 100 * p + i + 1).cpu().numpy()
        return level1, level2
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old_tf32


# ------------------------------------------------------------------------ index assembly
def encode_database(db, cfg: PqtConfig, level1: np.ndarray, level2: np.ndarray, hash_size: int,
                    chunk: int = 1 << 20):
    """Exact per-vector slots and line codes via pqtg_build_codes (on db's GPU)."""
    import torch

    dev = db.device
    sl = fine_slices(level1, cfg.p_line)
    sq = seq_sqnorm(sl)
    d2 = pair_d2(sl)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    l1, l2, tsl, tsq, td2 = t(level1), t(level2), t(sl), t(sq), t(d2)
    n = db.shape[0]
    L = cfg.p_line
    slots = torch.empty(n, dtype=torch.int64, device=dev)
    lam = torch.empty((n, L), dtype=torch.uint8, device=dev)
    pid = torch.empty((n, L), dtype=torch.int16, device=dev)
    pc = torch.empty((min(n, chunk), cfg.p_tree), dtype=torch.int32, device=dev)
    c = cfg.to_c()
    c.hash_size = hash_size
    stream = torch.cuda.current_stream(dev).cuda_stream
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        x = db[s:e].contiguous()
        check(lib().pqtg_build_codes(C.byref(c), l1.data_ptr(), l2.data_ptr(), tsl.data_ptr(), tsq.data_ptr(),
                                     td2.data_ptr(), x.data_ptr(), e - s, pc.data_ptr(), slots[s:e].data_ptr(),
                                     lam[s:e].data_ptr(), pid[s:e].data_ptr(), stream))
    torch.cuda.synchronize(dev)
    return slots, lam, pid, d2


def build_index(db, train, cfg: PqtConfig, iters: int | None = None) -> HostIndex:
    """Train, encode and assemble an index for `db` (a CUDA float32 tensor n × dim)."""
    import torch

    cfg.validate()
    n = int(db.shape[0])
    H = cfg.resolved_hash_size(n)
    level1, level2 = train_tree(train, cfg, iters)
    slots, lam, pid, d2 = encode_database(db, cfg, level1, level2, H)
    order = torch.sort(slots, stable=True).indices          # ascending ids within a slot
    counts = torch.bincount(slots, minlength=H)
    offsets = torch.zeros(H + 1, dtype=torch.int64, device=db.device)
    offsets[1:] = torch.cumsum(counts, 0)
    slopes, entries = slope_tables(4096)
    out_cfg = PqtConfig(**{**cfg.__dict__})
    out_cfg.hash_size = H
    return HostIndex(
        config=out_cfg, n=n, level1=level1, level2=level2, d2=d2, slopes=slopes, entries=entries,
        offsets=offsets.cpu().numpy().astype(np.uint64), ids=order.to(torch.int32).cpu().numpy().view(np.uint32),
        lambda_q=lam.cpu().numpy(), pair_id=pid.cpu().numpy().view(np.uint16),
    )


# ------------------------------------------------------------------------ sharded billion-scale build
def synth_chunks(n: int, dim: int, blobs: int, sigma: float, seed: int, device="cuda", chunk=1 << 20):
    """The synth_clustered stream chunk by chunk: yields (start, chunk tensor); the same call
    yields the same data again (one generator, consumed in the same order)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.rand((blobs, dim), generator=g, device=device) * 255.0
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = torch.randint(0, blobs, (e - s,), generator=g, device=device)
        yield s, means[pick] + sigma * torch.randn((e - s, dim), generator=g, device=device)


def synth_queries(nq: int, dim: int, blobs: int, sigma: float, seed: int, query_seed: int, device="cuda"):
    """Queries from the same blobs as synth_chunks(seed) but an independent sample stream."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.rand((blobs, dim), generator=g, device=device) * 255.0
    gq = torch.Generator(device=device)
    gq.manual_seed(query_seed)
    pick = torch.randint(0, blobs, (nq,), generator=gq, device=device)
    return means[pick] + sigma * torch.randn((nq, dim), generator=gq, device=device)


class ShardIndex:
    """One inverted-list position shard [shard_lo, shard_hi) of an index over n vectors, as a
    sharded deployment holds it: the whole index's codebooks, tables and offsets, and only this
    shard's ids and line codes, in position order (pqtg_index_create_shard)."""

    def __init__(self, config, n, level1, level2, d2, slopes, entries, offsets, shard_lo, shard_hi, ids,
                 lambda_q, pair_id):
        self.config, self.n = config, n
        self.level1, self.level2, self.d2 = level1, level2, d2
        self.slopes, self.entries, self.offsets = slopes, entries, offsets
        self.shard_lo, self.shard_hi = shard_lo, shard_hi
        self.ids, self.lambda_q, self.pair_id = ids, lambda_q, pair_id

    @property
    def pair_width(self) -> int:
        return 1 if self.config.pair_count <= 256 else 2

    def view(self):
        from .index import PqtgIndexView, _ptr

        v = PqtgIndexView()
        v.config = self.config.to_c()
        v.n = self.n
        v.level1 = _ptr(self.level1)
        v.level2 = _ptr(self.level2)
        v.d2 = _ptr(self.d2)
        v.table_count = len(self.slopes)
        v.table_len = self.entries.shape[1]
        v.table_slopes = _ptr(self.slopes)
        v.table_entries = _ptr(self.entries)
        v.offsets = _ptr(self.offsets)
        v.ids = _ptr(self.ids)  # the shard's ids (positions shard_lo ..)
        v.shard_lo = self.shard_lo
        v.shard_hi = self.shard_hi
        return v


def train_stream_tree(n: int, blobs: int, sigma: float, seed: int, cfg: PqtConfig, ntrain: int, device="cuda",
                      chunk=1 << 20, iters: int | None = None):
    """Codebooks (level1, level2) trained on the first ntrain vectors of synth_chunks(n, ...).
    GPU k-means is not bit-reproducible: a multi-process shard build trains once and
    broadcasts (bench.py)."""
    import torch

    parts = []
    got = 0
    for _, x in synth_chunks(n, cfg.dim, blobs, sigma, seed, device, chunk):
        parts.append(x[: ntrain - got])
        got += parts[-1].shape[0]
        if got >= ntrain:
            break
    train = torch.cat(parts)
    del parts
    return train_tree(train, cfg, iters)


def build_index_sharded(n: int, blobs: int, sigma: float, seed: int, cfg: PqtConfig, shards: int, rank: int,
                        ntrain: int, device="cuda", chunk=1 << 20, iters: int | None = None,
                        tree=None) -> ShardIndex:
    """Build shard `rank` of `shards` of the index over synth_chunks(n, ...) on one GPU without
    holding the whole index: pass 1 assigns every vector's bin (exact assign_bin/global_code),
    a stable sort gives the inverted lists; pass 2 regenerates the stream and encodes only the
    vectors whose list positions fall in this shard (exact encode_line). With the same trained
    codebooks (`tree` = (level1, level2); k-means on the GPU is not bit-reproducible), identical
    for the shard to build_index over all n vectors (tests/test_gpu_topk.py)."""
    import torch

    from .search import shard_range

    cfg.validate()
    dev = torch.device(device)
    H = cfg.resolved_hash_size(n)
    level1, level2 = tree if tree is not None else train_stream_tree(n, blobs, sigma, seed, cfg, ntrain, dev, chunk,
                                                                     iters)
    sl = fine_slices(level1, cfg.p_line)
    sq = seq_sqnorm(sl)
    d2 = pair_d2(sl)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    l1, l2, tsl, tsq, td2 = t(level1), t(level2), t(sl), t(sq), t(d2)
    c = cfg.to_c()
    c.hash_size = H
    stream = torch.cuda.current_stream(dev).cuda_stream
    L = cfg.p_line
    # pass 1: bins of all n vectors
    slots = torch.empty(n, dtype=torch.int32, device=dev)
    pc = torch.empty((chunk, cfg.p_tree), dtype=torch.int32, device=dev)
    sl64 = torch.empty(chunk, dtype=torch.int64, device=dev)
    for s, x in synth_chunks(n, cfg.dim, blobs, sigma, seed, dev, chunk):
        m = x.shape[0]
        check(lib().pqtg_build_codes(C.byref(c), l1.data_ptr(), l2.data_ptr(), tsl.data_ptr(), tsq.data_ptr(),
                                     td2.data_ptr(), x.data_ptr(), m, pc.data_ptr(), sl64.data_ptr(), None, None,
                                     stream))
        slots[s:s + m] = sl64[:m].to(torch.int32)
    counts = torch.bincount(slots, minlength=H)
    offsets = torch.zeros(H + 1, dtype=torch.int64, device=dev)
    offsets[1:] = torch.cumsum(counts, 0)
    del counts
    order = torch.sort(slots, stable=True).indices  # ascending ids within a slot (pqtree.cpp:40-57)
    del slots
    lo, hi = shard_range(n, shards, rank)
    ids = order[lo:hi].to(torch.int32)
    del order
    inv = torch.full((n,), -1, dtype=torch.int32, device=dev)
    inv[ids.long()] = torch.arange(hi - lo, dtype=torch.int32, device=dev)
    # pass 2: line codes of this shard's vectors, written at their positions
    lam = torch.zeros((hi - lo, L), dtype=torch.uint8, device=dev)
    pid = torch.zeros((hi - lo, L), dtype=torch.int16, device=dev)
    for s, x in synth_chunks(n, cfg.dim, blobs, sigma, seed, dev, chunk):
        pos = inv[s:s + x.shape[0]]
        keep = pos >= 0
        if not bool(keep.any()):
            continue
        xs = x[keep].contiguous()
        m = xs.shape[0]
        lc = torch.empty((m, L), dtype=torch.uint8, device=dev)
        pcd = torch.empty((m, L), dtype=torch.int16, device=dev)
        check(lib().pqtg_build_codes(C.byref(c), l1.data_ptr(), l2.data_ptr(), tsl.data_ptr(), tsq.data_ptr(),
                                     td2.data_ptr(), xs.data_ptr(), m, None, None, lc.data_ptr(), pcd.data_ptr(),
                                     stream))
        p = pos[keep].long()
        lam[p] = lc
        pid[p] = pcd
    torch.cuda.synchronize(dev)
    del inv
    slopes, entries = slope_tables(4096)
    out_cfg = PqtConfig(**{**cfg.__dict__})
    out_cfg.hash_size = H
    return ShardIndex(out_cfg, n, level1, level2, d2, slopes, entries, offsets.cpu().numpy().astype(np.uint64),
                      lo, hi, ids.cpu().numpy().view(np.uint32), lam.cpu().numpy(), pid.cpu().numpy().view(np.uint16))
