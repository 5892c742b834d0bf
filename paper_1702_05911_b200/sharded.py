"""Sharded search across GPUs through the C-ABI's query-partitioned protocol
(include/pqtg.h "sharded search", csrc/sharded.cpp).

Each rank holds the replicated small state (codebooks, slope streams, offsets, bitmap) and one
contiguous POSITION range of the slot-ordered ids / line codes (pqtg_shard_range). Per batch:

  1. rank g runs traversal + bin selection for its block of the queries only;
  2. the blocks' fine LUTs, candidate range lists and counters are all-gathered (NCCL);
  3. every rank re-ranks the batch's candidates that fall in its position range;
  4. all-to-all: rank j receives every rank's top-k lists for its query block and merges them
     by (dist, id) (candidate_less, search.cpp:39-41);
  5. the merged blocks are all-gathered, so every rank holds the whole batch's results --
     bit-identical to the unsharded search.

ShardedIndex: one process per GPU, NCCL communicator owned by libpqtg (its unique id is handed
out through the torch.distributed group). LocalShardedIndex: every shard in this process (one or
several GPUs), the same protocol with device copies -- what the single-GPU tests run.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from ._abi import PqtgError, check, lib
from .index import HostIndex
from .search import DeviceIndex, _raise, shard_range

_vp = C.c_void_p


def _arr(vals):
    return (_vp * len(vals))(*vals)


def load_shard(source, world: int, rank: int, device: int, max_batch: int = 4096) -> DeviceIndex:
    """This rank's position shard of `source` (a PQTINDEX path, a HostIndex, or a
    builder.ShardIndex built for exactly this rank's range)."""
    if hasattr(source, "shard_lo"):
        lo, hi = shard_range(source.n, world, rank)
        if (lo, hi) != (source.shard_lo, source.shard_hi):
            raise ValueError(f"rank {rank} of {world} owns positions {lo}..{hi}, the shard index holds "
                             f"{source.shard_lo}..{source.shard_hi}")
        return DeviceIndex(source, device=device, max_batch=max_batch)
    n = HostIndex.read_header(source)[1] if isinstance(source, str) else source.n
    lo, hi = shard_range(n, world, rank)
    return DeviceIndex(source, device=device, shard=(lo, hi) if world > 1 else (0, 0), max_batch=max_batch)


class _Handle:
    def _search(self, qs, k, ids, dists, counts, stats, streams, broadcast):
        try:
            check(lib().pqtg_sharded_search_device(self._sh, _arr(qs), self._nq, int(k), int(broadcast), _arr(ids),
                                                   _arr(dists), _arr(counts), _arr(stats), _arr(streams)))
        except PqtgError as e:
            _raise(e)

    def stage_ms(self) -> list[float]:
        """[traversal + bin selection of this rank's block, range exchange, re-rank, all-to-all +
        merge + result gather] of the last search, ms (local rank 0)."""
        ms = (C.c_float * 4)()
        check(lib().pqtg_sharded_stage_ms(self._sh, ms))
        return list(ms)

    def counters(self, nq: int, local_rank: int = 0) -> dict:
        """The last batch's per-query candidates (global), tuples consumed (this rank's query
        block only; 0 elsewhere) and candidates inside the rank's position shard."""
        ws = lib().pqtg_sharded_workspace(self._sh, local_rank)
        if not ws:
            raise RuntimeError(lib().pqtg_last_error().decode())
        dev = self.shards[local_rank] if hasattr(self, "shards") else self.local
        lo, hi = int(dev.info.shard_lo), int(dev.info.shard_hi)
        budget = max(min(dev.config.candidate_budget, dev.n), 1)
        pos = np.zeros((nq, budget), np.uint32)
        nc = np.zeros(nq, np.uint32)
        nt = np.zeros(nq, np.uint32)
        check(lib().pqtg_workspace_read(ws, nq, None, None, None, None, pos.ctypes.data, nc.ctypes.data,
                                        nt.ctypes.data))
        valid = np.arange(budget)[None, :] < nc[:, None]
        nl = np.count_nonzero(valid & (pos >= lo) & (pos < hi), axis=1).astype(np.uint32)
        rank = getattr(self, "rank", local_rank)
        world = self.world
        b0, b1 = shard_range(nq, world, rank)
        nt[:b0] = 0
        nt[b1:] = 0
        return dict(ncand=nc, ntuples=nt, nlocal=nl)

    def close(self):
        if getattr(self, "_sh", None):
            lib().pqtg_sharded_destroy(self._sh)
            self._sh = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedIndex(_Handle):
    """One rank of a torch.distributed job (one process per GPU). For the exact stage attach
    this rank's raw rows (its positions' vectors, db[ids[lo:hi]]) with self.local.attach_database."""

    def __init__(self, source, group=None, device: int | None = None, max_batch: int = 4096):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.cuda.current_device() if device is None else device
        # the shard's own workspace is unused (the sharded handle has its own): minimal
        self.local = load_shard(source, self.world, self.rank, self.device, 1)
        self.shard = (int(self.local.info.shard_lo), int(self.local.info.shard_hi))
        self.n = self.local.n
        self.dim = self.local.config.dim
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            check(lib().pqtg_nccl_unique_id(uid))
        if self.world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        sh = _vp()
        try:
            check(lib().pqtg_sharded_create_nccl(self.local.handle, uid, self.rank, self.world, max_batch,
                                                  C.byref(sh)))
        except PqtgError as e:
            _raise(e)
        self._sh = sh

    def search(self, d_queries: torch.Tensor, k: int, out_ids: torch.Tensor, out_dists: torch.Tensor,
               out_counts: torch.Tensor, d_stats: torch.Tensor | None = None, broadcast: bool = True) -> None:
        """Sharded search of the device batch d_queries [nq, dim] (rank 0's, broadcast first when
        `broadcast`) into out_* on every rank, ordered on the current stream. Collective."""
        self._nq = int(d_queries.shape[0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._search([d_queries.data_ptr()], k, [out_ids.data_ptr()], [out_dists.data_ptr()],
                     [out_counts.data_ptr()], [d_stats.data_ptr() if d_stats is not None else None], [stream],
                     broadcast)


class LocalShardedIndex(_Handle):
    """All `world` shards of `source` in this process (devices[g] holds shard g)."""

    def __init__(self, source, world: int, devices=None, max_batch: int = 4096):
        self.world = world
        devices = devices or [0] * world
        self.shards = [load_shard(source, world, g, devices[g], 1) for g in range(world)]
        self.devices = devices
        sh = _vp()
        try:
            check(lib().pqtg_sharded_create_local(_arr([s.handle.value for s in self.shards]), world, max_batch,
                                                   C.byref(sh)))
        except PqtgError as e:
            _raise(e)
        self._sh = sh

    def search(self, d_queries, k, out_ids, out_dists, out_counts, d_stats=None, broadcast=False) -> None:
        """Per-rank lists of device tensors (entry g on devices[g]); ordered on each device's
        current stream."""
        self._nq = int(d_queries[0].shape[0])
        streams = [torch.cuda.current_stream(d).cuda_stream for d in self.devices]
        self._search([q.data_ptr() if q is not None else None for q in d_queries], k,
                     [t.data_ptr() for t in out_ids], [t.data_ptr() for t in out_dists],
                     [t.data_ptr() for t in out_counts],
                     [t.data_ptr() if t is not None else None for t in (d_stats or [None] * self.world)], streams,
                     broadcast)

    def attach_database(self, db: np.ndarray, ids: np.ndarray) -> None:
        """PqtIndex::attach_database (search.cpp:44-49) for every shard: the full n × dim raw
        vectors in id order and the index's inverted-list ids; shard g receives the rows of its
        positions (db[ids[lo:hi]]), and searches then run the exact stage (search.cpp:229-249)
        across the shards."""
        db = np.ascontiguousarray(db, np.float32)
        for dev in self.shards:
            lo, hi = int(dev.info.shard_lo), int(dev.info.shard_hi)
            dev.attach_database(db[np.asarray(ids[lo:hi], np.int64)])

    def search_host(self, queries: np.ndarray, k: int):
        """pqtg_sharded_search: host queries in, host results (rank 0's view) out."""
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float32)
        counts = np.zeros(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        try:
            check(lib().pqtg_sharded_search(self._sh, q.ctypes.data if nq else None, nq, q.shape[1] if q.ndim == 2 else 0,
                                            int(k), ids.ctypes.data, dists.ctypes.data, counts.ctypes.data,
                                            stats.ctypes.data))
        except PqtgError as e:
            _raise(e)
        return ids[:, :k], dists[:, :k], counts, stats


class SimShardedIndex(_Handle):
    """Measurement harness (pqtg_sharded_create_sim): global rank `rank` of a `world`-GPU
    deployment on this one GPU, its peers simulated (their traversal + bin selection computed
    once per batch here, their transfers replaced by device copies of the same bytes). Only this
    rank's device work is timed; results outside its query block are stand-ins."""

    def __init__(self, source, rank: int, world: int, device: int = 0, max_batch: int = 4096):
        self.world, self.rank, self.device = world, rank, device
        self.local = load_shard(source, world, rank, device, 1)
        sh = _vp()
        try:
            check(lib().pqtg_sharded_create_sim(self.local.handle, rank, world, max_batch, C.byref(sh)))
        except PqtgError as e:
            _raise(e)
        self._sh = sh

    def search(self, d_queries, k, out_ids, out_dists, out_counts, d_stats=None, broadcast=False) -> None:
        self._nq = int(d_queries.shape[0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._search([d_queries.data_ptr()], k, [out_ids.data_ptr()], [out_dists.data_ptr()],
                     [out_counts.data_ptr()], [d_stats.data_ptr() if d_stats is not None else None], [stream], False)
