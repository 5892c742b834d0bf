"""Sharded search across the GPUs of one box: one process per GPU.

Each rank holds the replicated small state (codebooks, slope streams, offsets, bitmap) and one
contiguous POSITION range of the slot-ordered ids / line codes (pqtg_shard_range). Per batch:

  1. the query batch is broadcast from rank 0 (NCCL over NVLink),
  2. every rank runs traversal and bin selection for all queries (so bins_visited / candidates
     stay global) and re-ranks only the candidates inside its range -> a local top-k by
     (dist, id) (pqtg_search_device),
  3. the per-shard lists are all-gathered (NCCL, k·8 B + 4 B per query per shard),
  4. every rank merges them on its GPU (pqtg_merge_topk_device, the reference's candidate_less
     order), which is bit-identical to the unsharded search (tests/test_gpu_parity.py,
     tests/test_gloo_shard.py).

The exact re-rank stage (raw vectors) is not sharded (pqtg_index_attach_database refuses).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from ._abi import check, lib
from .index import HostIndex
from .search import DeviceIndex, shard_range


class ShardedIndex:
    def __init__(self, hix: "HostIndex | builder.ShardIndex", group=None, device: int | None = None, max_batch: int = 4096):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.cuda.current_device() if device is None else device
        if isinstance(hix, str):  # a PQTINDEX file: this rank loads only its position range
            cfg, n = HostIndex.read_header(hix)
            lo, hi = shard_range(n, self.world, self.rank)
            self.local = DeviceIndex(hix, device=self.device, shard=(lo, hi) if self.world > 1 else (0, 0),
                                     max_batch=max_batch)
            self.shard = (lo, hi)
            self.n = n
            self.dim = cfg.dim
            self._bufs = {}
            return
        if hasattr(hix, "shard_lo"):  # builder.ShardIndex: this rank's shard, built in place
            lo, hi = shard_range(hix.n, self.world, self.rank)
            if (lo, hi) != (hix.shard_lo, hix.shard_hi):
                raise ValueError(f"rank {self.rank} of {self.world} owns positions {lo}..{hi}, "
                                 f"the shard index holds {hix.shard_lo}..{hix.shard_hi}")
            self.local = DeviceIndex(hix, device=self.device, max_batch=max_batch)
        else:
            lo, hi = shard_range(hix.n, self.world, self.rank)
            self.local = DeviceIndex(hix, device=self.device, shard=(lo, hi) if self.world > 1 else (0, 0),
                                     max_batch=max_batch)
        self.shard = (lo, hi)
        self.n = hix.n
        self.dim = hix.config.dim
        self._bufs = {}

    def _buffers(self, nq: int, k: int):
        key = (nq, k)
        if key not in self._bufs:
            dev = torch.device("cuda", self.device)
            G = self.world
            self._bufs[key] = dict(
                ids=torch.empty((nq, k), dtype=torch.int32, device=dev),
                dists=torch.empty((nq, k), dtype=torch.float32, device=dev),
                counts=torch.empty(nq, dtype=torch.int32, device=dev),
                g_ids=torch.empty((G, nq, k), dtype=torch.int32, device=dev),
                g_dists=torch.empty((G, nq, k), dtype=torch.float32, device=dev),
                g_counts=torch.empty((G, nq), dtype=torch.int32, device=dev),
            )
        return self._bufs[key]

    def search(self, d_queries: torch.Tensor, k: int, out_ids: torch.Tensor, out_dists: torch.Tensor,
               out_counts: torch.Tensor, d_stats: torch.Tensor | None = None, broadcast: bool = True,
               exchange: bool | None = None) -> None:
        """Sharded search of the device batch d_queries [nq, dim] (rank 0's batch when
        broadcast) into out_* on every rank, on the current stream. exchange=True forces the
        all-gather + merge even for a single rank (tests)."""
        nq = d_queries.shape[0]
        stream = torch.cuda.current_stream(self.device)
        if self.world > 1 and broadcast:
            dist.broadcast(d_queries, src=0, group=self.group)
        if exchange and not dist.is_initialized():
            raise RuntimeError("exchange needs an initialized process group")
        if self.world == 1 and not exchange:
            self.local.search_device(d_queries.data_ptr(), nq, k, out_ids.data_ptr(), out_dists.data_ptr(),
                                     out_counts.data_ptr(), d_stats.data_ptr() if d_stats is not None else None,
                                     stream.cuda_stream)
            return
        b = self._buffers(nq, k)
        self.local.search_device(d_queries.data_ptr(), nq, k, b["ids"].data_ptr(), b["dists"].data_ptr(),
                                 b["counts"].data_ptr(), d_stats.data_ptr() if d_stats is not None else None,
                                 stream.cuda_stream)
        dist.all_gather_into_tensor(b["g_ids"], b["ids"], group=self.group)
        dist.all_gather_into_tensor(b["g_dists"], b["dists"], group=self.group)
        dist.all_gather_into_tensor(b["g_counts"], b["counts"], group=self.group)
        check(lib().pqtg_merge_topk_device(self.world, nq, k, b["g_ids"].data_ptr(), b["g_dists"].data_ptr(),
                                           b["g_counts"].data_ptr(), out_ids.data_ptr(), out_dists.data_ptr(),
                                           out_counts.data_ptr(), stream.cuda_stream))
