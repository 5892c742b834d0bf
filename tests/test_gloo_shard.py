"""Multi-process (world_size 2, gloo, CPU) check of the sharded query path's protocol
(csrc/sharded.cpp, include/pqtg.h "sharded search"): position-range shards, query blocks
(pqtg_shard_range over the batch), each rank's candidate lists for its block exchanged to
every rank, per-shard top-k of the whole batch, all-to-all by query block, merge by (dist, id)
on the block's owner, all-gather of the merged blocks.

The per-shard stages run in the C oracle here (no GPU in this container); on GPUs the same
steps run in libpqtg with NCCL (tests/test_gpu_sharded.py drives them with the local
transport)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, REPO, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir):
    import sys

    sys.path.insert(0, str(REPO))
    from oracle.bindings import Oracle
    from paper_1702_05911_b200 import merge_topk_host, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = load_golden(name)
    path = str(GOLDEN / f"{name}.pqt")
    o = Oracle(path)
    k = int(g["k"])
    lo, hi = shard_range(o.n, world, rank)
    Q = g["queries"]
    nq = len(Q)
    blocks = [shard_range(nq, world, j) for j in range(world)]
    # S1-S4: this rank's block's candidate positions, all-gathered (every rank: the whole batch)
    b0, b1 = blocks[rank]
    mine = [o.candidates(Q[q])[0] for q in range(b0, b1)]
    box = [None] * world
    dist.all_gather_object(box, mine)
    cand = [c for blk in box for c in blk]
    assert len(cand) == nq
    for q in (0, nq - 1):  # the exchanged lists are the global ones
        assert np.array_equal(cand[q], o.candidates(Q[q])[0])
    # S6: this shard's local top-k of the whole batch (its positions only)
    ids, dists, counts, stats = o.knn(Q, k, threads=2, shard=(lo, hi))
    # S7: all-to-all by query block
    send = [(ids[a:b], dists[a:b], counts[a:b]) for (a, b) in blocks]
    recv = [None] * world
    for j in range(world):
        box = [None] * world
        dist.all_gather_object(box, send[j])  # rank j keeps what every rank sent it
        if j == rank:
            recv = box
    # S8: merge this block
    mi, md, mc = merge_topk_host(np.stack([r[0] for r in recv]).astype(np.uint32), np.stack([r[1] for r in recv]),
                                 np.stack([r[2] for r in recv]).astype(np.uint32))
    # S9: all-gather of the merged blocks
    box = [None] * world
    dist.all_gather_object(box, (mi, md, mc))
    mi = np.concatenate([b[0] for b in box])
    md = np.concatenate([b[1] for b in box])
    mc = np.concatenate([b[2] for b in box])
    ok = np.array_equal(mc, g["counts"]) and np.array_equal(stats, g["stats"])
    for q in range(len(mc)):
        c = mc[q]
        ok = ok and np.array_equal(mi[q, :c], g["ids"][q, :c]) and \
            np.array_equal(md[q, :c].view(np.uint32), g["dists"][q, :c].view(np.uint32))
    # each shard really held only part of the candidates
    partial = bool((counts <= g["counts"]).all())
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(f"{int(ok)} {int(partial)}")
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["p2_sift", "p4_gist"])
def test_two_rank_sharded_merge_equals_unsharded(name, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok, partial = (tmp_path / f"r{r}.txt").read_text().split()
        assert ok == "1" and partial == "1"
