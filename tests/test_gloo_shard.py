"""Multi-process (world_size 2, gloo, CPU) check of the sharded query path's host logic:
position-range sharding, per-shard top-k, all-gather exchange, merge by (dist, id).

The per-shard re-rank runs in the C oracle here (no GPU in this container); on GPUs the same
exchange carries pqtg_search outputs of shard-restricted device indexes (bench/INTEGRATION)."""
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
    ids, dists, counts, stats = o.knn(g["queries"], k, threads=2, shard=(lo, hi))
    # exchange: every rank gets every shard's top-k (the query-partitioned variant is the same
    # merge on a slice of queries)
    t_ids = torch.from_numpy(ids.astype(np.int64))
    t_d = torch.from_numpy(dists)
    t_c = torch.from_numpy(counts.astype(np.int64))
    g_ids = [torch.zeros_like(t_ids) for _ in range(world)]
    g_d = [torch.zeros_like(t_d) for _ in range(world)]
    g_c = [torch.zeros_like(t_c) for _ in range(world)]
    dist.all_gather(g_ids, t_ids)
    dist.all_gather(g_d, t_d)
    dist.all_gather(g_c, t_c)
    mi, md, mc = merge_topk_host(np.stack([x.numpy() for x in g_ids]).astype(np.uint32),
                                 np.stack([x.numpy() for x in g_d]),
                                 np.stack([x.numpy() for x in g_c]).astype(np.uint32))
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
