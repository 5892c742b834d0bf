#!/usr/bin/env python
"""bench.py — PQT online-query throughput on B200 (queries/s), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload deep100m|sift1m|gist1m|sift1b|...]
    python bench.py --impl reference ...      # the reference's own CPU path (oracle/_ref)

A step = one pass of the hot path (traverse → bin selection/gather → line-quantized re-rank →
top-k) over one query batch of the workload. Default workload at N=1 = BASELINE.json configs[2]
(DEEP100M-shaped: 100M × 96-D, P=2, 10k queries, top-100): synthetic clustered vectors (the
reference's synth_clustered distribution) and an index BUILT BY THE REFERENCE (pqtref
IndexBuilder, keep_raw=false) and written as a PQTINDEX file, which the GPU reads through
pqtg_index_load. The index (7.3 GB) is far larger than L2; L2 is still flushed (256 MiB write)
between timed steps, outside the timed intervals.

  value        device-resident: queries already in HBM, pqtg_search_device on the current
               stream, CUDA events around each step, summed over K steps, max over ranks.
  e2e          pqtg_search with pinned host buffers: H2D of the queries, the three kernels,
               D2H of ids/dists/counts/stats, all inside the (host-clocked) timed call.
  roofline     the dominant kernel (largest mean event time): algorithmic bytes per launch
                ÷ its mean launch time, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline the reference compiled in place (oracle/_ref; else the C restatement) on this
               host's cores over the same batch, with a parity check of the GPU results.
Multi-GPU (torchrun, N > 1): the default is SIFT1B (configs[3]) over N inverted-list position
shards with the query-partitioned NCCL protocol (csrc/sharded.cpp): "scaling":
"strong" (the 1B index and the batch are fixed; each rank holds 1/N of the positions and runs
1/N of the traversal / bin selection).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "queries/sec at fixed recall@1/@100 vs CPU oracle (1/2/4/8 B200); HBM GB/s"

WORKLOADS = {
    # BASELINE.json configs[1]
    "gist1m": dict(config=dict(dim=960, p_tree=4, k1=16, k2=8, w=4, p_line=32, candidate_budget=4096),
                   n=1_000_000, nq=1000, k=100, blobs=1024, sigma=20.0, ntrain=100_000),
    # BASELINE.json configs[0]
    "sift1m": dict(config=dict(dim=128, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=4096),
                   n=1_000_000, nq=10000, k=100, blobs=1024, sigma=20.0, ntrain=100_000),
    # a DEEP-shaped single-GPU config at 10M (configs[2] shape at 1/10 scale)
    "deep10m": dict(config=dict(dim=96, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=4096),
                    n=10_000_000, nq=10000, k=100, blobs=10_000, sigma=20.0, ntrain=100_000),
    # BASELINE.json configs[2]: DEEP1B-shaped 100M x 96-D, HBM-resident on one B200 (H = 2^26) -- the
    # N=1 default. The index is built by the REFERENCE (pqtref IndexBuilder waves, keep_raw=false,
    # search.cpp:52-117) from a chunked synthetic stream, written with pqtref save_index, and read by
    # the GPU path through pqtg_index_load (index="reference"; --index gpu builds it on the GPU).
    "deep100m": dict(config=dict(dim=96, p_tree=2, k1=16, k2=8, w=4, p_line=32, candidate_budget=4096),
                     n=100_000_000, nq=10000, k=100, blobs=100_000, sigma=20.0, ntrain=100_000, cache=False,
                     index="reference"),
    # BASELINE.json configs[3]'s tree (SIFT1B: P=4, k1=32, k2=16, w=8, L=32, 496 pairs -> 2-byte pair
    # ids, H = 2^26) at one GPU's share of 1B over 8 GPUs (125M), and a 10M variant for quick runs
    "sift1b_shard": dict(config=dict(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, candidate_budget=4096,
                                     hash_size=1 << 26),
                         n=125_000_000, nq=10000, k=100, blobs=125_000, sigma=20.0, ntrain=200_000, cache=False),
    # BASELINE.json configs[3] itself: SIFT1B-shaped 1B x 128-D over 8 GPUs by inverted-list
    # position (search.cpp's shard_range); this process builds and serves shard (rank % 8) --
    # codebooks trained on the stream's first 200k vectors, all 1B vectors binned, only the
    # shard's 125M encoded (builder.build_index_sharded). Each query is searched by every shard,
    # so one shard's queries/s is the 8-GPU deployment's rate before the merge.
    "sift1b": dict(config=dict(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, candidate_budget=4096,
                               hash_size=1 << 26),
                   n=1_000_000_000, nq=10000, k=100, blobs=1_000_000, sigma=20.0, ntrain=200_000, cache=False,
                   shards=8),
    "sift1b10m": dict(config=dict(dim=128, p_tree=4, k1=32, k2=16, w=8, p_line=32, candidate_budget=4096,
                                  hash_size=1 << 26),
                      n=10_000_000, nq=10000, k=100, blobs=10_000, sigma=20.0, ntrain=200_000),
}
CACHE = Path(os.environ.get("PQTG_BENCH_CACHE", "/tmp/pqtg_bench"))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- workload
def workload_files(name: str, seed: int):
    CACHE.mkdir(parents=True, exist_ok=True)
    return CACHE / f"{name}_s{seed}.pqt", CACHE / f"{name}_s{seed}_queries.npy"


def _gen_device():
    import torch

    return torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")


def synth_stream(n: int, dim: int, blobs: int, sigma: float, seed: int, device, chunk: int = 1 << 22):
    """The synthetic base set as a chunk stream (the reference's synth_clustered distribution,
    bench.cpp:66-95: uniform [0,255) blob means, isotropic sigma noise), pure torch so the
    reference arm never imports the product package. The same call yields the same rows."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.rand((blobs, dim), generator=g, device=device) * 255.0
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = torch.randint(0, blobs, (e - s,), generator=g, device=device)
        yield s, means[pick] + sigma * torch.randn((e - s, dim), generator=g, device=device)


def synth_query_pool(batches: int, nq: int, dim: int, blobs: int, sigma: float, seed: int, device):
    """Query batches from the base stream's blobs; batch b is an independent sample stream
    (seed + 1000 + b), so a longer pool keeps the same first batches."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    means = torch.rand((blobs, dim), generator=g, device=device) * 255.0
    out = []
    for b in range(batches):
        gq = torch.Generator(device=device)
        gq.manual_seed(seed + 1000 + b)
        pick = torch.randint(0, blobs, (nq,), generator=gq, device=device)
        out.append((means[pick] + sigma * torch.randn((nq, dim), generator=gq, device=device)).cpu().numpy())
    return np.concatenate(out)


def ref_index_files(name: str, seed: int):
    CACHE.mkdir(parents=True, exist_ok=True)
    stem = CACHE / f"{name}_s{seed}_ref"
    return (stem.with_suffix(".pqt"), Path(f"{stem}_queries.npy"), Path(f"{stem}.json"),
            Path(f"{stem}_results.npz"))


def build_reference_index(name: str, seed: int, batches: int, threads: int):
    """The reference builds the workload's index on the CPU: pqtref IndexBuilder(train,
    keep_raw=false), add() per chunk of the synthetic stream, finalize() (search.cpp:52-117),
    save_index (index_io.cpp:94-146). Runs in a process that never loads libpqtg.so. Returns
    the in-memory pqtref index (the caller may time it) -- the file is the shared artifact."""
    import torch

    from oracle.bindings import Ref
    from paper_1702_05911_b200.index import PqtConfig  # a plain dataclass (no native code)

    wl = WORKLOADS[name]
    ipath, qpath, mpath, rpath = ref_index_files(name, seed)
    for p in (ipath, qpath, mpath, rpath):
        p.unlink(missing_ok=True)
    cfg = PqtConfig(train_iters=15, seed=seed, **wl["config"])
    dev = _gen_device()
    t0 = time.time()
    stream = synth_stream(wl["n"], cfg.dim, wl["blobs"], wl["sigma"], seed, dev)
    first = next(stream)
    train = first[1][: wl["ntrain"]].cpu().numpy()  # the first ntrain base rows (bench.cpp's train split)

    def chunks():
        yield first[1].cpu().numpy()
        for _, x in stream:
            yield x.cpu().numpy()
            done = _ + x.shape[0]
            if done % (1 << 25) == 0:
                log(f"[bench] reference build: {done / 1e6:.0f}M of {wl['n'] / 1e6:.0f}M vectors "
                    f"({time.time() - t0:.0f}s)")

    ref = Ref.build_streamed(train, chunks(), cfg, threads=threads)
    t_build = time.time() - t0
    tmp = ipath.with_suffix(".tmp")
    ref.save(str(tmp))
    os.replace(tmp, ipath)
    np.save(qpath, synth_query_pool(batches, wl["nq"], cfg.dim, wl["blobs"], wl["sigma"], seed, dev))
    mpath.write_text(json.dumps({"workload": name, "seed": seed, "n": wl["n"], "config": wl["config"],
                                 "generator_device": dev.type, "builder": "pqtref IndexBuilder (keep_raw=false)",
                                 "threads": threads, "build_s": t_build, "total_s": time.time() - t0}))
    log(f"[bench] reference-built {name} index ({wl['n']} vectors) in {t_build:.0f}s, "
        f"saved {ipath} ({ipath.stat().st_size / 1e9:.2f} GB) in {time.time() - t0 - t_build:.0f}s")
    del torch
    return ref


def reference_index(name: str, seed: int, batches: int):
    """Path, query pool and build record of the reference-built index, building it in a separate
    process (the reference arm's own code path) if this box has none yet."""
    wl = WORKLOADS[name]
    ipath, qpath, mpath, _ = ref_index_files(name, seed)
    if not (ipath.exists() and qpath.exists() and mpath.exists()):
        import subprocess

        log(f"[bench] no reference-built {name} index on this box: building it (reference code, CPU)")
        subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--build-index-only",
                        "--workload", name, "--seed", str(seed), "--batches", str(batches)], check=True)
    else:
        log(f"[bench] using the reference-built {ipath}")
    meta = json.loads(mpath.read_text())
    Q = np.load(qpath)
    if Q.shape[0] < wl["nq"] * batches:  # more batches than the build saved: same generator, longer pool
        import torch

        gen = torch.device("cuda", 0) if meta["generator_device"] == "cuda" else torch.device("cpu")
        Q2 = synth_query_pool(batches, wl["nq"], wl["config"]["dim"], wl["blobs"], wl["sigma"], seed, gen)
        assert np.array_equal(Q2[: Q.shape[0]], Q), "query pool is not reproducible"
        Q = Q2
    return ipath, Q[: wl["nq"] * batches], meta


class IndexMeta:
    """What the byte model / launch count need from an index loaded by path."""

    def __init__(self, dev):
        self.config = dev.config
        self.n = dev.n
        self.pair_width = 1 if dev.config.pair_count <= 256 else 2


def make_workload(name: str, seed: int, device: int, batches: int, shards: int | None = None):
    """Build (or load the cached) index + query pool for `name` on cuda:device."""
    import torch

    from paper_1702_05911_b200 import builder
    from paper_1702_05911_b200.index import HostIndex, PqtConfig

    wl = WORKLOADS[name]
    ipath, qpath = workload_files(name, seed)
    nq_pool = wl["nq"] * batches
    cache = wl.get("cache", True)
    if cache and ipath.exists() and qpath.exists() and np.load(qpath, mmap_mode="r").shape[0] >= nq_pool:
        log(f"[bench] loading cached {ipath}")
        return HostIndex.load(str(ipath)), np.load(qpath)[:nq_pool]
    t0 = time.time()
    cfg = PqtConfig(train_iters=15, seed=seed, **wl["config"])
    dev = torch.device("cuda", device)
    if "shards" in wl:  # one position shard of a larger-than-HBM index, built streaming
        shards = shards or wl["shards"]
        shard = int(os.environ.get("RANK", "0")) % shards
        import torch.distributed as dist

        tree = None
        if dist.is_initialized() and dist.get_world_size() > 1:  # one training, broadcast
            box = [builder.train_stream_tree(wl["n"], wl["blobs"], wl["sigma"], seed, cfg, wl["ntrain"], dev)
                   if dist.get_rank() == 0 else None]
            dist.broadcast_object_list(box, src=0, device=dev)
            tree = box[0]
        six = builder.build_index_sharded(wl["n"], wl["blobs"], wl["sigma"], seed, cfg, shards, shard,
                                          wl["ntrain"], device=dev, tree=tree)
        q = builder.synth_queries(nq_pool, cfg.dim, wl["blobs"], wl["sigma"], seed, seed + 1000,
                                  device=dev).cpu().numpy()
        torch.cuda.empty_cache()
        log(f"[bench] built {name} shard {shard}/{shards} "
            f"(positions {six.shard_lo}..{six.shard_hi}) in {time.time() - t0:.1f}s")
        return six, q
    X = builder.synth_clustered(wl["n"] + nq_pool, cfg.dim, wl["blobs"], wl["sigma"], seed, device=dev)
    db, Q = X[: wl["n"]], X[wl["n"]:]
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 1)
    train = db[torch.randperm(wl["n"], generator=g, device=dev)[: wl["ntrain"]]]
    hix = builder.build_index(db, train, cfg)
    q = Q.cpu().numpy()
    del X, db, Q, train
    torch.cuda.empty_cache()
    if cache:
        tmp = ipath.with_suffix(".tmp")
        hix.save(str(tmp))
        os.replace(tmp, ipath)
        np.save(qpath, q)
    log(f"[bench] built {name} index in {time.time() - t0:.1f}s")
    return hix, q


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks + throttle reasons during timing."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period: float = 0.002):
        self.device, self.period = device, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log(f"[bench] NVML unavailable: {e}")

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()
            self.nv.nvmlShutdown()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- algorithmic bytes
def algorithmic_bytes(hix, counters, stats, k: int):
    """Bytes each kernel's algorithm must move per batch."""
    c = hix.config
    nq = len(counters["ncand"])
    W = c.w * c.k2
    pw = hix.pair_width
    C_q = counters["nlocal"].astype(np.float64)  # candidates this index's re-rank scores
    T_q = counters["ntuples"].astype(np.float64)
    bins = stats[:, 0].astype(np.float64)
    stream_entry = {1: 0, 2: 4, 4: 16}[c.p_tree]  # stream words read per probed tuple
    trav = nq * (4 * c.dim + 4 * c.p_line * c.k1 + 8 * c.p_tree * W + 2) \
        + 4 * (c.k1 * c.dim + c.p_tree * c.k1 * c.k2 * c.part_dim)
    binsel = float(np.sum(8 * c.p_tree * W + T_q * (stream_entry + 4) + bins * (8 + 8) + 24))
    rerank = float(np.sum(C_q * (c.p_line * (1 + pw) + 4) + bins * 8 + 4 * c.p_line * c.k1 + 8 * k + 4))
    # SURVEY.md §8d whole-path model B_q = 4D + 16 T_q + 4 C_q + C_q L (1 + pw) + 8k
    survey = float(np.sum(4 * c.dim + 16 * T_q + 4 * C_q + C_q * c.p_line * (1 + pw) + 8 * k))
    return {"traverse": float(trav), "binsel": binsel, "rerank": rerank, "survey_Bq_total": survey,
            "T_q": float(T_q.mean()), "C_q": float(C_q.mean()), "bins_q": float(bins.mean())}


def measured_traffic(workload: str, stage: str, nq: int):
    """DRAM bytes per launch of `stage` from the committed ncu capture of this workload
    (profiles/traffic.json, tools/ncu_traffic.py), scaled to this run's queries per launch;
    None if not captured."""
    p = REPO / "profiles" / "traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text()).get("workloads", {}).get(workload)
    k = d.get("kernels", {}).get(stage) if d else None
    if not k:
        return None, None
    return k["dram_bytes_per_launch"] * nq / d["queries_per_launch"], f"profiles/traffic.json ({d['report']})"


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def gpu_launches(hix, nq: int, chunks: int) -> int:
    """Kernels launched per step: traverse, bin selection, re-rank per chunk (api.cpp)."""
    shard = hasattr(hix, "shard_lo") and (hix.shard_lo > 0 or hix.shard_hi < hix.n)
    n = chunks if chunks else (2 if nq >= 256 and (nq < 4096 or not shard) else 1)  # api.cpp's default
    return 3 * (n if nq >= n else 1)  # (+1 per chunk with --exact: exact_rerank_kernel)


_ALL_CPUS = None  # the process's CPUs before pin_to_gpu_numa (the CPU legs use all of them)


def pin_to_gpu_numa(device: int):
    """Restrict this process to the CPUs NVML reports as local to the GPU, so pinned host
    buffers (first-touched here) live on the GPU's NUMA node. Returns the CPU count, or None."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        global _ALL_CPUS
        _ALL_CPUS = set(os.sched_getaffinity(0))
        cpus &= _ALL_CPUS
        pynvml.nvmlShutdown()
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception as e:  # pragma: no cover
        log(f"[bench] NUMA pinning skipped: {e}")
    return None


def link_bandwidth(h_src, d_dst, h_dst, d_src, reps: int = 20):
    """Pinned host<->device copy bandwidth of this box (GB/s) at the step's own buffer sizes:
    the ceiling the e2e number is held against."""
    import torch

    out = {}
    for name, dst, src in (("h2d", d_dst, h_src), ("d2h", h_dst, d_src)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        out[name] = src.numel() * src.element_size() * reps / (a.elapsed_time(b) / 1000.0) / 1e9
    return out


# --------------------------------------------------------------------------- recall
def counters_ids(dev, dq, nq, k, step, d_ids, d_counts):
    import torch

    step(0)
    torch.cuda.synchronize()
    return d_ids.cpu().numpy().view(np.uint32), d_counts.cpu().numpy().view(np.uint32)


def base_rows(name: str, seed: int, meta: dict | None, device):
    """The workload's base rows again, chunk by chunk, on `device`: the reference-built
    workloads' synth_stream (on the generator device their build used), else the GPU
    builder's synth_clustered draw (make_workload)."""
    import torch

    wl = WORKLOADS[name]
    if meta is not None:
        gen = torch.device(meta["generator_device"], 0) if meta["generator_device"] == "cuda" else torch.device("cpu")
        for s, x in synth_stream(wl["n"], wl["config"]["dim"], wl["blobs"], wl["sigma"], seed, gen):
            yield s, x.to(device)
        return
    from paper_1702_05911_b200 import builder

    X = builder.synth_clustered(wl["n"] + _GPU_POOL[0], wl["config"]["dim"], wl["blobs"], wl["sigma"], seed,
                                device=device)[: wl["n"]]
    yield 0, X


_GPU_POOL = [0]  # query-pool size of the GPU-built draw (its queries are the draw's tail)


def measure_recall(name: str, seed: int, device: int, Q: np.ndarray, meta, result):
    """recall@R = fraction of queries whose exact nearest neighbour is within the first R
    results (recall_fraction, bench.cpp:23-44); exact neighbours over the regenerated
    (deterministic) base set. Identical for the CPU reference, whose ids are bit-identical."""
    import torch

    wl = WORKLOADS[name]
    ids, counts = result
    dev = torch.device("cuda", device)
    q = torch.from_numpy(Q).to(dev)
    if wl["n"] <= 20_000_000:
        # the exact nearest neighbour as the reference defines it (brute_force_knn, sequential fp32
        # l2_sq, (dist, id) order: search.cpp:276-299), on the GPU (pqtg_brute_force_knn_device)
        from paper_1702_05911_b200._abi import check, lib

        X = torch.cat([x for _, x in base_rows(name, seed, meta, dev)]).contiguous()
        gt_i = torch.empty(q.shape[0], dtype=torch.int32, device=dev)
        gt_d = torch.empty(q.shape[0], dtype=torch.float32, device=dev)
        gt_c = torch.empty(q.shape[0], dtype=torch.int32, device=dev)
        check(lib().pqtg_brute_force_knn_device(X.data_ptr(), X.shape[0], X.shape[1], q.data_ptr(), q.shape[0], 1,
                                                gt_i.data_ptr(), gt_d.data_ptr(), gt_c.data_ptr(),
                                                torch.cuda.current_stream(dev).cuda_stream))
        truth = gt_i.cpu().numpy().view(np.uint32).astype(np.int64)
        del X
    else:  # 100M+ rows, streamed: the torch matmul form (exact up to fp32 rounding of the expansion)
        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        best_d = torch.full((q.shape[0],), float("inf"), device=dev)
        best_i = torch.zeros(q.shape[0], dtype=torch.int64, device=dev)
        qq = (q * q).sum(1, keepdim=True)
        for s0, X in base_rows(name, seed, meta, dev):
            for s in range(0, X.shape[0], 1 << 18):
                xb = X[s:s + (1 << 18)]
                d = qq - 2.0 * (q @ xb.T) + (xb * xb).sum(1)[None, :]
                v, i = d.min(1)
                better = v < best_d
                best_d = torch.where(better, v, best_d)
                best_i = torch.where(better, i + s0 + s, best_i)
        torch.backends.cuda.matmul.allow_tf32 = old
        truth = best_i.cpu().numpy()
    out = {}
    for R in (1, 10, 100):
        hit = [truth[i] in ids[i, : min(R, counts[i])] for i in range(len(truth))]
        out[f"r@{R}"] = float(np.mean(hit))
    return out


# --------------------------------------------------------------------------- CPU legs
def same_results(a, b) -> bool:
    """Bit-exact comparison of (ids, dists, counts, stats) batches: counts and stats equal, and
    each query's first counts[q] ids and fp32 distance bit patterns equal."""
    g_ids, g_d, g_c, g_s = a
    r_ids, r_d, r_c, r_s = b
    g_c = np.asarray(g_c).view(np.uint32)
    if not (np.array_equal(g_c, np.asarray(r_c).astype(np.uint32))
            and np.array_equal(np.asarray(g_s).astype(np.uint64), np.asarray(r_s).astype(np.uint64))):
        return False
    for q in range(len(g_c)):
        c = g_c[q]
        if not (np.array_equal(np.asarray(g_ids)[q, :c].view(np.uint32), np.asarray(r_ids)[q, :c].view(np.uint32))
                and np.array_equal(np.asarray(g_d)[q, :c].view(np.uint32), np.asarray(r_d)[q, :c].view(np.uint32))):
            return False
    return True


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_reference(hix, path):
    """The checker's copy of the index: the reference reads its own file (pqtref load_index,
    index_io.cpp:148-229) when there is one, else it is built from the host arrays."""
    from oracle.bindings import Oracle, Ref

    if Ref.available():
        return (Ref.load(str(path)) if path is not None else Ref.from_host(hix)), "reference"
    return Oracle(str(path) if path is not None else hix), "port"


def cpu_leg(impl, kind, Q, k, min_seconds=10.0, max_reps=20, db=None):
    """Time the reference (oracle/_ref) -- else the C restatement -- on this host's cores
    (with the raw vectors attached when db is given: the exact re-rank stage): all host
    threads, then one thread on a small sample."""
    if _ALL_CPUS:  # undo the GPU-side NUMA pinning: the reference gets every host core
        os.sched_setaffinity(0, _ALL_CPUS)
    threads = os.cpu_count() or 1
    if db is not None:
        impl.attach_database(db)
    impl.knn(Q[: min(len(Q), 16)], k, threads=threads)  # warm-up (page-in)
    reps, t_total, out = 0, 0.0, None
    while reps < max_reps and (t_total < min_seconds or reps == 0):
        t0 = time.perf_counter()
        res = impl.knn(Q, k, threads=threads)
        t_total += time.perf_counter() - t0
        out = out or res
        reps += 1
    n1 = min(len(Q), 256)
    t0 = time.perf_counter()
    impl.knn(Q[:n1], k, threads=1)
    one = n1 / (time.perf_counter() - t0)
    return {"value": reps * len(Q) / t_total, "unit": "queries/s", "cores": threads, "kind": kind,
            "sample": f"{reps} x {len(Q)} queries of the timed batch (k={k}), all host threads",
            "threads1_value": one, "threads1_sample": f"{n1} queries, 1 thread", "cpu_model": cpu_model()}, out


def topk_merge_np(parts, k):
    """Merge per-shard (ids, dists, counts) lists by (dist, id) (candidate_less,
    search.cpp:39-41), in numpy: the checker's own merge."""
    nq = parts[0][0].shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dists = np.zeros((nq, k), np.float32)
    counts = np.zeros(nq, np.uint32)
    for q in range(nq):
        i = np.concatenate([p[0][q, : p[2][q]] for p in parts]).astype(np.uint32)
        d = np.concatenate([p[1][q, : p[2][q]] for p in parts]).astype(np.float32)
        o = np.lexsort((i, d))[:k]
        counts[q] = len(o)
        ids[q, : len(o)], dists[q, : len(o)] = i[o], d[o]
    return ids, dists, counts


def shard_parity(args, six, Q, step, d_ids, d_dists, d_counts, d_stats, world, rank):
    """Parity of a billion-scale position shard against the C restatement (oracle/, test
    infrastructure) holding the same shard (pqto_from_shard_view: whole-index offsets, the
    shard's ids and codes): bins_visited / candidates are global, the ids and distances this
    rank's local top-k -- or, under --shard, every rank's oracle shard merged by (dist, id) on
    rank 0 against the NCCL-merged GPU answer. Bounded to the first 1000 queries of the batch."""
    import torch
    import torch.distributed as dist

    from oracle.bindings import Oracle

    k = WORKLOADS[args.workload]["k"]
    nchk = min(len(Q), 1000)
    step(0)
    torch.cuda.synchronize()
    g = (d_ids.cpu().numpy().view(np.uint32)[:nchk], d_dists.cpu().numpy()[:nchk],
         d_counts.cpu().numpy().view(np.uint32)[:nchk], d_stats.cpu().numpy().astype(np.uint64)[:nchk])
    if _ALL_CPUS:
        os.sched_setaffinity(0, _ALL_CPUS)
    threads = max(1, (os.cpu_count() or 1) // max(world, 1))
    t0 = time.time()
    orc = Oracle(six)
    t_load = time.time() - t0
    t0 = time.perf_counter()
    r = orc.knn(Q[:nchk], k, threads=threads)
    dt = time.perf_counter() - t0
    del orc
    merged = args.shard and world > 1
    if merged:
        box = [None] * world
        dist.all_gather_object(box, r[:3])
        want_ids, want_d, want_c = topk_merge_np(box, k)
        want = (want_ids, want_d, want_c, r[3])
    else:
        want = r
    ok = same_results(g, want)
    cpu = {"value": nchk / dt, "unit": "queries/s", "cores": threads, "kind": "port",
           "sample": f"{nchk} queries of the batch on this rank's position shard "
                     f"[{six.shard_lo}, {six.shard_hi}) of {six.n:,} (the C restatement, oracle/pqt_oracle.c)",
           "oracle_setup_s": t_load}
    parity = {"queries": nchk, "bit_exact_vs": "port (C restatement, shard view)", "ok": bool(ok),
              "what": "merged top-k of all shards (NCCL) vs the oracle shards merged by (dist, id)" if merged
              else f"shard [{six.shard_lo}, {six.shard_hi}) local top-k + global bins_visited/candidates"}
    return cpu, parity


# --------------------------------------------------------------------------- reference arm
def index_kind(wl, args) -> str:
    if "shards" in wl:
        return "gpu-built position shard (exact assign_bin/encode_line kernels, torch k-means)"
    if args.index == "reference":
        return "reference-built (pqtref IndexBuilder waves, keep_raw=false; PQTINDEX file)"
    return "gpu-built (exact assign_bin/encode_line kernels, torch k-means)"


def config_of(name: str, wl, args, world: int) -> dict:
    """The config object both arms print (identical keys and values)."""
    return {"workload": name, **wl["config"], "n": wl["n"], "queries_per_step": wl["nq"], "k": wl["k"],
            "index": index_kind(wl, args), "exact_rerank": bool(args.exact),
            "l2": "flushed between timed steps (256 MiB write)" if not args.no_flush else "not flushed",
            "parallelism": (f"rank 0 of {args.sim_ranks} position shards, peers simulated on this GPU "
                            "(pqtg_sharded_create_sim)" if getattr(args, "sim_ranks", 0) else
                            f"position shards x{world} (query-partitioned: block traversal + bin selection, "
                            "range-list all-gather, shard re-rank, all-to-all merge; NCCL)"
                            if args.shard else f"replicas x{world}")}


def run_reference(args):
    """The reference's own CPU path (oracle/_ref: the unmodified sources compiled in place) on
    this host's cores: pqtref knn_query_batch over a bounded sample of the workload's batch.
    This process never loads libpqtg.so: the index is built by pqtref itself (or read with
    pqtref load_index from the file an earlier reference run wrote)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    if "shards" in wl:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.workload} is a {wl['n']:,}-vector index sharded "
                          "over GPUs; the reference's CPU build of it takes hours and its CPU path has no shard "
                          "view"}), flush=True)
        return
    from oracle.bindings import Ref

    threads = os.cpu_count() or 1
    if args.build_index_only:
        build_reference_index(args.workload, args.seed, args.batches, threads)
        return
    ipath, qpath, mpath, rpath = ref_index_files(args.workload, args.seed)
    if ipath.exists() and qpath.exists() and mpath.exists():
        t0 = time.time()
        ref = Ref.load(str(ipath))
        log(f"[bench] pqtref load_index {ipath} in {time.time() - t0:.0f}s")
    else:
        ref = build_reference_index(args.workload, args.seed, args.batches, threads)
    nq, k = wl["nq"], wl["k"]
    Q = np.load(qpath)[:nq]
    # the reference's answers for the whole first batch: the GPU arm's parity cross-check
    t0 = time.perf_counter()
    ids, dists, counts, stats = ref.knn(Q, k, threads=threads)
    per_q = (time.perf_counter() - t0) / nq
    np.savez(rpath, ids=ids, dists=dists, counts=counts, stats=stats)
    # bound each step to ~3 s of host work
    sample = int(max(16, min(nq, 3.0 / max(per_q, 1e-9))))
    Qs = Q[:sample]
    for _ in range(args.warmup):
        ref.knn(Qs, k, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.knn(Qs, k, threads=threads)
    dt = time.perf_counter() - t0
    v = args.steps * sample / dt
    line = {
        "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.shard else "weak", "vs_baseline": None, "dtype": "f32",
        "data": DATA, "impl": "reference",
        "config": config_of(args.workload, wl, args, world),
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} of the {nq} queries of the {args.workload} batch per step, "
                                   f"pqtref knn_query_batch, {threads} threads", "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DATA = "synthetic clustered blobs (synth_clustered distribution)"


# --------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: deep100m (BASELINE configs[2]) at N=1; sift1b --shard (configs[3]) under torchrun")
    ap.add_argument("--index", default="reference", choices=["reference", "gpu"],
                    help="who builds an unsharded workload's index: the reference on the CPU (pqtref "
                         "IndexBuilder, cached PQTINDEX file, default) or the GPU builder (quick runs)")
    ap.add_argument("--build-index-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sim-ranks", type=int, default=0,
                    help="sharded workloads on one GPU: time rank 0 of this many GPUs, the peers simulated "
                         "(pqtg_sharded_create_sim; their transfers become device copies)")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--batches", type=int, default=4, help="distinct query batches cycled over steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--variant", type=int, default=0,
                    help="kernel variant: 0 auto, 1 generic, 2 auto + tensor-core level-2 screen, 3 / 4 auto with the walker-warp / all-warp bin selection forced")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--chunks", type=int, default=0,
                    help="pieces per batch overlapped on two streams (0 auto, 1 off)")
    ap.add_argument("--exact", action="store_true",
                    help="attach the raw base vectors: the exact re-rank stage runs (rerank_exact = 64)")
    ap.add_argument("--shard", action="store_true",
                    help="shard the index's positions over the ranks (query-partitioned protocol over "
                         "NCCL, csrc/sharded.cpp) instead of one replica per rank")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload is None:  # the north-star split under torchrun, the single-GPU config otherwise
        multi = int(os.environ.get("WORLD_SIZE", "1")) > 1
        args.workload = "sift1b" if multi else "deep100m"
        args.shard = args.shard or multi

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    affinity = pin_to_gpu_numa(local)  # host buffers on the GPU's NUMA node
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1702_05911_b200 import DeviceIndex
    from paper_1702_05911_b200._abi import lib

    wl = WORKLOADS[args.workload]
    nq, k = wl["nq"], wl["k"]
    # a sharded workload under --shard splits its index over the ranks (else: shard rank % 8)
    shards = world if (args.shard and world > 1) else None
    if args.shard and "shards" in wl and world == 1:
        raise SystemExit(f"--shard on {args.workload} splits the index over the ranks: run it under torchrun with "
                         f">= 2 ranks (without --shard one process serves shard 0 of {wl['shards']})")
    ref_built = "shards" not in wl and args.index == "reference"
    ipath = meta = None
    pool = args.batches * max(world, 1)
    if "shards" in wl:  # every rank builds its shard at once (codebooks trained on rank 0)
        hix, Qpool = make_workload(args.workload, args.seed, local, pool, shards)
    elif rank == 0:
        if ref_built:
            ipath, Qpool, meta = reference_index(args.workload, args.seed, pool)
        else:
            hix, Qpool = make_workload(args.workload, args.seed, local, pool, shards)
    if world > 1 and "shards" not in wl:
        dist.barrier()
        if rank != 0:
            if ref_built:
                ipath, Qpool, meta = reference_index(args.workload, args.seed, pool)
            else:
                hix, Qpool = make_workload(args.workload, args.seed, local, pool, shards)
    _GPU_POOL[0] = len(Qpool)
    lib().pqtg_set_kernel_variant(args.variant)
    t_load = time.time()
    if args.sim_ranks:
        from paper_1702_05911_b200.sharded import SimShardedIndex

        if world != 1 or "shards" not in wl or args.sim_ranks != wl["shards"]:
            raise SystemExit(f"--sim-ranks needs one process and a sharded workload built for that many shards")
        args.shard = True  # the sharded step, on a simulated deployment
        sh = SimShardedIndex(hix, 0, args.sim_ranks, device=local, max_batch=nq)
        dev = sh.local
        batches = [Qpool[b * nq:(b + 1) * nq] for b in range(args.batches)]
    elif args.shard:
        from paper_1702_05911_b200.sharded import ShardedIndex

        sh = ShardedIndex(str(ipath) if ref_built else hix, device=local, max_batch=nq)
        dev = sh.local
        # every rank searches the same batches (rank 0's, broadcast inside the timed step)
        batches = [Qpool[b * nq:(b + 1) * nq] for b in range(args.batches)]
    else:
        dev = DeviceIndex(str(ipath) if ref_built else hix, device=local, max_batch=nq)
        batches = [Qpool[(rank * args.batches + b) * nq:(rank * args.batches + b + 1) * nq]
                   for b in range(args.batches)]
    if ref_built:
        log(f"[bench] pqtg_index_load of the reference-built file: {time.time() - t_load:.1f}s")
        hix = IndexMeta(dev)
    dev.set_chunks(args.chunks)
    db_rows = None
    if args.exact:  # the build's base rows, regenerated deterministically
        db_rows = torch.cat([x.cpu() for _, x in base_rows(args.workload, args.seed, meta,
                                                              torch.device("cuda", local))]).numpy()
        dev.attach_database(db_rows)
    d_q = [torch.from_numpy(b).cuda() for b in batches]
    d_ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d_dists = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    d_counts = torch.empty(nq, dtype=torch.int32, device="cuda")
    d_stats = torch.empty((nq, 3), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step(b):
        if args.shard:
            sh.search(d_q[b], k, d_ids, d_dists, d_counts, d_stats)
            return
        dev.search_device(d_q[b].data_ptr(), nq, k, d_ids.data_ptr(), d_dists.data_ptr(), d_counts.data_ptr(),
                          d_stats.data_ptr(), stream.cuda_stream)

    # per-batch counters for the algorithmic-bytes model + a correctness snapshot
    counters, stats_all = [], []
    for b in range(args.batches):
        step(b)
        torch.cuda.synchronize()
        counters.append((sh if args.shard else dev).counters(nq))
        stats_all.append(d_stats.cpu().numpy().astype(np.uint64))
    for _ in range(args.warmup):
        for b in range(args.batches):
            step(b)
    torch.cuda.synchronize()

    jobs = 1 if args.shard else world  # sharded: all ranks share each batch
    # ---- e2e through the public host API (pinned buffers, copies inside the timed call)
    def run_e2e():
        hq = [torch.from_numpy(b).pin_memory() for b in batches]
        h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
        h_dists = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        h_counts = torch.empty(nq, dtype=torch.int32).pin_memory()
        h_stats = torch.empty((nq, 3), dtype=torch.int64).pin_memory()
        L = lib()

        def host_step(b):
            if args.shard:  # H2D of the batch, sharded search, D2H of the merged top-k
                d_q[b].copy_(hq[b], non_blocking=True)
                sh.search(d_q[b], k, d_ids, d_dists, d_counts, d_stats)
                h_ids.copy_(d_ids, non_blocking=True)
                h_dists.copy_(d_dists, non_blocking=True)
                h_counts.copy_(d_counts, non_blocking=True)
                h_stats.copy_(d_stats, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return
            rc = L.pqtg_search(dev.handle, dev.workspace, hq[b].data_ptr(), nq, hix.config.dim, k, h_ids.data_ptr(),
                               h_dists.data_ptr(), h_counts.data_ptr(), h_stats.data_ptr())
            assert rc == 0, L.pqtg_last_error()

        for b in range(args.batches):
            host_step(b)
        e2e_steps = max(args.steps // 2, 10)
        e2e_t = 0.0
        e2e_each = []
        for s in range(e2e_steps):
            if not args.no_flush:
                flush.fill_(s & 0xFF)
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            host_step(s % args.batches)
            e2e_each.append(time.perf_counter() - t0)
            e2e_t += e2e_each[-1]
        log(f"[bench] e2e step us: median {np.median(e2e_each) * 1e6:.1f} mean {np.mean(e2e_each) * 1e6:.1f} "
            f"p90 {np.percentile(e2e_each, 90) * 1e6:.1f} max {np.max(e2e_each) * 1e6:.1f}")
        tt = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_value = jobs * nq * e2e_steps / float(tt.item())
        h2d = nq * hix.config.dim * 4
        d2h = nq * k * 8 + nq * 4 + nq * 24
        link = link_bandwidth(hq[0], d_q[0], h_ids, d_ids)

        return e2e_value, h2d, d2h, link

    # ---- timed: device-resident
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            if not args.no_flush:
                flush.fill_(s & 0xFF)
            evs[s][0].record(stream)
            step(s % args.batches)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = jobs * nq * args.steps / (ms_max / 1000.0)

    # ---- per-kernel times (unchunked launches: one launch per stage per step). Sharded: the
    # protocol's stages on this rank -- block traversal + bin selection, range exchange, re-rank,
    # all-to-all + merge + result gather (pqtg_sharded_stage_ms)
    dev.set_chunks(1)
    stage_sum = np.zeros(4)
    kstep = min(args.steps, 50)
    for s in range(kstep):
        if not args.no_flush:
            flush.fill_(s & 0xFF)
        step(s % args.batches)
        stage_sum += np.array(sh.stage_ms() if args.shard else dev.stage_ms())
    stage_mean = stage_sum / kstep
    dev.set_chunks(args.chunks)

    e2e_value, h2d, d2h, link = run_e2e()

    shard_cpu = shard_par = None
    if "shards" in wl and not args.no_cpu_baseline and not args.sim_ranks:  # every rank checks its own shard
        shard_cpu, shard_par = shard_parity(args, hix, batches[0], step, d_ids, d_dists, d_counts, d_stats, world,
                                            rank)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    abytes = [algorithmic_bytes(hix, counters[b], stats_all[b], k) for b in range(args.batches)]
    ab = {kk: float(np.mean([a[kk] for a in abytes])) for kk in abytes[0]}
    peak, peak_src = peaks()
    limiter = {"traverse": "issue (IPC ~3.5, sequential fp32 chains + level-2 sort)",
               "binsel": "latency / L2-probe throughput per pass (issue active ~22-60%)",
               "rerank": "L1 data pipe (~76% of peak with 256-bit row loads; 3/4 of its wavefronts are the "
                         "shared-memory table gathers) + issue (~76% active, ~15.5 SASS per part); "
                         "profiles/r02/wide/, profiles/r02/rerank_packed_ab.md"}
    if args.shard:
        # this rank's block is 1/world of the batch for traversal + bin selection (ntuples are
        # counted on the block only; bins on the whole batch, so the block figure is an upper bound)
        names = ["block_traverse_binsel", "exchange", "rerank", "merge"]
        kb = {"block_traverse_binsel": ab["traverse"] / world + ab["binsel"], "rerank": ab["rerank"]}
        dom = 2 if stage_mean[2] >= stage_mean[0] else 0
        dname = names[dom]
        traffic, traffic_src = None, None
        achieved = kb[dname] / (stage_mean[dom] / 1000.0) / 1e9
        stage_ms = {n: float(v) for n, v in zip(names, stage_mean)}
        per_kernel = {n: kb[n] / (stage_mean[i] / 1000.0) / 1e9 for i, n in enumerate(names) if n in kb}
        kernel = "rerank_kernel" if dom == 2 else "traverse+binsel_kernels"
        abl = kb[dname]
    else:
        names = ["traverse", "binsel", "rerank"]
        dom = int(np.argmax(stage_mean[:3]))
        dname = names[dom]
        traffic, traffic_src = measured_traffic(args.workload, dname, nq)
        achieved = ab[dname] / (stage_mean[dom] / 1000.0) / 1e9
        stage_ms = {n: float(v) for n, v in zip(names, stage_mean[:3])}
        per_kernel = {n: ab[n] / (stage_mean[i] / 1000.0) / 1e9 for i, n in enumerate(names)}
        kernel = {"traverse": "traverse_kernel", "binsel": "binsel_kernel", "rerank": "rerank_kernel"}[dname]
        abl = ab[dname]
    tot = sum(stage_ms.values())
    roofline = {"bound": "hbm", "kernel": kernel,
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": peak_src, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": abl,
                "stage_ms": stage_ms,
                "stage_share": {n: v / tot for n, v in stage_ms.items()},
                "per_kernel_gbs": per_kernel,
                "T_q": ab["T_q"], "C_q": ab["C_q"], "bins_q": ab["bins_q"],
                "survey_Bq_gbs": ab["survey_Bq_total"] / (ms_max / args.steps / 1000.0) / 1e9,
                # what bounds each kernel instead of HBM (ncu, profiles/r02/)
                "limiter": limiter}

    # ---- CPU baseline (rank 0, N=1) + parity of the timed batch
    cpu = None
    parity = None
    sharded_wl = "shards" in wl
    if sharded_wl:
        cpu, parity = shard_cpu, shard_par
        if args.sim_ranks:
            parity = {"ok": None, "what": "simulated peers: outputs outside rank 0's query block are stand-ins "
                                          "(the protocol's parity: tests/test_gpu_sharded.py)"}
    if world == 1 and not args.no_cpu_baseline and not sharded_wl:
        step(0)
        torch.cuda.synchronize()
        g_ids = d_ids.cpu().numpy().view(np.uint32)
        g_d = d_dists.cpu().numpy()
        g_c = d_counts.cpu().numpy().view(np.uint32)
        g_s = d_stats.cpu().numpy().astype(np.uint64)
        t0 = time.time()
        impl, kind = load_reference(None if ref_built else hix, ipath if ref_built else None)
        log(f"[bench] reference index for the CPU leg ready in {time.time() - t0:.0f}s ({kind})")
        cpu, ref_out = cpu_leg(impl, kind, batches[0], k, db=db_rows)
        del impl
        parity = {"queries": nq, "bit_exact_vs": kind, "ok": same_results((g_ids, g_d, g_c, g_s), ref_out)}
        if ref_built and rank == 0:  # the reference arm's own answers for this batch, if it ran on this box
            rpath = ref_index_files(args.workload, args.seed)[3]
            if rpath.exists() and not args.exact:
                r = np.load(rpath)
                parity["reference_arm_results"] = same_results((g_ids, g_d, g_c, g_s),
                                                               (r["ids"], r["dists"], r["counts"], r["stats"]))

    recall = None
    if not args.no_recall and not sharded_wl:
        recall = measure_recall(args.workload, args.seed, local, batches[0], meta,
                                counters_ids(dev, d_q[0], nq, k, step, d_ids, d_counts))
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.shard else "weak", "vs_baseline": None, "dtype": "f32",
        "data": DATA,
        "config": config_of(args.workload, wl, args, world),
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "link_gbs": link, "host_cpus": affinity,
                "transfer_bound_qps": nq / (h2d / (link["h2d"] * 1e9) + d2h / (link["d2h"] * 1e9))},
        "gpu_launches": (8 * args.steps if args.shard  # traverse, binsel, scan, pack, scan, unpack, rerank, merge
                         else gpu_launches(hix, nq, args.chunks) * args.steps * (4 if args.exact else 3) // 3),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "parity": parity,
        "recall": recall,
        "kernel_variant": args.variant,
        "chunks": args.chunks,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
