// api.cpp — the C ABI (include/pqtg.h): index lifecycle, PQTINDEX v1 loader, workspaces and
// the search orchestration (K1 traverse → K3 bin selection/gather → K5 re-rank/top-k).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "pqtg_internal.h"

namespace pqtg {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

namespace {
std::atomic<int> g_variant{0};
}
int kernel_variant() { return g_variant.load(std::memory_order_relaxed); }
const char* last_error() { return g_last_error.c_str(); }

Workspace::~Workspace() {
    if (index) cudaSetDevice(index->device);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (join) cudaEventDestroy(join);
    if (fork) cudaEventDestroy(fork);
    if (done) cudaEventDestroy(done);
    if (h_qtime) cudaFreeHost(h_qtime);
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    for (void* p : allocations) cudaFree(p);
}

// throws the error the kernels flagged in the workspace's error word (the stream is synchronised)
void check_ws_error(const Workspace& ws) {
    uint32_t e = 0;
    PQTG_CUDA_CHECK(cudaMemcpy(&e, ws.err, sizeof(e), cudaMemcpyDeviceToHost));
    if (e & PQTG_WS_ERR_HEAP)
        throw Error{PQTG_ERR_UNSUPPORTED, "exact bin order: the tuple heap outgrew shared memory"};
}

WsSlice Workspace::slice(uint64_t q0) const {
    const DevParams& p = index->prm;
    WsSlice s;
    s.fine = fine + q0 * p.L * p.k1;
    s.l2_dist = l2_dist + q0 * p.P * p.W;
    s.l2_code = l2_code + q0 * p.P * p.W;
    s.slope = slope + q0 * 2;
    s.ranges = ranges + q0 * std::max<uint64_t>(p.budget, 1);
    s.nranges = nranges + q0;
    s.ncand = ncand + q0;
    s.ntuples = ntuples + q0;
    s.err = err;
    s.keys = keys ? keys + q0 * std::max<uint64_t>(p.budget, 1) : nullptr;
    s.split_keys = split_keys;
    s.split_ctr = split_ctr;
    s.split_q = split_q;
    s.split_k = split_k;
    s.hash = hash ? hash + q0 * hash_stride : nullptr;
    s.bscr = bscr ? bscr + q0 * bscr_stride : nullptr;
    s.scr = scr ? scr + q0 * p.P * p.scr_nj : nullptr;
    return s;
}

namespace {

template <class F>
int guarded(F&& fn) {
    try {
        return fn();
    } catch (const Error& e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return PQTG_ERR_OOM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PQTG_ERR_ARG;
    }
}

void ensure_staging(Workspace& ws, uint64_t k) {
    const DevParams& p = ws.index->prm;
    if (!ws.d_queries) {
        ws.d_queries = dev_alloc<float>(ws.allocations, ws.max_batch * p.D);
        ws.d_counts = dev_alloc<uint32_t>(ws.allocations, ws.max_batch);
        ws.d_stats = dev_alloc<pqtg_query_stats>(ws.allocations, ws.max_batch);
    }
    if (k > ws.stage_k) {
        // grow: old buffers stay owned by the workspace until it is destroyed
        ws.d_ids = dev_alloc<uint32_t>(ws.allocations, ws.max_batch * k);
        ws.d_dists = dev_alloc<float>(ws.allocations, ws.max_batch * k);
        ws.stage_k = k;
        ++ws.gen;
    }
}

// Chunk boundaries of a host-buffer sub-batch of b queries: chunk c+1's H2D copy hides under
// chunk c's kernels. Two equal chunks measured best on B200 (tools/e2e_probe.py: growing
// plans such as 1:3:4 expose less of the first copy but pay the latency-bound traversal and
// bin-selection kernels once more). ws.chunks > 0 forces that many equal chunks;
// PQTG_CHUNK_PLAN="w1,w2,..." sets relative chunk sizes (experiments).
std::vector<uint64_t> host_chunks(const Workspace& ws, uint64_t b) {
    std::vector<uint64_t> w;
    if (ws.chunks) {
        w.assign(ws.chunks, 1);
    } else if (const char* env = std::getenv("PQTG_CHUNK_PLAN")) {
        for (const char* c = env; *c;) {
            char* end = nullptr;
            const unsigned long v = std::strtoul(c, &end, 10);
            if (end == c) break;
            if (v) w.push_back(v);
            c = *end ? end + 1 : end;
        }
    } else if (b >= 4096) {
        // small first / last chunks: only they expose their copies (the first H2D, the last D2H);
        // DEEP100M 10k queries, host-call median: 1,1,1,1 1.75 ms, 1,2,2,1 1.64, 1,3,3,3,1 1.65,
        // 1,4,4,1 1.60 ms (profiles/r02/e2e_chunk_plans.md)
        w = {1, 4, 4, 1};
    } else if (b >= 256) {
        w = {1, 1};
    }
    if (w.empty()) w = {1};
    uint64_t tot = 0;
    for (uint64_t x : w) tot += x;
    std::vector<uint64_t> bounds{0};
    uint64_t acc = 0;
    for (uint64_t x : w) {
        acc += x;
        const uint64_t e = b * acc / tot;
        if (e > bounds.back()) bounds.push_back(e);
    }
    if (bounds.back() != b) bounds.push_back(b);
    return bounds;
}

// k' of the line-ranked prefix the exact stage re-ranks: max(k, rerank_exact), at most the
// candidate budget (C <= budget).
uint32_t exact_prefix(const DevParams& p, uint32_t k) {
    const uint32_t kp = std::max(k, p.rerank_exact);
    return std::min(kp, std::max<uint32_t>(p.budget, 1));
}

// Buffers of the line-ranked prefix for the exact stage (only with raw vectors attached).
// the re-rank's key buffer in HBM when a query's keys do not fit shared memory (large budgets)
void ensure_keys(Workspace& ws, uint32_t k) {
    const DevParams& p = ws.index->prm;
    const uint32_t kk = (p.db && p.rerank_exact > 0 && k) ? exact_prefix(p, k) : k;
    // the split re-rank of small batches: per-(slice, query) lists
    const uint64_t sq = std::min<uint64_t>(ws.max_batch, kSplitBelow);
    if (kk && rerank_split(p, 1, kk) > 1 && (ws.split_k < kk || ws.split_q < sq)) {
        ws.split_keys = dev_alloc<uint64_t>(ws.allocations, (uint64_t)kSplitMax * sq * kk);
        ws.split_ctr = dev_alloc<uint32_t>(ws.allocations, sq);
        PQTG_CUDA_CHECK(cudaMemset(ws.split_ctr, 0, sq * sizeof(uint32_t)));
        ws.split_q = sq;
        ws.split_k = kk;
        ++ws.gen;
    }
    if (ws.keys || kk == 0 || !rerank_needs_gkeys(p, kk)) return;
    ws.keys = dev_alloc<uint64_t>(ws.allocations, ws.max_batch * std::max<uint64_t>(p.budget, 1));
    ++ws.gen;
}

void ensure_exact(Workspace& ws, uint32_t k) {
    const DevParams& p = ws.index->prm;
    if (!p.db || p.rerank_exact == 0 || k == 0) return;
    const uint32_t kp = exact_prefix(p, k);
    if (!ws.ex_counts) ws.ex_counts = dev_alloc<uint32_t>(ws.allocations, ws.max_batch);
    if (kp > ws.ex_cap) {  // grow: old buffers stay owned by the workspace
        ws.ex_ids = dev_alloc<uint32_t>(ws.allocations, ws.max_batch * kp);
        ws.ex_dists = dev_alloc<float>(ws.allocations, ws.max_batch * kp);
        ws.ex_cap = kp;
        ++ws.gen;
    }
    ws.ex_k = kp;
}


}  // namespace

// a position shard's exact stage needs the other shards' prefixes: it runs in the sharded search
void refuse_shard_exact(const DevParams& p) {
    if (p.db && p.rerank_exact > 0 && (p.shard_lo != 0 || p.shard_hi != p.n))
        throw Error{PQTG_ERR_UNSUPPORTED, "exact re-ranking of a position shard runs in the sharded search (pqtg_sharded_*)"};
}

void prepare_workspace(Workspace& ws, uint32_t k) {
    ensure_exact(ws, k);
    ensure_keys(ws, k);
}

namespace {

// A stage event: an external event node when s is being captured (a plain record there only
// orders the capture and is never timed), a plain record otherwise.
void record_stage(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    PQTG_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
    PQTG_CUDA_CHECK(cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                                        : cudaEventRecord(e, s));
}

// The three stages for queries [q0, q0 + nq) of the current sub-batch on stream s. Events
// ev[0..3] bracket the stages when `timed` (the first chunk of a call); recorded as external
// events, so a captured search (CUDA graph) records them when it replays.
void run_chunk(const DevIndex& ix, Workspace& ws, uint64_t q0, const float* d_queries, uint64_t nq, uint32_t k,
               uint32_t* d_ids, float* d_dists, uint32_t* d_counts, pqtg_query_stats* d_stats, cudaStream_t s,
               bool timed, unsigned long long* h_qt = nullptr) {
    DevParams p = ix.prm;
    // small chunks are launch-latency bound: their stages run as one PDL chain, without the stage
    // events between the kernels (pqtg_workspace_stage_ms then reports the whole search only;
    // pqtg_workspace_query_times has the per-stage clocks). PQTG_CHAIN=0 disables, =all chains
    // every chunk.
    static const int chain_mode = [] {
        const char* e = std::getenv("PQTG_CHAIN");
        return !e ? 1 : std::strcmp(e, "0") == 0 ? 0 : std::strcmp(e, "all") == 0 ? 2 : 1;
    }();
    p.chain = chain_mode == 2 || (chain_mode == 1 && nq < kChainBelow) ? 1u : 0u;
    if (timed) ws.stages_timed = !p.chain;
    if (ws.qtime_on && nq) {  // per-query stage clocks of this chunk (pqtg_workspace_query_times)
        p.qtime = ws.qtime + q0 * 6;
        PQTG_CUDA_CHECK(cudaMemsetAsync(p.qtime, 0, nq * 6 * sizeof(unsigned long long), s));
    }
    if (timed) record_stage(ws.ev[0], s);
    if (nq == 0 || k == 0 || ix.n == 0) {  // search.cpp:130-132: empty results, zero stats
        if (nq) {
            PQTG_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, nq * sizeof(uint32_t), s));
            if (d_stats) PQTG_CUDA_CHECK(cudaMemsetAsync(d_stats, 0, nq * sizeof(pqtg_query_stats), s));
            if (k && ix.n == 0) {
                PQTG_CUDA_CHECK(cudaMemsetAsync(d_ids, 0xFF, nq * k * sizeof(uint32_t), s));
                PQTG_CUDA_CHECK(cudaMemsetAsync(d_dists, 0x7F, nq * k * sizeof(float), s));
            }
        }
        if (timed)
            for (int i = 1; i < 4; ++i) record_stage(ws.ev[i], s);
        if (h_qt && p.qtime && nq)
            PQTG_CUDA_CHECK(cudaMemcpyAsync(h_qt, p.qtime, nq * 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        return;
    }
    const WsSlice sl = ws.slice(q0);
    launch_traverse(p, d_queries, nq, sl, s);
    if (timed && !p.chain) record_stage(ws.ev[1], s);
    launch_binsel(p, nq, sl, d_stats, s);
    if (timed && !p.chain) record_stage(ws.ev[2], s);
    if (p.db && p.rerank_exact > 0) {
        // exact re-rank (search.cpp:229-249): K5 keeps the k' = max(k, rerank_exact) best by
        // line distance (the reference's partial_sort prefix, :239-240), K6 replaces their
        // distances by exact ones and returns the first min(k, C)
        const uint32_t kp = exact_prefix(p, k);
        launch_rerank(p, nq, kp, sl, ws.ex_ids + q0 * ws.ex_k, ws.ex_dists + q0 * ws.ex_k, ws.ex_counts + q0, s);
        launch_exact(p, d_queries, nq, (uint32_t)ws.ex_k, ws.ex_ids + q0 * ws.ex_k, ws.ex_counts + q0, k, d_ids,
                     d_dists, d_counts, d_stats, s);
    } else {
        launch_rerank(p, nq, k, sl, d_ids, d_dists, d_counts, s);
    }
    if (timed) record_stage(ws.ev[3], s);
    if (h_qt && p.qtime)
        PQTG_CUDA_CHECK(cudaMemcpyAsync(h_qt, p.qtime, nq * 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
}

// The cached CUDA graph of `enqueue` (work captured on stream cs, which forks to and joins
// back from the workspace's aux stream) for these arguments, captured on a miss; least
// recently used of at most 8 evicted.
template <class F>
cudaGraphExec_t cached_graph(Workspace& ws, const uint64_t (&key)[12], cudaStream_t cs, F&& enqueue) {
    Workspace::GraphEntry* hit = nullptr;
    for (auto& g : ws.graphs)
        if (std::memcmp(g.key, key, sizeof(key)) == 0) hit = &g;
    if (!hit) {
        cudaGraph_t graph = nullptr;
        PQTG_CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            PQTG_CUDA_CHECK(cudaEventRecord(ws.fork, cs));
            PQTG_CUDA_CHECK(cudaStreamWaitEvent(ws.aux_stream, ws.fork, 0));
            enqueue();
            PQTG_CUDA_CHECK(cudaEventRecord(ws.fork, ws.aux_stream));
            PQTG_CUDA_CHECK(cudaStreamWaitEvent(cs, ws.fork, 0));
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            throw;
        }
        PQTG_CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        PQTG_CUDA_CHECK(e);
        if (ws.graphs.size() >= 8) {  // evict the least recently used
            auto lru = std::min_element(ws.graphs.begin(), ws.graphs.end(),
                                        [](const auto& x, const auto& y) { return x.used < y.used; });
            cudaGraphExecDestroy(lru->exec);
            ws.graphs.erase(lru);
        }
        Workspace::GraphEntry g{};
        std::memcpy(g.key, key, sizeof(key));
        g.exec = exec;
        ws.graphs.push_back(g);
        hit = &ws.graphs.back();
    }
    hit->used = ++ws.graph_clock;
    return hit->exec;
}

}  // namespace
}  // namespace pqtg

using namespace pqtg;

extern "C" {

int pqtg_abi_version(void) { return PQTG_ABI_VERSION; }

int pqtg_set_kernel_variant(int variant) {
    if (variant < 0 || variant > 4) {
        set_error("variant must be 0 (auto), 1 (generic), 2 (auto with the tensor-core level-2 screen), 3 "
                  "(auto with the walker-warp bin selection) or 4 (auto with the all-warp bin selection)");
        return PQTG_ERR_ARG;
    }
    g_variant.store(variant);
    return PQTG_OK;
}

const char* pqtg_last_error(void) { return last_error(); }

int pqtg_device_ok(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return 0;
    }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
    return prop.major == 10 ? 1 : 0;
}

int pqtg_index_create(const pqtg_index_view* v, int device, pqtg_index** out) {
    return guarded([&] {
        if (!v || !out) throw Error{PQTG_ERR_ARG, "null argument"};
        *out = nullptr;
        validate_config(v->config);
        const uint64_t n = v->n;
        if (!v->level1 || !v->level2 || !v->d2 || !v->offsets || (n && (!v->ids || !v->lambda_q || !v->pair_id)) ||
            (v->table_count && (!v->table_entries || !v->table_slopes)))
            throw Error{PQTG_ERR_ARG, "index view has null arrays"};
        Source s;
        s.cfg = v->config;
        s.n = n;
        s.level1 = v->level1;
        s.level2 = v->level2;
        s.d2 = v->d2;
        s.table_count = v->table_count;
        s.table_len = v->table_len;
        s.slopes = v->table_slopes;
        s.entries = v->table_entries;
        s.offsets = v->offsets;
        s.ids = v->ids;
        s.lambda_q = v->lambda_q;
        s.pair_id = v->pair_id;
        auto* h = new pqtg_index;
        h->dev.reset(build_device_index(s, device, v->shard_lo, v->shard_hi));
        *out = h;
        return PQTG_OK;
    });
}

int pqtg_index_create_shard(const pqtg_index_view* v, const uint8_t* shard_lambda_q, const uint16_t* shard_pair_id,
                            int device, pqtg_index** out) {
    return guarded([&] {
        if (!v || !out) throw Error{PQTG_ERR_ARG, "null argument"};
        *out = nullptr;
        validate_config(v->config);
        const uint64_t n = v->n;
        if (v->shard_hi <= v->shard_lo || v->shard_hi > n) throw Error{PQTG_ERR_ARG, "bad shard range"};
        if (!v->level1 || !v->level2 || !v->d2 || !v->offsets || !v->ids || !shard_lambda_q || !shard_pair_id ||
            (v->table_count && (!v->table_entries || !v->table_slopes)))
            throw Error{PQTG_ERR_ARG, "index view has null arrays"};
        Source s;
        s.cfg = v->config;
        s.n = n;
        s.level1 = v->level1;
        s.level2 = v->level2;
        s.d2 = v->d2;
        s.table_count = v->table_count;
        s.table_len = v->table_len;
        s.slopes = v->table_slopes;
        s.entries = v->table_entries;
        s.offsets = v->offsets;
        s.ids = v->ids;
        s.pos_lambda_q = shard_lambda_q;
        s.pos_pair_id = shard_pair_id;
        auto* h = new pqtg_index;
        h->dev.reset(build_device_index(s, device, v->shard_lo, v->shard_hi));
        *out = h;
        return PQTG_OK;
    });
}

int pqtg_index_load(const char* path, int device, uint64_t shard_lo, uint64_t shard_hi, pqtg_index** out) {
    return guarded([&] {
        if (!path || !out) throw Error{PQTG_ERR_ARG, "null argument"};
        *out = nullptr;
        LoadedFile lf;
        parse_index(path, lf);
        auto* h = new pqtg_index;
        h->dev.reset(build_device_index(lf.src, device, shard_lo, shard_hi));
        *out = h;
        return PQTG_OK;
    });
}

int pqtg_index_info_get(const pqtg_index* index, pqtg_index_info* out) {
    return guarded([&] {
        if (!index || !out) throw Error{PQTG_ERR_ARG, "null argument"};
        const DevIndex& d = *index->dev;
        std::memset(out, 0, sizeof(*out));
        out->config = d.cfg;
        out->n = d.n;
        out->shard_lo = d.prm.shard_lo;
        out->shard_hi = d.prm.shard_hi;
        out->list_len = d.prm.W;
        out->pair_count = d.prm.npairs;
        out->pair_width = d.prm.pw;
        out->code_row_bytes = d.prm.row_bytes;
        out->device_bytes = d.bytes;
        out->device = d.device;
        return PQTG_OK;
    });
}

int pqtg_index_attach_database(pqtg_index* index, const float* rows, uint64_t n, uint32_t dim) {
    return guarded([&] {
        if (!index) throw Error{PQTG_ERR_ARG, "null argument"};
        DevIndex& d = *index->dev;
        PQTG_CUDA_CHECK(cudaSetDevice(d.device));
        auto release = [&] {
            if (d.db || d.id2row) PQTG_CUDA_CHECK(cudaDeviceSynchronize());
            if (d.db) cudaFree(d.db);
            if (d.id2row) cudaFree(d.id2row);
            d.db = nullptr;
            d.id2row = nullptr;
            d.prm.db = nullptr;
            d.prm.id2row = nullptr;
        };
        if (!rows) {  // detach
            release();
            return PQTG_OK;
        }
        // search.cpp:44-49: the vector set must match the index -- all n rows in id order, or, on a
        // position shard, the shard's rows in position order (db[ids[lo..hi)])
        const bool shard = d.prm.shard_lo != 0 || d.prm.shard_hi != d.n;
        const uint64_t want = shard ? d.prm.shard_hi - d.prm.shard_lo : d.n;
        if (n != want || dim != d.prm.D)
            throw Error{PQTG_ERR_BAD_DIM, "attach_database: vector set does not match index"};
        float* buf = nullptr;
        uint32_t* map = nullptr;
        const uint32_t stride = (dim + 3) / 4 * 4;  // 16-byte rows for the exact stage's bulk copies
        const size_t bytes = (size_t)n * stride * sizeof(float);
        cudaError_t e = cudaMalloc(&buf, bytes ? bytes : 16);
        if (e == cudaSuccess && shard) e = cudaMalloc(&map, (size_t)std::max<uint64_t>(d.n, 1) * sizeof(uint32_t));
        if (e != cudaSuccess) {
            cudaFree(buf);
            throw Error{PQTG_ERR_OOM, std::string("attach_database: ") + cudaGetErrorString(e)};
        }
        if (stride != dim) e = cudaMemset(buf, 0, bytes);
        if (e == cudaSuccess && n)
            e = cudaMemcpy2D(buf, stride * sizeof(float), rows, dim * sizeof(float), dim * sizeof(float), n,
                             cudaMemcpyHostToDevice);
        if (e == cudaSuccess && shard) {  // id -> row of this shard's rows (ids of other shards: none)
            e = cudaMemset(map, 0xFF, (size_t)d.n * sizeof(uint32_t));
            if (e == cudaSuccess) {
                launch_fill_id2row(d.prm.ids, n, map, nullptr);
                e = cudaDeviceSynchronize();
            }
        }
        if (e != cudaSuccess) {
            cudaFree(buf);
            cudaFree(map);
            throw Error{PQTG_ERR_CUDA, std::string("attach_database: ") + cudaGetErrorString(e)};
        }
        release();
        d.db = buf;
        d.id2row = map;
        d.prm.db = buf;
        d.prm.id2row = map;
        d.prm.db_stride = stride;
        return PQTG_OK;
    });
}

void pqtg_index_destroy(pqtg_index* index) { delete index; }

int pqtg_workspace_create(const pqtg_index* index, uint64_t max_batch, pqtg_workspace** out) {
    return guarded([&] {
        if (!index || !out || max_batch == 0) throw Error{PQTG_ERR_ARG, "bad workspace arguments"};
        *out = nullptr;
        const DevIndex& d = *index->dev;
        const DevParams& p = d.prm;
        PQTG_CUDA_CHECK(cudaSetDevice(d.device));
        auto ws = std::make_unique<Workspace>();
        ws->index = &d;
        ws->max_batch = max_batch;
        PQTG_CUDA_CHECK(cudaStreamCreateWithFlags(&ws->own_stream, cudaStreamNonBlocking));
        PQTG_CUDA_CHECK(cudaStreamCreateWithFlags(&ws->aux_stream, cudaStreamNonBlocking));
        PQTG_CUDA_CHECK(cudaEventCreateWithFlags(&ws->join, cudaEventDisableTiming));
        PQTG_CUDA_CHECK(cudaEventCreateWithFlags(&ws->fork, cudaEventDisableTiming));
        PQTG_CUDA_CHECK(cudaEventCreateWithFlags(&ws->done, cudaEventDisableTiming));
        PQTG_CUDA_CHECK(cudaEventRecord(ws->done, ws->own_stream));
        for (auto& e : ws->ev) PQTG_CUDA_CHECK(cudaEventCreate(&e));
        const uint64_t B = max_batch;
        ws->fine = dev_alloc<float>(ws->allocations, B * p.L * p.k1);
        ws->l2_dist = dev_alloc<float>(ws->allocations, B * p.P * p.W);
        ws->l2_code = dev_alloc<uint32_t>(ws->allocations, B * p.P * p.W);
        ws->slope = dev_alloc<uint8_t>(ws->allocations, B * 2);
        ws->ranges = dev_alloc<uint2>(ws->allocations, B * std::max<uint64_t>(p.budget, 1));
        ws->nranges = dev_alloc<uint32_t>(ws->allocations, B);
        ws->ncand = dev_alloc<uint32_t>(ws->allocations, B);
        ws->ntuples = dev_alloc<uint32_t>(ws->allocations, B);
        ws->err = dev_alloc<uint32_t>(ws->allocations, 1);
        PQTG_CUDA_CHECK(cudaMemset(ws->err, 0, sizeof(uint32_t)));
        ws->hash_words = binsel_fast_ok(p) ? binsel_hash_words(p, B) : 0;
        ws->hash_stride = ws->hash_words ? std::max(binsel_hash_stride(p), binsel_par_hash_stride(p)) : 0;
        ws->hash_words = ws->hash_stride * B;
        if (ws->hash_words) ws->hash = dev_alloc<uint32_t>(ws->allocations, ws->hash_words);
        ws->bscr_stride = binsel_scratch_stride(p);
        if (ws->bscr_stride) ws->bscr = dev_alloc<uint64_t>(ws->allocations, B * ws->bscr_stride);
        if (screen_ok(p)) {
            ws->scr = dev_alloc<float>(ws->allocations, B * p.P * p.scr_nj);
        }
        auto* h = new pqtg_workspace;
        h->ws = std::move(ws);
        *out = h;
        return PQTG_OK;
    });
}

void pqtg_workspace_destroy(pqtg_workspace* ws) { delete ws; }

int pqtg_workspace_set_chunks(pqtg_workspace* h, uint32_t chunks) {
    return guarded([&] {
        if (!h) throw Error{PQTG_ERR_ARG, "null argument"};
        h->ws->chunks = chunks;
        ++h->ws->gen;
        return PQTG_OK;
    });
}

int pqtg_workspace_stage_ms(pqtg_workspace* h, float* ms4) {
    return guarded([&] {
        if (!h || !ms4) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        PQTG_CUDA_CHECK(cudaEventSynchronize(ws.ev[3]));
        for (int i = 0; i < 3; ++i) {
            ms4[i] = -1.0f;  // a chained search has no events between its stages
            if (ws.stages_timed) PQTG_CUDA_CHECK(cudaEventElapsedTime(&ms4[i], ws.ev[i], ws.ev[i + 1]));
        }
        PQTG_CUDA_CHECK(cudaEventElapsedTime(&ms4[3], ws.ev[0], ws.ev[3]));
        check_ws_error(ws);
        return PQTG_OK;
    });
}

// diagnostic: the re-rank's phase clocks of CTA (0, 0) of its last launch (PQTG_PHASES=1), ns
int pqtg_debug_rerank_phases(uint64_t* out16) {
    return guarded([&] {
        unsigned long long* b = phase_buffer();
        if (!b || !out16) throw Error{PQTG_ERR_ARG, "phase clocks are off (PQTG_PHASES=1 enables them)"};
        PQTG_CUDA_CHECK(cudaDeviceSynchronize());
        PQTG_CUDA_CHECK(cudaMemcpy(out16, b, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        return PQTG_OK;
    });
}

int pqtg_workspace_query_times(pqtg_workspace* h, int enable) {
    return guarded([&] {
        if (!h) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        std::lock_guard<std::mutex> lock(ws.mu);
        PQTG_CUDA_CHECK(cudaSetDevice(ws.index->device));
        if (enable && !ws.qtime) ws.qtime = dev_alloc<unsigned long long>(ws.allocations, ws.max_batch * 6);
        ws.qtime_on = enable != 0;
        ++ws.gen;
        return PQTG_OK;
    });
}

int pqtg_workspace_read_query_times(pqtg_workspace* h, uint64_t nq, float* us) {
    return guarded([&] {
        if (!h || (nq && !us)) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        std::lock_guard<std::mutex> lock(ws.mu);
        if (!ws.qtime_on) throw Error{PQTG_ERR_ARG, "per-query times are not enabled on this workspace"};
        PQTG_CUDA_CHECK(cudaSetDevice(ws.index->device));
        std::vector<unsigned long long> raw;
        const unsigned long long* src = nullptr;
        if (ws.qtime_host) {
            if (nq > ws.qtime_cap) throw Error{PQTG_ERR_ARG, "nq exceeds the last search"};
            PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.own_stream));
            src = ws.h_qtime;
        } else {
            if (nq > ws.last_nq) throw Error{PQTG_ERR_ARG, "nq exceeds the last searched batch"};
            if (ws.last_stream) PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.last_stream));
            PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.aux_stream));
            raw.resize(nq * 6);
            PQTG_CUDA_CHECK(cudaMemcpy(raw.data(), ws.qtime, nq * 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            src = raw.data();
        }
        for (uint64_t q = 0; q < nq * 3; ++q) {
            const unsigned long long start = ~src[2 * q], end = src[2 * q + 1];
            us[q] = (src[2 * q] && end >= start) ? (float)((double)(end - start) * 1e-3) : 0.0f;
        }
        return PQTG_OK;
    });
}

// diagnostic: the raw per-query stage clocks (globaltimer ns: [q][stage][start, end]) of the last
// pqtg_search_device call with per-query times on
int pqtg_debug_query_clocks(pqtg_workspace* h, uint64_t nq, uint64_t* out) {
    return guarded([&] {
        if (!h || (nq && !out)) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        std::lock_guard<std::mutex> lock(ws.mu);
        if (!ws.qtime_on || ws.qtime_host || nq > ws.last_nq)
            throw Error{PQTG_ERR_ARG, "no per-query clocks of a device-entry search of this size"};
        if (ws.last_stream) PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.last_stream));
        PQTG_CUDA_CHECK(cudaMemcpy(out, ws.qtime, nq * 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < nq * 3; ++i) out[2 * i] = ~out[2 * i];
        return PQTG_OK;
    });
}

int pqtg_workspace_status(pqtg_workspace* h) {
    return guarded([&] {
        if (!h) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        std::lock_guard<std::mutex> lock(ws.mu);
        PQTG_CUDA_CHECK(cudaSetDevice(ws.index->device));
        if (ws.last_stream) PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.last_stream));
        PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.aux_stream));
        check_ws_error(ws);
        return PQTG_OK;
    });
}

int pqtg_workspace_read(pqtg_workspace* h, uint64_t nq, float* fine, uint32_t* l2_code, float* l2_dist,
                        uint8_t* slope, uint32_t* positions, uint32_t* ncand, uint32_t* ntuples) {
    return guarded([&] {
        if (!h) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *h->ws;
        const DevParams& p = ws.index->prm;
        if (nq > ws.last_nq) throw Error{PQTG_ERR_ARG, "nq exceeds the last searched batch"};
        PQTG_CUDA_CHECK(cudaSetDevice(ws.index->device));
        if (ws.last_stream || ws.own_stream) PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.last_stream));
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) PQTG_CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        };
        cp(fine, ws.fine, nq * p.L * p.k1 * sizeof(float));
        cp(l2_code, ws.l2_code, nq * p.P * p.W * sizeof(uint32_t));
        cp(l2_dist, ws.l2_dist, nq * p.P * p.W * sizeof(float));
        cp(slope, ws.slope, nq * 2);
        std::vector<uint32_t> nc(nq), nr(nq);
        cp(nc.data(), ws.ncand, nq * 4);
        cp(nr.data(), ws.nranges, nq * 4);
        if (ncand) std::memcpy(ncand, nc.data(), nq * 4);
        cp(ntuples, ws.ntuples, nq * 4);
        if (positions && p.budget) {
            std::vector<uint2> rg(nq * p.budget);
            cp(rg.data(), ws.ranges, rg.size() * sizeof(uint2));
            for (uint64_t q = 0; q < nq; ++q) {
                uint32_t* out = positions + q * p.budget;
                const uint2* r = rg.data() + q * p.budget;
                for (uint32_t b = 0; b < nr[q]; ++b) {
                    const uint32_t end = b + 1 < nr[q] ? r[b + 1].y : nc[q];
                    for (uint32_t j = r[b].y; j < end; ++j) out[j] = r[b].x + (j - r[b].y);
                }
            }
        }
        return PQTG_OK;
    });
}

int pqtg_search_device(pqtg_index* index, pqtg_workspace* wsh, const float* d_queries, uint64_t nq, uint32_t k,
                       uint32_t* d_ids, float* d_dists, uint32_t* d_counts, pqtg_query_stats* d_stats,
                       void* stream) {
    return guarded([&] {
        if (!index || !wsh || (nq && (!d_queries || !d_counts || (k && (!d_ids || !d_dists)))))
            throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *wsh->ws;
        if (ws.index != index->dev.get()) throw Error{PQTG_ERR_ARG, "workspace belongs to another index"};
        if (nq > ws.max_batch) throw Error{PQTG_ERR_ARG, "nq exceeds the workspace max_batch"};
        std::lock_guard<std::mutex> lock(ws.mu);  // the workspace's host state (buffers, chunking)
        PQTG_CUDA_CHECK(cudaSetDevice(index->dev->device));
        refuse_shard_exact(index->dev->prm);
        ensure_exact(ws, k);
        ensure_keys(ws, k);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // every previous call's work on these slices, its aux-stream chunks included (they are
        // joined back before it records ws.done), is behind ws.done; a call on the same stream as
        // the last one is ordered after it already (one API call less on the latency path)
        if (s != ws.last_stream) PQTG_CUDA_CHECK(cudaStreamWaitEvent(s, ws.done, 0));
        if (index->dev->prm.exact_order) PQTG_CUDA_CHECK(cudaMemsetAsync(ws.err, 0, sizeof(uint32_t), s));
        ws.last_stream = s;
        ws.qtime_host = false;
        ws.last_nq = nq;
        // device-resident batches: two chunks on two streams, so the next chunk's traversal and bin
        // selection fill the SMs the re-rank's last wave leaves idle (tools/e2e_probe.py on B200,
        // 1000 GIST queries: 1 chunk 234 us, 2 chunks 207 us, 4 chunks 261 us). A position shard's
        // short re-rank gains nothing from the overlap once every stage runs many waves (SIFT1B
        // shard, 10k queries: 0.97 ms unchunked vs 1.13 ms; SIFT1M, unsharded: 1.26 vs 1.24 ms).
        const DevParams& pp = index->dev->prm;
        const bool shard = pp.shard_hi > pp.shard_lo && (pp.shard_lo > 0 || pp.shard_hi < pp.n);
        const uint64_t nch = ws.chunks ? ws.chunks : (nq >= 256 && (nq < 4096 || !shard) ? 2 : 1);
        if (nch <= 1 || nq < nch) {
            // Small batches are launch-bound (batch 1: ~3 µs in each kernel, ~7 µs of host API time
            // between them): the second call in a row with the same arguments captures the stages
            // as a CUDA graph and every later one replays it (PQTG_NO_GRAPH=1 disables).
            static const bool no_graph = std::getenv("PQTG_NO_GRAPH") != nullptr;
            const uint64_t key[12] = {(uint64_t)(uintptr_t)d_queries, nq, k, (uint64_t)(uintptr_t)d_ids,
                                      (uint64_t)(uintptr_t)d_dists, (uint64_t)(uintptr_t)d_counts,
                                      (uint64_t)(uintptr_t)d_stats, ws.gen, (uint64_t)kernel_variant(),
                                      (uint64_t)(uintptr_t)index->dev->db, pp.rerank_exact,
                                      0x9d5ea7c4f1e2b3a1ull};  // device-path tag
            const bool repeat = std::memcmp(ws.dev_last_key, key, sizeof(key)) == 0;
            std::memcpy(ws.dev_last_key, key, sizeof(key));
            if (no_graph || nq == 0 || nq >= 256 || !repeat) {
                run_chunk(*index->dev, ws, 0, d_queries, nq, k, d_ids, d_dists, d_counts, d_stats, s, true);
            } else {
                const cudaGraphExec_t exec = cached_graph(ws, key, ws.own_stream, [&] {
                    run_chunk(*index->dev, ws, 0, d_queries, nq, k, d_ids, d_dists, d_counts, d_stats, ws.own_stream,
                              true);
                });
                PQTG_CUDA_CHECK(cudaGraphLaunch(exec, s));
            }
            PQTG_CUDA_CHECK(cudaEventRecord(ws.done, s));
            return PQTG_OK;
        }
        // chunks alternate between the caller's stream and the workspace's aux stream (forked
        // from and joined back into the caller's), so one chunk's re-rank overlaps the next
        // chunk's traversal / bin selection
        PQTG_CUDA_CHECK(cudaEventRecord(ws.join, s));
        PQTG_CUDA_CHECK(cudaStreamWaitEvent(ws.aux_stream, ws.join, 0));
        const uint64_t per = (nq + nch - 1) / nch;
        const uint64_t kk = std::max<uint32_t>(k, 1);
        for (uint64_t c = 0; c * per < nq; ++c) {
            const uint64_t c0 = c * per, cn = std::min(per, nq - c0);
            run_chunk(*index->dev, ws, c0, d_queries + c0 * index->dev->prm.D, cn, k, d_ids ? d_ids + c0 * kk : nullptr,
                      d_dists ? d_dists + c0 * kk : nullptr, d_counts + c0, d_stats ? d_stats + c0 : nullptr,
                      (c & 1) ? ws.aux_stream : s, c == 0);
        }
        PQTG_CUDA_CHECK(cudaEventRecord(ws.join, ws.aux_stream));
        PQTG_CUDA_CHECK(cudaStreamWaitEvent(s, ws.join, 0));
        PQTG_CUDA_CHECK(cudaEventRecord(ws.done, s));
        return PQTG_OK;
    });
}

int pqtg_search(pqtg_index* index, pqtg_workspace* wsh, const float* queries, uint64_t nq, uint32_t dim,
                uint32_t k, uint32_t* ids, float* dists, uint32_t* counts, pqtg_query_stats* stats) {
    return guarded([&] {
        if (!index || !wsh) throw Error{PQTG_ERR_ARG, "null argument"};
        const DevIndex& d = *index->dev;
        if (nq > 0 && dim != d.prm.D)  // search.cpp:264-266
            throw Error{PQTG_ERR_BAD_DIM, "knn_query_batch: query dimension mismatch"};
        if (nq && (!queries || !counts || (k && (!ids || !dists)))) throw Error{PQTG_ERR_ARG, "null argument"};
        Workspace& ws = *wsh->ws;
        if (ws.index != &d) throw Error{PQTG_ERR_ARG, "workspace belongs to another index"};
        std::lock_guard<std::mutex> lock(ws.mu);
        PQTG_CUDA_CHECK(cudaSetDevice(d.device));
        refuse_shard_exact(d.prm);
        PQTG_CUDA_CHECK(cudaStreamWaitEvent(ws.own_stream, ws.done, 0));  // a previous pqtg_search_device call
        ensure_staging(ws, std::max<uint32_t>(k, 1));
        if (ws.qtime_on && ws.qtime_cap < nq) {  // the per-query clocks of the whole call (pinned)
            PQTG_CUDA_CHECK(cudaStreamSynchronize(ws.own_stream));
            if (ws.h_qtime) cudaFreeHost(ws.h_qtime);
            ws.h_qtime = nullptr;
            PQTG_CUDA_CHECK(cudaMallocHost(&ws.h_qtime, nq * 6 * sizeof(unsigned long long)));
            ws.qtime_cap = nq;
            ++ws.gen;
        }
        ws.qtime_host = true;
        ensure_exact(ws, k);
        ensure_keys(ws, k);
        const uint64_t D = d.prm.D;
        cudaStream_t st[2] = {ws.own_stream, ws.aux_stream};
        ws.last_stream = ws.own_stream;
        auto enqueue = [&] {
            if (d.prm.exact_order) PQTG_CUDA_CHECK(cudaMemsetAsync(ws.err, 0, sizeof(uint32_t), st[0]));
            // Sub-batches of <= max_batch queries; each is cut into chunks that alternate between
            // two streams, so chunk c's kernels overlap chunk c+1's H2D and chunk c-1's D2H.
            for (uint64_t q0 = 0; q0 < nq || (nq == 0 && q0 == 0); q0 += ws.max_batch) {
                const uint64_t b = std::min(ws.max_batch, nq - q0);
                if (b == 0) {
                    run_chunk(d, ws, 0, ws.d_queries, 0, k, ws.d_ids, ws.d_dists, ws.d_counts, ws.d_stats, st[0], true);
                    ws.last_nq = 0;
                    break;
                }
                // reusing the slices: the other stream's chunks of the previous sub-batch must be done
                PQTG_CUDA_CHECK(cudaEventRecord(ws.join, st[1]));
                PQTG_CUDA_CHECK(cudaStreamWaitEvent(st[0], ws.join, 0));
                const std::vector<uint64_t> bounds = host_chunks(ws, b);
                for (uint64_t c = 0; c + 1 < bounds.size(); ++c) {
                    const uint64_t c0 = bounds[c], cn = bounds[c + 1] - c0;
                    cudaStream_t s = st[c & 1];
                    if (c == 1) PQTG_CUDA_CHECK(cudaStreamWaitEvent(s, ws.join, 0));  // after the epoch bump
                    if (c == 0) PQTG_CUDA_CHECK(cudaEventRecord(ws.join, s));
                    PQTG_CUDA_CHECK(cudaMemcpyAsync(ws.d_queries + c0 * D, queries + (q0 + c0) * D, cn * D * sizeof(float),
                                                    cudaMemcpyHostToDevice, s));
                    run_chunk(d, ws, c0, ws.d_queries + c0 * D, cn, k, ws.d_ids + c0 * std::max<uint32_t>(k, 1),
                              ws.d_dists + c0 * std::max<uint32_t>(k, 1), ws.d_counts + c0, ws.d_stats + c0, s, c == 0,
                              ws.qtime_on ? ws.h_qtime + (q0 + c0) * 6 : nullptr);
                    if (k) {
                        PQTG_CUDA_CHECK(cudaMemcpyAsync(ids + (q0 + c0) * k, ws.d_ids + c0 * k, cn * k * sizeof(uint32_t),
                                                        cudaMemcpyDeviceToHost, s));
                        PQTG_CUDA_CHECK(cudaMemcpyAsync(dists + (q0 + c0) * k, ws.d_dists + c0 * k, cn * k * sizeof(float),
                                                        cudaMemcpyDeviceToHost, s));
                    }
                    PQTG_CUDA_CHECK(cudaMemcpyAsync(counts + q0 + c0, ws.d_counts + c0, cn * sizeof(uint32_t),
                                                    cudaMemcpyDeviceToHost, s));
                    if (stats)
                        PQTG_CUDA_CHECK(cudaMemcpyAsync(stats + q0 + c0, ws.d_stats + c0, cn * sizeof(pqtg_query_stats),
                                                        cudaMemcpyDeviceToHost, s));
                }
                ws.last_nq = b;
            }
        };
        // The whole search is one CUDA graph, replayed when the same arguments come back: one
        // launch instead of ~10 API calls per chunk (PQTG_NO_GRAPH=1 disables).
        static const bool no_graph = std::getenv("PQTG_NO_GRAPH") != nullptr;
        auto pinned = [](const void* ptr) {  // graph memcpy nodes want page-locked host memory
            if (!ptr) return true;
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return a.type == cudaMemoryTypeHost;
        };
        // exact bin order: a query whose heap outgrew shared memory sets the workspace's error
        // word (kernels.cu binsel_kernel<EXACT>), whichever sub-batch it was in
        auto check_exact = [&] {
            if (d.prm.exact_order) check_ws_error(ws);
        };
        if (no_graph || nq == 0 || !pinned(queries) || !pinned(ids) || !pinned(dists) || !pinned(counts) ||
            !pinned(stats)) {
            enqueue();
            PQTG_CUDA_CHECK(cudaStreamSynchronize(st[0]));
            PQTG_CUDA_CHECK(cudaStreamSynchronize(st[1]));
            PQTG_CUDA_CHECK(cudaEventRecord(ws.done, st[0]));
            check_exact();
            return PQTG_OK;
        }
        // Small batches (<= zc_max) write their results straight into the caller's page-locked buffers
        // (mapped into the device's address space): the replayed graph is the query copy and the
        // three kernels, with no result copies behind them (PQTG_ZERO_COPY=0 disables).
        static const bool zero_copy = [] {
            const char* e = std::getenv("PQTG_ZERO_COPY");
            return !(e && std::strcmp(e, "0") == 0);
        }();
        auto mapped = [&](void* ptr) -> void* {  // the device view of a page-locked buffer of this device
            if (!ptr) return nullptr;
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            return a.type == cudaMemoryTypeHost && a.device == d.device ? a.devicePointer : nullptr;
        };
        void* zc_out[4] = {mapped(ids), mapped(dists), mapped(counts), mapped(stats)};
        // (Zero-copy for larger batches -- queries read by the traversal and results written by the
        // re-rank straight over the link -- measured far slower: DEEP100M e2e 6.35 -> 4.25 M q/s,
        // the re-rank's scattered 4-byte result stores do not suit the link.)
        // up to 128 queries (SIFT1M e2e, zero-copy vs copies: batch 100 78.4 vs 88.2 µs, batch 200
        // 104.6 vs 94.0, batch 1000 232 vs 215); PQTG_ZC_MAX overrides for experiments
        static const uint64_t zc_max = [] {
            const char* e = std::getenv("PQTG_ZC_MAX");
            return e ? (uint64_t)std::strtoull(e, nullptr, 10) : (uint64_t)128;
        }();
        const bool zc = zero_copy && nq <= zc_max && nq <= ws.max_batch && (zc_out[0] || !ids) && (zc_out[1] || !dists) &&
                        zc_out[2] && (zc_out[3] || !stats);
        auto enqueue_zc = [&] {
            if (d.prm.exact_order) PQTG_CUDA_CHECK(cudaMemsetAsync(ws.err, 0, sizeof(uint32_t), st[0]));
            PQTG_CUDA_CHECK(cudaMemcpyAsync(ws.d_queries, queries, nq * D * sizeof(float), cudaMemcpyHostToDevice, st[0]));
            run_chunk(d, ws, 0, ws.d_queries, nq, k, static_cast<uint32_t*>(zc_out[0]), static_cast<float*>(zc_out[1]),
                      static_cast<uint32_t*>(zc_out[2]), static_cast<pqtg_query_stats*>(zc_out[3]), st[0], true,
                      ws.qtime_on ? ws.h_qtime : nullptr);
        };
        const uint64_t key[12] = {(uint64_t)(uintptr_t)queries, nq, k, (uint64_t)(uintptr_t)ids,
                                  (uint64_t)(uintptr_t)dists, (uint64_t)(uintptr_t)counts,
                                  (uint64_t)(uintptr_t)stats, ws.gen, (uint64_t)kernel_variant(),
                                  (uint64_t)(uintptr_t)d.db, d.prm.rerank_exact,
                                  (uint64_t)std::hash<std::string>{}(std::getenv("PQTG_CHUNK_PLAN") ? std::getenv("PQTG_CHUNK_PLAN") : "") ^
                                      (zc ? 0x5a5a5a5a5a5a5a5aull : 0ull)};
        if (zc) {
            const cudaGraphExec_t exec = cached_graph(ws, key, st[0], enqueue_zc);
            ws.last_nq = nq;
            PQTG_CUDA_CHECK(cudaGraphLaunch(exec, st[0]));
            PQTG_CUDA_CHECK(cudaStreamSynchronize(st[0]));
            PQTG_CUDA_CHECK(cudaEventRecord(ws.done, st[0]));
            check_exact();
            return PQTG_OK;
        }
        const bool cached = std::any_of(ws.graphs.begin(), ws.graphs.end(),
                                        [&](const auto& g) { return std::memcmp(g.key, key, sizeof(key)) == 0; });
        const cudaGraphExec_t exec = cached_graph(ws, key, st[0], enqueue);
        if (cached) ws.last_nq = nq - (nq - 1) / ws.max_batch * ws.max_batch;  // the last sub-batch
        PQTG_CUDA_CHECK(cudaGraphLaunch(exec, st[0]));
        PQTG_CUDA_CHECK(cudaStreamSynchronize(st[0]));
        PQTG_CUDA_CHECK(cudaEventRecord(ws.done, st[0]));
        check_exact();
        return PQTG_OK;
    });
}

int64_t pqtg_bin_stream_host(const pqtg_index_view* v, const float* lists, uint64_t max_tuples, uint32_t* out) {
    int64_t produced = 0;
    const int rc = guarded([&] {
        if (!v || !lists || (max_tuples && !out)) throw Error{PQTG_ERR_ARG, "null argument"};
        validate_config(v->config);
        const uint32_t P = v->config.p_tree;
        if (!(P == 1 || P == 2 || P == 4)) unsupported("p_tree must be 1, 2 or 4");
        if (P > 1 && v->table_count != kSlopeTables) unsupported("slope tables missing");
        const uint64_t W64 = (uint64_t)v->config.w * v->config.k2;
        if (W64 > 65535) unsupported("w*k2 must be < 65536");
        const uint32_t W = (uint32_t)W64;
        HostStreams hs = build_streams(v->table_entries, v->table_len, W, P);
        // pick_slope_table (binorder.cpp:52-65), host libm
        auto pick = [&](const float* a, const float* b) -> uint32_t {
            if (W < 2) return kSlopeOne;
            const double ga = (double)a[1] - a[0], gb = (double)b[1] - b[0];
            if (!(ga > 0.0) || !(gb > 0.0)) return kSlopeOne;
            long k = std::lround(std::log(gb / ga) / std::log(1.08));
            k = std::clamp(k, -5L, 4L);
            return (uint32_t)(k + 5);
        };
        const uint32_t ta = P >= 2 ? pick(lists, lists + W) : kSlopeOne;
        const uint32_t tb = P == 4 ? pick(lists + 2 * W, lists + 3 * W) : kSlopeOne;
        const uint64_t cnt = std::min<uint64_t>(max_tuples, hs.total);
        for (uint64_t s = 0; s < cnt; ++s) hs.tuple_at(s, ta, tb, out + s * P);
        produced = (int64_t)cnt;
        return PQTG_OK;
    });
    return rc != PQTG_OK ? rc : produced;
}

int pqtg_merge_topk_host(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* ids, const float* dists,
                         const uint32_t* counts, uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        if (shards == 0 || (nq && (!ids || !dists || !counts || !out_ids || !out_dists || !out_counts)))
            throw Error{PQTG_ERR_ARG, "bad merge arguments"};
        std::vector<uint32_t> cur(shards);
        for (uint64_t q = 0; q < nq; ++q) {
            std::fill(cur.begin(), cur.end(), 0u);
            uint32_t out = 0;
            while (out < k) {
                int best = -1;
                for (uint32_t g = 0; g < shards; ++g) {
                    if (cur[g] >= counts[(uint64_t)g * nq + q]) continue;
                    const uint64_t o = ((uint64_t)g * nq + q) * k + cur[g];
                    if (best < 0) {
                        best = (int)g;
                        continue;
                    }
                    const uint64_t ob = ((uint64_t)best * nq + q) * k + cur[best];
                    // candidate_less (search.cpp:39-41)
                    const bool less = dists[o] != dists[ob] ? dists[o] < dists[ob] : ids[o] < ids[ob];
                    if (less) best = (int)g;
                }
                if (best < 0) break;
                const uint64_t o = ((uint64_t)best * nq + q) * k + cur[best];
                out_ids[q * k + out] = ids[o];
                out_dists[q * k + out] = dists[o];
                ++cur[best];
                ++out;
            }
            for (uint32_t i = out; i < k; ++i) {
                out_ids[q * k + i] = 0xFFFFFFFFu;
                out_dists[q * k + i] = __builtin_inff();
            }
            out_counts[q] = out;
        }
        return PQTG_OK;
    });
}

int pqtg_merge_topk_device(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* d_ids, const float* d_dists,
                           const uint32_t* d_counts, uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_counts,
                           void* stream) {
    return guarded([&] {
        if (shards == 0 || shards > 16) throw Error{PQTG_ERR_ARG, "shards must be in [1, 16]"};
        launch_merge(shards, nq, k, d_ids, d_dists, d_counts, d_out_ids, d_out_dists, d_out_counts,
                     static_cast<cudaStream_t>(stream));
        return PQTG_OK;
    });
}

int pqtg_brute_force_knn_device(const float* d_db, uint64_t n, uint32_t dim, const float* d_queries, uint64_t nq,
                                uint32_t k, uint32_t* d_ids, float* d_dists, uint32_t* d_counts, void* stream) {
    return guarded([&] {
        if (nq && (!d_queries || !d_counts || (k && (!d_ids || !d_dists)) || (n && !d_db)))
            throw Error{PQTG_ERR_ARG, "null argument"};
        if (dim == 0) throw Error{PQTG_ERR_BAD_DIM, "brute_force_knn: dim must be positive"};
        if (n >= (1ull << 32)) throw Error{PQTG_ERR_UNSUPPORTED, "brute_force_knn: n must be < 2^32"};
        if (!brute_force_ok(dim, k)) throw Error{PQTG_ERR_UNSUPPORTED, "brute_force_knn: k or dim too large"};
        launch_brute_force(d_db, n, dim, d_queries, nq, k, d_ids, d_dists, d_counts, static_cast<cudaStream_t>(stream));
        return PQTG_OK;
    });
}

int pqtg_brute_force_knn(const float* db, uint64_t n, uint32_t dim, const float* queries, uint64_t nq, uint32_t k,
                         int device, uint32_t* ids, float* dists, uint32_t* counts, pqtg_query_stats* stats) {
    return guarded([&] {
        if (nq && (!queries || !counts || (k && (!ids || !dists)) || (n && !db))) throw Error{PQTG_ERR_ARG, "null argument"};
        if (dim == 0) throw Error{PQTG_ERR_BAD_DIM, "brute_force_knn: dim must be positive"};
        if (n >= (1ull << 32)) throw Error{PQTG_ERR_UNSUPPORTED, "brute_force_knn: n must be < 2^32"};
        PQTG_CUDA_CHECK(cudaSetDevice(device));
        if (!brute_force_ok(dim, k)) throw Error{PQTG_ERR_UNSUPPORTED, "brute_force_knn: k or dim too large"};
        if (nq == 0) return PQTG_OK;
        std::vector<void*> held;
        auto alloc = [&](size_t bytes) {
            void* p = nullptr;
            PQTG_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
            held.push_back(p);
            return p;
        };
        try {
            float* d_db = static_cast<float*>(alloc(n * dim * 4));
            float* d_q = static_cast<float*>(alloc(nq * dim * 4));
            uint32_t* d_ids = static_cast<uint32_t*>(alloc(nq * std::max<uint32_t>(k, 1) * 4));
            float* d_d = static_cast<float*>(alloc(nq * std::max<uint32_t>(k, 1) * 4));
            uint32_t* d_c = static_cast<uint32_t*>(alloc(nq * 4));
            if (n) PQTG_CUDA_CHECK(cudaMemcpy(d_db, db, n * dim * 4, cudaMemcpyHostToDevice));
            PQTG_CUDA_CHECK(cudaMemcpy(d_q, queries, nq * dim * 4, cudaMemcpyHostToDevice));
            launch_brute_force(d_db, n, dim, d_q, nq, k, d_ids, d_d, d_c, nullptr);
            if (k) {
                PQTG_CUDA_CHECK(cudaMemcpy(ids, d_ids, nq * k * 4, cudaMemcpyDeviceToHost));
                PQTG_CUDA_CHECK(cudaMemcpy(dists, d_d, nq * k * 4, cudaMemcpyDeviceToHost));
            }
            PQTG_CUDA_CHECK(cudaMemcpy(counts, d_c, nq * 4, cudaMemcpyDeviceToHost));
        } catch (...) {
            for (void* p : held) cudaFree(p);
            throw;
        }
        for (void* p : held) cudaFree(p);
        if (stats)
            for (uint64_t q = 0; q < nq; ++q) {
                stats[q].bins_visited = 0;
                stats[q].candidates = k && n ? n : 0;  // search.cpp:279-296: empty result when min(k, n) == 0
                stats[q].exact_evals = k && n ? n : 0;
            }
        return PQTG_OK;
    });
}

int pqtg_shard_range(uint64_t n, uint32_t shards, uint32_t rank, uint64_t* lo, uint64_t* hi) {
    return guarded([&] {
        if (shards == 0 || rank >= shards || !lo || !hi) throw Error{PQTG_ERR_ARG, "bad shard arguments"};
        const uint64_t per = n / shards, extra = n % shards;
        *lo = rank * per + std::min<uint64_t>(rank, extra);
        *hi = *lo + per + (rank < extra ? 1 : 0);
        return PQTG_OK;
    });
}

}  // extern "C"
