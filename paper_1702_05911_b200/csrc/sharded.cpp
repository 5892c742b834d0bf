// sharded.cpp — query-partitioned sharded search over G position shards (include/pqtg.h
// "sharded search"). The reference has no multi-node path: this is the
// billion-scale deployment of pqt::knn_query_batch (src/search.cpp:262-274) whose result is
// bit-identical to the unsharded search.
//
// One protocol, two transports:
//   NCCL   one process per GPU (pqtg_sharded_create_nccl): broadcasts / all-gather / send-recv
//          on the rank's stream, libnccl.so.2 loaded with dlopen (the one a torch process already
//          holds, else the system's);
//   local  every shard in this process (pqtg_sharded_create_local): the same steps with
//          device-to-device copies between the ranks' buffers, ordered by events.
// Per batch of nq queries, block g = pqtg_shard_range(nq, G, g):
//   S1  rank g: traversal + bin selection of block g (its workspace rows [lo_g, hi_g));
//   S2  rank g: its block's range lists packed densely (scan of nranges, gather);
//   S3  the packed sizes are all-gathered (the only host round trip of the call);
//   S4  all-gather-v of the blocks' nranges, ncand, stats and packed ranges;
//   S5  every rank recomputes the batch's fine LUTs (L·k1·fd multiply-adds per query: cheaper
//       than moving 4·L·k1 bytes per query) and unpacks the whole batch's ranges;
//   S6  every rank re-ranks the batch's candidates inside its position range (local top-k);
//   S7  all-to-all: rank j receives every rank's lists of block j;
//   S8  rank j merges them by (dist, id) (candidate_less, search.cpp:39-41);
//   S9  all-gather-v of the merged blocks: every rank holds the whole batch's results.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the library is loaded at run time

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "pqtg_internal.h"

namespace pqtg {
namespace {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string load_error;

    static Nccl& get() {
        static Nccl api = [] {
            Nccl a;
            const char* env = std::getenv("PQTG_NCCL_LIB");
            void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) {
                a.load_error = std::string("cannot load NCCL: ") + dlerror();
                return a;
            }
            auto sym = [&](auto& fn, const char* name) {
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
                if (!fn && a.load_error.empty()) a.load_error = std::string("NCCL symbol missing: ") + name;
            };
            sym(a.get_unique_id, "ncclGetUniqueId");
            sym(a.comm_init_rank, "ncclCommInitRank");
            sym(a.comm_destroy, "ncclCommDestroy");
            sym(a.group_start, "ncclGroupStart");
            sym(a.group_end, "ncclGroupEnd");
            sym(a.broadcast, "ncclBroadcast");
            sym(a.all_gather, "ncclAllGather");
            sym(a.send, "ncclSend");
            sym(a.recv, "ncclRecv");
            sym(a.error_string, "ncclGetErrorString");
            return a;
        }();
        if (!api.load_error.empty()) throw Error{PQTG_ERR_NCCL, api.load_error};
        return api;
    }
};

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const Nccl& a = Nccl::get();
        throw Error{PQTG_ERR_NCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "error")};
    }
}

struct Block {
    uint64_t lo = 0, n = 0;
};

std::vector<Block> blocks_of(uint64_t nq, uint32_t G) {
    std::vector<Block> b(G);
    const uint64_t per = nq / G, extra = nq % G;
    for (uint32_t g = 0; g < G; ++g) {
        b[g].lo = g * per + std::min<uint64_t>(g, extra);
        b[g].n = per + (g < extra ? 1 : 0);
    }
    return b;
}

// one rank's device state
struct Rank {
    uint32_t g = 0;                 // global rank
    DevIndex* ix = nullptr;         // borrowed shard
    std::unique_ptr<pqtg_workspace> wsh;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;     // this rank's last queued step
    cudaEvent_t ev[5] = {};         // stage timing (local rank 0)
    cudaEvent_t sized = nullptr;    // the packed sizes are on the host (S3)
    std::vector<void*> allocations;
    uint64_t* blk_off = nullptr;    // [max_batch + 1] scan of this block's nranges
    uint64_t* all_off = nullptr;    // [max_batch + 1] scan of the batch's nranges
    uint64_t* d_totals = nullptr;   // [G] packed sizes (NCCL all-gather target)
    uint64_t* h_totals = nullptr;   // pinned [G]
    uint2* packed = nullptr;        // this block's ranges, dense [block_max * budget]
    uint2* all_packed = nullptr;    // the batch's ranges, dense
    uint64_t all_cap = 0;
    pqtg_query_stats* stats = nullptr;  // [max_batch] when the caller passes none
    // k-dependent: local lists of the whole batch and received lists of this block
    uint64_t lk = 0;
    uint32_t* l_ids = nullptr;
    float* l_dists = nullptr;
    uint32_t* l_counts = nullptr;
    uint32_t* r_ids = nullptr;
    float* r_dists = nullptr;
    uint32_t* r_counts = nullptr;
    float* l_exact = nullptr;       // the exact stage: exact distances of the local line prefix
    float* r_exact = nullptr;
    // host-call staging (k-dependent outputs share lk)
    float* q = nullptr;
    uint32_t* o_ids = nullptr;
    float* o_dists = nullptr;
    uint32_t* o_counts = nullptr;
    pqtg_query_stats* o_stats = nullptr;

    Workspace& ws() { return *wsh->ws; }
    ~Rank() {
        if (ix) cudaSetDevice(ix->device);
        if (h_totals) cudaFreeHost(h_totals);
        for (void* p : allocations) cudaFree(p);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (done) cudaEventDestroy(done);
        if (sized) cudaEventDestroy(sized);
        if (stream) cudaStreamDestroy(stream);
    }
};

}  // namespace
}  // namespace pqtg

struct pqtg_sharded {
    uint32_t world = 0;
    bool nccl = false;
    // measurement harness (pqtg_sharded_create_sim): one real rank; the peers' pieces come from a
    // one-time computation of the whole batch on this GPU, their transfers are device copies
    bool sim = false;
    struct SimCache {  // one per query batch seen (keyed by its device pointer and size)
        const float* q = nullptr;
        uint64_t nq = 0;
        std::vector<void*> allocations;
        uint32_t* nranges = nullptr;
        uint32_t* ncand = nullptr;
        pqtg_query_stats* stats = nullptr;
        uint2* packed = nullptr;
        uint64_t* off = nullptr;
        std::vector<uint64_t> total, toff;
        ~SimCache() {
            for (void* p : allocations) cudaFree(p);
        }
    };
    std::vector<std::unique_ptr<SimCache>> simcs;
    SimCache* simc = nullptr;  // the current batch's
    ncclComm_t comm = nullptr;
    uint64_t max_batch = 0, block_max = 0;
    uint64_t n = 0;
    uint32_t D = 0, L = 0, k1 = 0, budget = 0;
    std::vector<std::unique_ptr<pqtg::Rank>> ranks;  // local ranks
    std::mutex mu;
    ~pqtg_sharded() {
        if (comm) pqtg::Nccl::get().comm_destroy(comm);
    }
};

namespace pqtg {
namespace {

template <class F>
int guarded_sh(F&& fn) {
    try {
        return fn();
    } catch (const Error& e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return PQTG_ERR_OOM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PQTG_ERR_ARG;
    }
}

void setup_rank(pqtg_sharded& sh, Rank& r) {
    const DevParams& p = r.ix->prm;
    PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device));
    pqtg_workspace* w = nullptr;
    pqtg_index tmp;  // pqtg_workspace_create reads only ->dev
    tmp.dev.reset(r.ix);
    const int rc = pqtg_workspace_create(&tmp, sh.max_batch, &w);
    tmp.dev.release();
    if (rc != PQTG_OK) throw Error{rc, std::string("sharded workspace: ") + last_error()};
    r.wsh.reset(w);
    PQTG_CUDA_CHECK(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
    PQTG_CUDA_CHECK(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    for (auto& e : r.ev) PQTG_CUDA_CHECK(cudaEventCreate(&e));
    PQTG_CUDA_CHECK(cudaEventCreateWithFlags(&r.sized, cudaEventDisableTiming));
    r.blk_off = dev_alloc<uint64_t>(r.allocations, sh.max_batch + 1);
    r.all_off = dev_alloc<uint64_t>(r.allocations, sh.max_batch + 1);
    r.d_totals = dev_alloc<uint64_t>(r.allocations, sh.world);
    PQTG_CUDA_CHECK(cudaMallocHost(&r.h_totals, sh.world * sizeof(uint64_t)));
    r.packed = dev_alloc<uint2>(r.allocations, std::max<uint64_t>(sh.block_max * std::max<uint32_t>(p.budget, 1), 1));
    r.stats = dev_alloc<pqtg_query_stats>(r.allocations, sh.max_batch);
    r.q = dev_alloc<float>(r.allocations, sh.max_batch * p.D);
}

void ensure_k(pqtg_sharded& sh, Rank& r, uint32_t k) {
    if (r.lk >= k) return;
    PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device));
    PQTG_CUDA_CHECK(cudaStreamSynchronize(r.stream));
    const uint64_t B = sh.max_batch;
    r.l_ids = dev_alloc<uint32_t>(r.allocations, B * k);
    r.l_dists = dev_alloc<float>(r.allocations, B * k);
    r.l_counts = dev_alloc<uint32_t>(r.allocations, B);
    r.r_ids = dev_alloc<uint32_t>(r.allocations, (uint64_t)sh.world * sh.block_max * k);
    r.r_dists = dev_alloc<float>(r.allocations, (uint64_t)sh.world * sh.block_max * k);
    r.r_counts = dev_alloc<uint32_t>(r.allocations, (uint64_t)sh.world * sh.block_max);
    r.l_exact = dev_alloc<float>(r.allocations, B * k);
    r.r_exact = dev_alloc<float>(r.allocations, (uint64_t)sh.world * sh.block_max * k);
    r.o_ids = dev_alloc<uint32_t>(r.allocations, B * k);
    r.o_dists = dev_alloc<float>(r.allocations, B * k);
    r.o_counts = dev_alloc<uint32_t>(r.allocations, B);
    r.o_stats = dev_alloc<pqtg_query_stats>(r.allocations, B);
    r.lk = k;
}

void ensure_all_packed(Rank& r, uint64_t entries) {
    if (entries <= r.all_cap) return;
    PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device));
    PQTG_CUDA_CHECK(cudaStreamSynchronize(r.stream));
    const uint64_t cap = std::max<uint64_t>(entries + entries / 4, 1024);
    r.all_packed = dev_alloc<uint2>(r.allocations, cap);
    r.all_cap = cap;
}

// all-gather-v over the ranks: rank g contributes bytes [off_g, off_g + len_g) of `buf` (the
// same offsets on every rank: in place) -- NCCL: one broadcast per root in a group; local:
// copies into every other rank's buffer. src(g) may differ from the in-place region (packed).
struct Piece {
    const void* src;  // root's send buffer (on the root rank); nullptr = in place
    void* dst;        // this rank's receive buffer for root g's piece
    size_t bytes;
};

// the peers' inputs of a simulated step: traversal + bin selection of the WHOLE batch on this GPU,
// each block's ranges packed as its owner would send them (done once per batch, outside timing)
void sim_fill(pqtg_sharded& sh, Rank& r, const float* q, uint64_t nq, const std::vector<uint64_t>& blo,
              const std::vector<uint64_t>& bn) {
    for (auto& c : sh.simcs)
        if (c->q == q && c->nq == nq) {
            sh.simc = c.get();
            return;
        }
    if (sh.simcs.size() >= 8) sh.simcs.erase(sh.simcs.begin());
    sh.simcs.push_back(std::make_unique<pqtg_sharded::SimCache>());
    auto& c = *sh.simcs.back();
    const DevParams& p = r.ix->prm;
    const uint32_t budget = std::max<uint32_t>(p.budget, 1);
    PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device));
    c.nranges = dev_alloc<uint32_t>(c.allocations, nq);
    c.ncand = dev_alloc<uint32_t>(c.allocations, nq);
    c.stats = dev_alloc<pqtg_query_stats>(c.allocations, nq);
    c.off = dev_alloc<uint64_t>(c.allocations, nq + 1);
    const WsSlice sl = r.ws().slice(0);
    launch_traverse(p, q, nq, sl, r.stream);
    launch_binsel(p, nq, sl, c.stats, r.stream);
    PQTG_CUDA_CHECK(cudaMemcpyAsync(c.nranges, r.ws().nranges, nq * 4, cudaMemcpyDeviceToDevice, r.stream));
    PQTG_CUDA_CHECK(cudaMemcpyAsync(c.ncand, r.ws().ncand, nq * 4, cudaMemcpyDeviceToDevice, r.stream));
    launch_scan_counts(c.nranges, nq, c.off, r.stream);
    std::vector<uint64_t> off(nq + 1);
    PQTG_CUDA_CHECK(cudaMemcpyAsync(off.data(), c.off, (nq + 1) * 8, cudaMemcpyDeviceToHost, r.stream));
    PQTG_CUDA_CHECK(cudaStreamSynchronize(r.stream));
    c.packed = dev_alloc<uint2>(c.allocations, std::max<uint64_t>(off[nq], 1));
    launch_pack_ranges(r.ws().ranges, budget, c.nranges, c.off, nq, c.packed, r.stream);
    PQTG_CUDA_CHECK(cudaStreamSynchronize(r.stream));
    c.total.assign(sh.world, 0);
    c.toff.assign(sh.world + 1, 0);
    for (uint32_t g = 0; g < sh.world; ++g) {
        c.total[g] = off[blo[g] + bn[g]] - off[blo[g]];
        c.toff[g] = off[blo[g]];
    }
    c.q = q;
    c.nq = nq;
    sh.simc = &c;
}

}  // namespace

// ---------------------------------------------------------------- the search
static void sharded_search(pqtg_sharded& sh, const float* const* d_queries, uint64_t nq, uint32_t k, bool bcast,
                           uint32_t* const* d_ids, float* const* d_dists, uint32_t* const* d_counts,
                           pqtg_query_stats* const* d_stats, void* const* streams) {
    const uint32_t G = sh.world;
    const uint32_t R = (uint32_t)sh.ranks.size();
    if (nq > sh.max_batch) throw Error{PQTG_ERR_ARG, "nq exceeds the sharded handle's max_batch"};
    for (uint32_t i = 0; i < R; ++i)
        if (nq && (!d_queries || !d_counts || !d_counts[i] || (k && (!d_ids || !d_dists || !d_ids[i] || !d_dists[i])) ||
                   (!d_queries[i] && !(bcast && sh.ranks[i]->g != 0))))
            throw Error{PQTG_ERR_ARG, "null argument"};
    if (nq == 0) return;
    const std::vector<Block> blk = blocks_of(nq, G);
    const uint32_t D = sh.D, budget = sh.budget;
    const uint64_t kk = std::max<uint32_t>(k, 1);
    Nccl* nc = sh.nccl ? &Nccl::get() : nullptr;
    auto caller = [&](uint32_t i) -> cudaStream_t {
        return streams ? static_cast<cudaStream_t>(streams[i]) : static_cast<cudaStream_t>(nullptr);
    };
    auto stats_of = [&](uint32_t i) -> pqtg_query_stats* {
        return d_stats && d_stats[i] ? d_stats[i] : sh.ranks[i]->stats;
    };
    auto on = [&](Rank& r) { PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device)); };
    auto rank_index = [&](const Rank& self) {
        uint32_t i = 0;
        while (sh.ranks[i].get() != &self) ++i;
        return i;
    };
    // the exact stage (search.cpp:229-249) when the shards hold their raw rows: each rank's
    // line-ranked prefix of R = max(k, rerank_exact) with exact distances travels as
    // (id, line, exact) triples and the merge cuts the global prefix min(R, C) before ranking by
    // exact distance; lists then have R entries instead of k
    const bool exact = sh.ranks[0]->ix->prm.db && sh.ranks[0]->ix->prm.rerank_exact > 0 && k > 0;
    const uint32_t Rx = exact ? std::min(std::max(k, sh.ranks[0]->ix->prm.rerank_exact), std::max(budget, 1u)) : k;
    const uint64_t lk = std::max<uint32_t>(Rx, 1);  // list stride of S6-S8
    for (uint32_t i = 0; i < R; ++i) {
        Rank& r = *sh.ranks[i];
        on(r);
        if (((bool)r.ix->prm.db && r.ix->prm.rerank_exact > 0) != exact)
            throw Error{PQTG_ERR_ARG, "sharded exact re-rank: every shard must hold its raw rows, or none"};
        if (exact && sh.sim) throw Error{PQTG_ERR_UNSUPPORTED, "the simulated transport has no exact stage"};
        prepare_workspace(r.ws(), k);
        ensure_k(sh, r, (uint32_t)std::max<uint64_t>(kk, lk));
        // start after the caller's queued work
        PQTG_CUDA_CHECK(cudaEventRecord(r.done, caller(i)));
        PQTG_CUDA_CHECK(cudaStreamWaitEvent(r.stream, r.done, 0));
        if (i == 0) PQTG_CUDA_CHECK(cudaEventRecord(r.ev[0], r.stream));
    }
    // local transport: dst's stream waits for every other rank's last step
    auto wait_all = [&](Rank& dst) {
        for (auto& o : sh.ranks)
            if (o.get() != &dst) PQTG_CUDA_CHECK(cudaStreamWaitEvent(dst.stream, o->done, 0));
    };
    auto mark = [&](Rank& r) { PQTG_CUDA_CHECK(cudaEventRecord(r.done, r.stream)); };
    // local transport: one copy kernel when every rank lives on one device, else peer memcpys
    bool one_device = true;
    for (auto& rp : sh.ranks) one_device = one_device && rp->ix->device == sh.ranks[0]->ix->device;
    auto copies = [&](Rank& dst, const std::vector<CopySegment>& cs) {
        if (one_device) {
            launch_copy_segments(cs, dst.stream);
            return;
        }
        for (const auto& c : cs)
            PQTG_CUDA_CHECK(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDefault, dst.stream));
    };
    // all-gather-v of per-root pieces
    auto gather = [&](auto piece_of /* (Rank& self, uint32_t root) -> Piece */) {
        if (nc) {
            Rank& r = *sh.ranks[0];
            on(r);
            nccl_check(nc->group_start(), "ncclGroupStart");
            for (uint32_t g = 0; g < G; ++g) {
                const Piece pc = piece_of(r, g);
                if (pc.bytes == 0) continue;  // every rank skips the same roots (sizes are global)
                const void* send = g == r.g ? (pc.src ? pc.src : pc.dst) : pc.dst;
                nccl_check(nc->broadcast(send, pc.dst, pc.bytes, ncclUint8, (int)g, sh.comm, r.stream), "ncclBroadcast");
            }
            nccl_check(nc->group_end(), "ncclGroupEnd");
            return;
        }
        for (auto& rp : sh.ranks) mark(*rp);
        for (auto& rp : sh.ranks) {
            Rank& dst = *rp;
            on(dst);
            wait_all(dst);
            std::vector<CopySegment> cs;
            for (auto& sp : sh.ranks) {
                Rank& src = *sp;
                const Piece mine = piece_of(src, src.g);  // the root's own view of its piece
                const Piece there = piece_of(dst, src.g);
                const void* from = mine.src ? mine.src : mine.dst;
                if (from == there.dst || there.bytes == 0) continue;
                cs.push_back({there.dst, from, there.bytes});
            }
            copies(dst, cs);
        }
        for (auto& rp : sh.ranks) mark(*rp);
    };

    // queries from global rank 0
    if (bcast && G > 1 && !sh.sim) {
        gather([&](Rank& self, uint32_t root) -> Piece {
            const uint32_t i = rank_index(self);
            float* q = const_cast<float*>(d_queries[i] ? d_queries[i] : self.q);
            return Piece{nullptr, q, root == 0 ? nq * D * sizeof(float) : 0};
        });
    }
    auto qptr = [&](uint32_t i) -> const float* {
        Rank& r = *sh.ranks[i];
        return d_queries[i] ? d_queries[i] : r.q;
    };
    if (k == 0 || sh.n == 0) {  // search.cpp:130-132
        for (uint32_t i = 0; i < R; ++i) {
            Rank& r = *sh.ranks[i];
            on(r);
            PQTG_CUDA_CHECK(cudaMemsetAsync(d_counts[i], 0, nq * sizeof(uint32_t), r.stream));
            if (d_stats && d_stats[i]) PQTG_CUDA_CHECK(cudaMemsetAsync(d_stats[i], 0, nq * sizeof(pqtg_query_stats), r.stream));
            if (k && sh.n == 0) {
                PQTG_CUDA_CHECK(cudaMemsetAsync(d_ids[i], 0xFF, nq * k * sizeof(uint32_t), r.stream));
                PQTG_CUDA_CHECK(cudaMemsetAsync(d_dists[i], 0x7F, nq * k * sizeof(float), r.stream));
            }
        }
    } else {
        if (sh.sim) {
            std::vector<uint64_t> blo(G), bn(G);
            for (uint32_t g = 0; g < G; ++g) {
                blo[g] = blk[g].lo;
                bn[g] = blk[g].n;
            }
            sim_fill(sh, *sh.ranks[0], qptr(0), nq, blo, bn);
            PQTG_CUDA_CHECK(cudaEventRecord(sh.ranks[0]->ev[0], sh.ranks[0]->stream));
        }
        // S1 + S2: this block's traversal, bin selection and packed ranges
        for (uint32_t i = 0; i < R; ++i) {
            Rank& r = *sh.ranks[i];
            on(r);
            const DevParams& p = r.ix->prm;
            const Block b = blk[r.g];
            if (b.n) {
                const WsSlice sl = r.ws().slice(b.lo);
                launch_traverse(p, qptr(i) + b.lo * D, b.n, sl, r.stream);
                launch_binsel(p, b.n, sl, stats_of(i) + b.lo, r.stream);
            }
            launch_scan_counts(r.ws().nranges + b.lo, b.n, r.blk_off, r.stream);
            launch_pack_ranges(r.ws().ranges + b.lo * (uint64_t)std::max<uint32_t>(budget, 1), std::max<uint32_t>(budget, 1),
                               r.ws().nranges + b.lo, r.blk_off, b.n, r.packed, r.stream);
            if (i == 0) PQTG_CUDA_CHECK(cudaEventRecord(r.ev[1], r.stream));
        }
        // S3: packed sizes (host round trip). The batch's fine LUTs (S5) are queued behind the
        // size copy, so the GPU computes them while the host waits for the sizes.
        auto fine_luts = [&] {
            for (uint32_t i = 0; i < R; ++i) {
                Rank& r = *sh.ranks[i];
                on(r);
                launch_fine_lut(r.ix->prm, qptr(i), nq, r.ws().fine, r.stream);  // cheaper than exchanging the LUTs
            }
        };
        std::vector<uint64_t> total(G, 0);
        if (sh.sim) {
            Rank& r = *sh.ranks[0];
            PQTG_CUDA_CHECK(cudaMemcpyAsync(r.h_totals, r.blk_off + blk[r.g].n, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                            r.stream));
            PQTG_CUDA_CHECK(cudaEventRecord(r.sized, r.stream));
            fine_luts();
            PQTG_CUDA_CHECK(cudaEventSynchronize(r.sized));
            for (uint32_t g = 0; g < G; ++g) total[g] = g == r.g ? r.h_totals[0] : sh.simc->total[g];
        } else if (nc) {
            Rank& r = *sh.ranks[0];
            on(r);
            const Block b = blk[r.g];
            nccl_check(nc->all_gather(r.blk_off + b.n, r.d_totals, 1, ncclUint64, sh.comm, r.stream), "ncclAllGather");
            PQTG_CUDA_CHECK(cudaMemcpyAsync(r.h_totals, r.d_totals, G * sizeof(uint64_t), cudaMemcpyDeviceToHost, r.stream));
            PQTG_CUDA_CHECK(cudaEventRecord(r.sized, r.stream));
            fine_luts();
            PQTG_CUDA_CHECK(cudaEventSynchronize(r.sized));
            for (uint32_t g = 0; g < G; ++g) total[g] = r.h_totals[g];
        } else {
            for (auto& rp : sh.ranks) {
                Rank& r = *rp;
                on(r);
                PQTG_CUDA_CHECK(cudaMemcpyAsync(r.h_totals, r.blk_off + blk[r.g].n, sizeof(uint64_t),
                                                cudaMemcpyDeviceToHost, r.stream));
                PQTG_CUDA_CHECK(cudaEventRecord(r.sized, r.stream));
            }
            fine_luts();
            for (auto& rp : sh.ranks) {
                on(*rp);
                PQTG_CUDA_CHECK(cudaEventSynchronize(rp->sized));
                total[rp->g] = rp->h_totals[0];
            }
        }
        std::vector<uint64_t> toff(G + 1, 0);
        for (uint32_t g = 0; g < G; ++g) toff[g + 1] = toff[g] + total[g];
        for (auto& rp : sh.ranks) ensure_all_packed(*rp, toff[G]);
        if (sh.sim) {  // S4 simulated: every peer's piece arrives as a device copy of its bytes
            Rank& r = *sh.ranks[0];
            auto& c = *sh.simc;
            std::vector<CopySegment> cs;
            for (uint32_t g = 0; g < G; ++g) {
                const Block b = blk[g];
                if (g == r.g) {
                    cs.push_back({r.all_packed + toff[g], r.packed, total[g] * sizeof(uint2)});
                    if (b.n) cs.push_back({r.all_off + b.lo, r.blk_off, b.n * sizeof(uint64_t)});
                    continue;
                }
                // the cache's offsets are over its whole packed batch (= this batch's toff[g] + the
                // block's own offsets): base 0 for these blocks below
                cs.push_back({r.all_off + b.lo, c.off + b.lo, b.n * sizeof(uint64_t)});
                cs.push_back({r.ws().ncand + b.lo, c.ncand + b.lo, b.n * 4});
                cs.push_back({stats_of(0) + b.lo, c.stats + b.lo, b.n * sizeof(pqtg_query_stats)});
                cs.push_back({r.all_packed + toff[g], c.packed + c.toff[g], total[g] * sizeof(uint2)});
            }
            launch_copy_segments(cs, r.stream);
        } else {
        // S4: the blocks' fine LUTs, counters, stats and packed ranges to every rank
        gather([&](Rank& self, uint32_t root) -> Piece {  // the blocks' own range offsets (counts follow)
            const Block b = blk[root];
            return Piece{self.g == root ? self.blk_off : nullptr, self.all_off + b.lo, b.n * sizeof(uint64_t)};
        });
        gather([&](Rank& self, uint32_t root) -> Piece {
            const Block b = blk[root];
            return Piece{nullptr, self.ws().ncand + b.lo, b.n * sizeof(uint32_t)};
        });
        gather([&](Rank& self, uint32_t root) -> Piece {
            const Block b = blk[root];
            return Piece{nullptr, stats_of(rank_index(self)) + b.lo, b.n * sizeof(pqtg_query_stats)};
        });
        gather([&](Rank& self, uint32_t root) -> Piece {
            return Piece{self.g == root ? self.packed : nullptr, self.all_packed + toff[root], total[root] * sizeof(uint2)};
        });
        }
        // S5 + S6: the whole batch's ranges, then the re-rank of this shard's candidates
        for (uint32_t i = 0; i < R; ++i) {
            Rank& r = *sh.ranks[i];
            on(r);
            if (i == 0) PQTG_CUDA_CHECK(cudaEventRecord(r.ev[2], r.stream));
            const DevParams& p = r.ix->prm;
            BlockMap m{};
            m.G = G;
            for (uint32_t g = 0; g < G; ++g) {
                const bool cached = sh.sim && g != r.g;  // offsets over the simulation cache's batch
                m.lo[g] = blk[g].lo;
                m.base[g] = cached ? 0 : toff[g];
                m.vend[g] = cached ? toff[g] + total[g] : total[g];
            }
            m.lo[G] = nq;
            launch_unpack_blocks(r.all_packed, r.all_off, m, nq, std::max<uint32_t>(budget, 1), r.ws().ranges,
                                 r.ws().nranges, r.stream);
            launch_rerank(p, nq, (uint32_t)lk, r.ws().slice(0), r.l_ids, r.l_dists, r.l_counts, r.stream);
            if (exact) launch_exact_prefix(p, qptr(i), nq, (uint32_t)lk, r.l_ids, r.l_counts, r.l_exact, r.stream);
            r.ws().last_nq = nq;  // pqtg_workspace_read of this rank's view (pqtg_sharded_workspace)
            r.ws().last_stream = r.stream;
            if (i == 0) PQTG_CUDA_CHECK(cudaEventRecord(r.ev[3], r.stream));
        }
        // S7: all-to-all of the local lists by query block
        if (sh.sim) {  // the peers' lists of this block: stand-ins of the same size (this rank's own)
            Rank& r = *sh.ranks[0];
            const Block mine = blk[r.g];
            std::vector<CopySegment> cs;
            for (uint32_t j = 0; j < G && mine.n; ++j) {
                cs.push_back({r.r_ids + (uint64_t)j * mine.n * k, r.l_ids + mine.lo * k, mine.n * k * sizeof(uint32_t)});
                cs.push_back({r.r_dists + (uint64_t)j * mine.n * k, r.l_dists + mine.lo * k, mine.n * k * sizeof(float)});
                cs.push_back({r.r_counts + (uint64_t)j * mine.n, r.l_counts + mine.lo, mine.n * sizeof(uint32_t)});
            }
            launch_copy_segments(cs, r.stream);
        } else if (nc) {
            Rank& r = *sh.ranks[0];
            on(r);
            const Block mine = blk[r.g];
            nccl_check(nc->group_start(), "ncclGroupStart");
            for (uint32_t j = 0; j < G; ++j) {
                const Block bj = blk[j];
                nccl_check(nc->send(r.l_ids + bj.lo * lk, bj.n * lk, ncclUint32, (int)j, sh.comm, r.stream), "ncclSend");
                nccl_check(nc->send(r.l_dists + bj.lo * lk, bj.n * lk, ncclFloat32, (int)j, sh.comm, r.stream), "ncclSend");
                nccl_check(nc->send(r.l_counts + bj.lo, bj.n, ncclUint32, (int)j, sh.comm, r.stream), "ncclSend");
                if (exact)
                    nccl_check(nc->send(r.l_exact + bj.lo * lk, bj.n * lk, ncclFloat32, (int)j, sh.comm, r.stream),
                               "ncclSend");
                nccl_check(nc->recv(r.r_ids + (uint64_t)j * mine.n * lk, mine.n * lk, ncclUint32, (int)j, sh.comm, r.stream),
                           "ncclRecv");
                nccl_check(nc->recv(r.r_dists + (uint64_t)j * mine.n * lk, mine.n * lk, ncclFloat32, (int)j, sh.comm,
                                    r.stream), "ncclRecv");
                nccl_check(nc->recv(r.r_counts + (uint64_t)j * mine.n, mine.n, ncclUint32, (int)j, sh.comm, r.stream),
                           "ncclRecv");
                if (exact)
                    nccl_check(nc->recv(r.r_exact + (uint64_t)j * mine.n * lk, mine.n * lk, ncclFloat32, (int)j, sh.comm,
                                        r.stream), "ncclRecv");
            }
            nccl_check(nc->group_end(), "ncclGroupEnd");
        } else {
            for (auto& rp : sh.ranks) mark(*rp);
            for (auto& dp : sh.ranks) {
                Rank& dst = *dp;
                on(dst);
                wait_all(dst);
                const Block mine = blk[dst.g];
                if (!mine.n) continue;
                std::vector<CopySegment> cs;
                for (auto& sp : sh.ranks) {
                    Rank& src = *sp;
                    const uint64_t j = src.g;
                    cs.push_back({dst.r_ids + j * mine.n * lk, src.l_ids + mine.lo * lk, mine.n * lk * sizeof(uint32_t)});
                    cs.push_back({dst.r_dists + j * mine.n * lk, src.l_dists + mine.lo * lk, mine.n * lk * sizeof(float)});
                    cs.push_back({dst.r_counts + j * mine.n, src.l_counts + mine.lo, mine.n * sizeof(uint32_t)});
                    if (exact)
                        cs.push_back({dst.r_exact + j * mine.n * lk, src.l_exact + mine.lo * lk, mine.n * lk * sizeof(float)});
                }
                copies(dst, cs);
            }
        }
        // S8: merge of this block
        for (uint32_t i = 0; i < R; ++i) {
            Rank& r = *sh.ranks[i];
            on(r);
            const Block b = blk[r.g];
            if (b.n && exact)
                launch_merge_exact(G, b.n, (uint32_t)lk, Rx, k, r.r_ids, r.r_dists, r.r_exact, r.r_counts,
                                   stats_of(i) + b.lo, d_ids[i] + b.lo * k, d_dists[i] + b.lo * k, d_counts[i] + b.lo,
                                   r.stream);
            else if (b.n)
                launch_merge(G, b.n, k, r.r_ids, r.r_dists, r.r_counts, d_ids[i] + b.lo * k, d_dists[i] + b.lo * k,
                             d_counts[i] + b.lo, r.stream);
        }
        // S9: the merged blocks to every rank
        if (sh.sim) {  // the peers' merged blocks arrive: stand-in copies of the same bytes
            Rank& r = *sh.ranks[0];
            const Block mine = blk[r.g];
            std::vector<CopySegment> cs;
            for (uint32_t g = 0; g < G; ++g) {
                const Block b = blk[g];
                if (g == r.g || !b.n || !mine.n) continue;
                const uint64_t n = std::min(b.n, mine.n);
                cs.push_back({d_ids[0] + b.lo * k, d_ids[0] + mine.lo * k, n * k * 4});
                cs.push_back({d_dists[0] + b.lo * k, d_dists[0] + mine.lo * k, n * k * 4});
                cs.push_back({d_counts[0] + b.lo, d_counts[0] + mine.lo, n * 4});
            }
            launch_copy_segments(cs, r.stream);
        } else {
        gather([&](Rank& self, uint32_t root) -> Piece {
            const Block b = blk[root];
            return Piece{nullptr, d_ids[rank_index(self)] + b.lo * k, b.n * k * sizeof(uint32_t)};
        });
        gather([&](Rank& self, uint32_t root) -> Piece {
            const Block b = blk[root];
            return Piece{nullptr, d_dists[rank_index(self)] + b.lo * k, b.n * k * sizeof(float)};
        });
        gather([&](Rank& self, uint32_t root) -> Piece {
            const Block b = blk[root];
            return Piece{nullptr, d_counts[rank_index(self)] + b.lo, b.n * sizeof(uint32_t)};
        });
        if (exact)  // exact_evals were set by the block's merge
            gather([&](Rank& self, uint32_t root) -> Piece {
                const Block b = blk[root];
                return Piece{nullptr, stats_of(rank_index(self)) + b.lo, b.n * sizeof(pqtg_query_stats)};
            });
        }
    }
    // the caller's streams continue after the search
    for (uint32_t i = 0; i < R; ++i) {
        Rank& r = *sh.ranks[i];
        on(r);
        if (i == 0) PQTG_CUDA_CHECK(cudaEventRecord(r.ev[4], r.stream));
        if (!nc) wait_all(r);
        PQTG_CUDA_CHECK(cudaEventRecord(r.done, r.stream));
        PQTG_CUDA_CHECK(cudaStreamWaitEvent(caller(i), r.done, 0));
    }
}

}  // namespace pqtg

using namespace pqtg;

extern "C" {

int pqtg_nccl_unique_id(uint8_t* id) {
    return guarded_sh([&] {
        if (!id) throw Error{PQTG_ERR_ARG, "null argument"};
        ncclUniqueId u;
        nccl_check(Nccl::get().get_unique_id(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == PQTG_NCCL_ID_BYTES, "NCCL unique id size");
        std::memcpy(id, &u, sizeof(u));
        return PQTG_OK;
    });
}

static void check_shard(const DevIndex& ix, uint32_t world, uint32_t g) {
    const uint64_t per = ix.n / world, extra = ix.n % world;
    const uint64_t lo = g * per + std::min<uint64_t>(g, extra), hi = lo + per + (g < extra ? 1 : 0);
    const bool whole = world == 1 && ix.prm.shard_lo == 0 && ix.prm.shard_hi == ix.n;
    if (!whole && (ix.prm.shard_lo != lo || ix.prm.shard_hi != hi))
        throw Error{PQTG_ERR_ARG, "shard " + std::to_string(g) + " of " + std::to_string(world) + " must hold positions [" +
                                      std::to_string(lo) + ", " + std::to_string(hi) + ")"};
}

int pqtg_sharded_create_nccl(pqtg_index* shard, const uint8_t* nccl_id, uint32_t rank, uint32_t world,
                             uint64_t max_batch, pqtg_sharded** out) {
    return guarded_sh([&] {
        if (!shard || !nccl_id || !out || world == 0 || world > kMaxBlocks || rank >= world || max_batch == 0)
            throw Error{PQTG_ERR_ARG, "bad sharded arguments"};
        *out = nullptr;
        DevIndex& ix = *shard->dev;
        check_shard(ix, world, rank);
        auto sh = std::make_unique<pqtg_sharded>();
        sh->world = world;
        sh->nccl = true;
        sh->max_batch = max_batch;
        sh->block_max = (max_batch + world - 1) / world;
        sh->n = ix.n;
        sh->D = ix.prm.D;
        sh->L = ix.prm.L;
        sh->k1 = ix.prm.k1;
        sh->budget = ix.prm.budget;
        auto r = std::make_unique<Rank>();
        r->g = rank;
        r->ix = &ix;
        setup_rank(*sh, *r);
        sh->ranks.push_back(std::move(r));
        ncclUniqueId u;
        std::memcpy(&u, nccl_id, sizeof(u));
        PQTG_CUDA_CHECK(cudaSetDevice(ix.device));
        nccl_check(Nccl::get().comm_init_rank(&sh->comm, (int)world, u, (int)rank), "ncclCommInitRank");
        *out = sh.release();
        return PQTG_OK;
    });
}

int pqtg_sharded_create_local(pqtg_index* const* shards, uint32_t world, uint64_t max_batch, pqtg_sharded** out) {
    return guarded_sh([&] {
        if (!shards || !out || world == 0 || world > 16 || max_batch == 0) throw Error{PQTG_ERR_ARG, "bad sharded arguments"};
        *out = nullptr;
        auto sh = std::make_unique<pqtg_sharded>();
        sh->world = world;
        sh->max_batch = max_batch;
        sh->block_max = (max_batch + world - 1) / world;
        for (uint32_t g = 0; g < world; ++g) {
            if (!shards[g]) throw Error{PQTG_ERR_ARG, "null shard"};
            DevIndex& ix = *shards[g]->dev;
            if (g == 0) {
                sh->n = ix.n;
                sh->D = ix.prm.D;
                sh->L = ix.prm.L;
                sh->k1 = ix.prm.k1;
                sh->budget = ix.prm.budget;
            } else if (ix.n != sh->n || ix.prm.D != sh->D || ix.prm.L != sh->L || ix.prm.k1 != sh->k1 ||
                       ix.prm.budget != sh->budget) {
                throw Error{PQTG_ERR_ARG, "shards of different indexes"};
            }
            check_shard(ix, world, g);
            auto r = std::make_unique<Rank>();
            r->g = g;
            r->ix = &ix;
            setup_rank(*sh, *r);
            sh->ranks.push_back(std::move(r));
        }
        *out = sh.release();
        return PQTG_OK;
    });
}

int pqtg_sharded_create_sim(pqtg_index* shard, uint32_t rank, uint32_t world, uint64_t max_batch, pqtg_sharded** out) {
    return guarded_sh([&] {
        if (!shard || !out || world == 0 || world > 16 || rank >= world || max_batch == 0)
            throw Error{PQTG_ERR_ARG, "bad sharded arguments"};
        *out = nullptr;
        DevIndex& ix = *shard->dev;
        check_shard(ix, world, rank);
        auto sh = std::make_unique<pqtg_sharded>();
        sh->world = world;
        sh->sim = true;
        sh->max_batch = max_batch;
        sh->block_max = (max_batch + world - 1) / world;
        sh->n = ix.n;
        sh->D = ix.prm.D;
        sh->L = ix.prm.L;
        sh->k1 = ix.prm.k1;
        sh->budget = ix.prm.budget;
        auto r = std::make_unique<Rank>();
        r->g = rank;
        r->ix = &ix;
        setup_rank(*sh, *r);
        sh->ranks.push_back(std::move(r));
        *out = sh.release();
        return PQTG_OK;
    });
}

int pqtg_sharded_local_ranks(const pqtg_sharded* sh) { return sh ? (int)sh->ranks.size() : 0; }

pqtg_workspace* pqtg_sharded_workspace(pqtg_sharded* sh, uint32_t local_rank) {
    if (!sh || local_rank >= sh->ranks.size()) {
        set_error("bad sharded handle or local rank");
        return nullptr;
    }
    return sh->ranks[local_rank]->wsh.get();
}

int pqtg_sharded_search_device(pqtg_sharded* sh, const float* const* d_queries, uint64_t nq, uint32_t k, int broadcast,
                               uint32_t* const* d_ids, float* const* d_dists, uint32_t* const* d_counts,
                               pqtg_query_stats* const* d_stats, void* const* streams) {
    return guarded_sh([&] {
        if (!sh) throw Error{PQTG_ERR_ARG, "null argument"};
        std::lock_guard<std::mutex> lock(sh->mu);
        sharded_search(*sh, d_queries, nq, k, broadcast != 0, d_ids, d_dists, d_counts, d_stats, streams);
        return PQTG_OK;
    });
}

int pqtg_sharded_search(pqtg_sharded* sh, const float* queries, uint64_t nq, uint32_t dim, uint32_t k, uint32_t* ids,
                        float* dists, uint32_t* counts, pqtg_query_stats* stats) {
    return guarded_sh([&] {
        if (!sh) throw Error{PQTG_ERR_ARG, "null argument"};
        std::lock_guard<std::mutex> lock(sh->mu);
        if (nq > 0 && dim != sh->D) throw Error{PQTG_ERR_BAD_DIM, "knn_query_batch: query dimension mismatch"};
        if (nq > sh->max_batch) throw Error{PQTG_ERR_ARG, "nq exceeds the sharded handle's max_batch"};
        Rank& r0 = *sh->ranks[0];
        if (nq && r0.g == 0 && !queries) throw Error{PQTG_ERR_ARG, "rank 0 must pass the queries"};
        const uint32_t R = (uint32_t)sh->ranks.size();
        const uint32_t kk = std::max<uint32_t>(k, 1);
        std::vector<const float*> q(R);
        std::vector<uint32_t*> i(R), c(R);
        std::vector<float*> d(R);
        std::vector<pqtg_query_stats*> s(R);
        for (uint32_t x = 0; x < R; ++x) {
            Rank& r = *sh->ranks[x];
            ensure_k(*sh, r, kk);
            q[x] = r.q;
            i[x] = r.o_ids;
            d[x] = r.o_dists;
            c[x] = r.o_counts;
            s[x] = r.o_stats;
        }
        PQTG_CUDA_CHECK(cudaSetDevice(r0.ix->device));
        if (nq && r0.g == 0)
            PQTG_CUDA_CHECK(cudaMemcpyAsync(r0.q, queries, nq * sh->D * sizeof(float), cudaMemcpyHostToDevice, r0.stream));
        std::vector<void*> st(R);
        for (uint32_t x = 0; x < R; ++x) st[x] = sh->ranks[x]->stream;
        sharded_search(*sh, q.data(), nq, k, true, i.data(), d.data(), c.data(), s.data(), st.data());
        PQTG_CUDA_CHECK(cudaSetDevice(r0.ix->device));
        if (nq) {
            if (k && ids) PQTG_CUDA_CHECK(cudaMemcpyAsync(ids, r0.o_ids, nq * k * sizeof(uint32_t), cudaMemcpyDeviceToHost, r0.stream));
            if (k && dists)
                PQTG_CUDA_CHECK(cudaMemcpyAsync(dists, r0.o_dists, nq * k * sizeof(float), cudaMemcpyDeviceToHost, r0.stream));
            if (counts) PQTG_CUDA_CHECK(cudaMemcpyAsync(counts, r0.o_counts, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, r0.stream));
            if (stats)
                PQTG_CUDA_CHECK(cudaMemcpyAsync(stats, r0.o_stats, nq * sizeof(pqtg_query_stats), cudaMemcpyDeviceToHost,
                                                r0.stream));
        }
        for (auto& r : sh->ranks) {
            PQTG_CUDA_CHECK(cudaSetDevice(r->ix->device));
            PQTG_CUDA_CHECK(cudaStreamSynchronize(r->stream));
        }
        return PQTG_OK;
    });
}

int pqtg_sharded_stage_ms(pqtg_sharded* sh, float* ms4) {
    return guarded_sh([&] {
        if (!sh || !ms4) throw Error{PQTG_ERR_ARG, "null argument"};
        Rank& r = *sh->ranks[0];
        PQTG_CUDA_CHECK(cudaSetDevice(r.ix->device));
        PQTG_CUDA_CHECK(cudaEventSynchronize(r.ev[4]));
        for (int x = 0; x < 4; ++x) PQTG_CUDA_CHECK(cudaEventElapsedTime(&ms4[x], r.ev[x], r.ev[x + 1]));
        return PQTG_OK;
    });
}

void pqtg_sharded_destroy(pqtg_sharded* sh) { delete sh; }

}  // extern "C"
