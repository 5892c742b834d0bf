// index_prep.cpp — host side of the device index: validation, re-layout and upload.
//
// Inputs are the arrays of pqt::PqtIndex (include/pqt/search.hpp:34-47) — from a
// pqtg_index_view or from a PQTINDEX v1 file (src/index_io.cpp:148-229). Outputs live in
// HBM in kernel-friendly layouts:
//   fine_t   [L][fd][k1]      level-1 centroid slices (build_fine_centroids, linequant.cpp:13-46)
//   l2_t     [P][k1][m][k2]   level-2 codebooks, child-fastest for coalesced traversal loads
//   pairs    [npairs]         lexicographic (i, j) pair enumeration (linequant.cpp:76-82)
//   c2       [L][npairs]      the stored d2[f][i][j] per pair (index_io.cpp:188-190)
//   streams  10 × W²          every slope table's full PairCursor order (binorder.cpp:69-110)
//   merge    materialized prefix of the slope-1 merge over pair ranks (binorder.cpp:229-240)
//   bitmap   H bits           non-empty slots
//   offsets  H+1 u32          InvertedLists::offsets narrowed (n < 2^32)
//   ids      positions        InvertedLists::ids of this shard
//   codes    positions × row  line codes permuted into SLOT order; pair width 1: interleaved
//                             (λ_f, pair_f) bytes; width 2: [λ_0..λ_{L-1}][u16 pair ids]
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <memory>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <unordered_set>

#include "pqtg_internal.h"

namespace pqtg {

DevIndex::~DevIndex() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (void* p : allocations) cudaFree(p);
    if (db) cudaFree(db);
    if (id2row) cudaFree(id2row);
    cudaSetDevice(prev);
}

// PqtConfig::validate (src/codebook.cpp:15-35)
void validate_config(const pqtg_config& c) {
    auto fail = [](const char* m) { throw Error{PQTG_ERR_CONFIG, std::string("config: ") + m}; };
    if (c.dim == 0 || c.p_tree == 0 || c.p_line == 0) fail("dim, p_tree and p_line must be positive");
    if (c.dim % c.p_tree != 0) fail("dim must be divisible by p_tree");
    if (c.p_line % c.p_tree != 0) fail("p_line must be a multiple of p_tree");
    if (c.dim % c.p_line != 0) fail("dim must be divisible by p_line");
    if (c.k1 < 1 || c.k2 < 1) fail("k1 and k2 must be at least 1");
    if (c.w < 1 || c.w > c.k1) fail("w must be in [1, k1]");
}

[[noreturn]] void unsupported(const std::string& m) { throw Error{PQTG_ERR_UNSUPPORTED, m}; }
[[noreturn]] void format(const std::string& m) { throw Error{PQTG_ERR_FORMAT, m}; }

namespace {


// PairCursor::next to exhaustion (binorder.cpp:80-110): table entries inside the grid in
// table order, then a row-major sweep of every cell the table did not emit.
std::vector<uint32_t> pair_stream(const uint32_t* entries, uint32_t tlen, uint32_t la, uint32_t lb) {
    std::vector<uint32_t> out;
    out.reserve((size_t)la * lb);
    std::vector<uint8_t> emitted((size_t)la * lb, 0);
    for (uint32_t e = 0; e < tlen; ++e) {
        const uint32_t a = entries[2 * e], b = entries[2 * e + 1];
        if (a < la && b < lb) {
            // a table may repeat a cell; PairCursor re-emits it (the emitted set is only
            // consulted by the sweep), so mirror that exactly
            emitted[(size_t)a * lb + b] = 1;
            out.push_back(a | (b << 16));
        }
    }
    for (uint32_t a = 0; a < la; ++a) {
        for (uint32_t b = 0; b < lb; ++b) {
            if (!emitted[(size_t)a * lb + b]) out.push_back(a | (b << 16));
        }
    }
    return out;
}

// Per-part bank map of the 1-byte line codes (k1 <= 16). The re-rank reads its per-query table
// T[f][t] = (E, c2) with 8-byte gathers, 16 lanes at a time, and entries whose slots t share the
// low nibble share a bank pair. The 16 lanes hold 16 consecutive candidates -- consecutive
// positions of an inverted list -- so which pairs meet there is a property of the index: sample
// groups of 16 consecutive positions, count per part how often two pairs meet, and give every
// pair (i, j) a nibble n (slot t = i << 4 | n; the pairs of one i need distinct nibbles) so that
// pairs that meet often sit in different bank pairs: greedy by how often a pair meets others,
// then passes of moves / swaps within an i while they lower the count. Returns t per [f][pair];
// empty when there are too few positions to sample.
std::vector<uint8_t> bank_map(uint32_t L, const std::vector<uint32_t>& pairs, uint64_t npos,
                              const std::function<uint32_t(uint64_t, uint32_t)>& pid_at) {
    const uint32_t np = (uint32_t)pairs.size();
    const uint64_t ng = std::min<uint64_t>(16384, npos / 16);
    if (np < 2 || ng < 256) return {};
    std::vector<uint8_t> out((size_t)L * np);
    auto one_part = [&](uint32_t f) {
        std::vector<uint32_t> w((size_t)np * np, 0);
        for (uint64_t g = 0; g < ng; ++g) {
            const uint64_t start = (npos - 16) * g / ng;
            uint32_t u[16];
            uint32_t m = 0;
            for (uint32_t r = 0; r < 16; ++r) {
                const uint32_t pid = pid_at(start + r, f);
                if (pid >= np) continue;
                bool seen = false;
                for (uint32_t x = 0; x < m && !seen; ++x) seen = u[x] == pid;
                if (!seen) u[m++] = pid;
            }
            for (uint32_t a = 0; a < m; ++a)
                for (uint32_t b = a + 1; b < m; ++b) {
                    ++w[(size_t)u[a] * np + u[b]];
                    ++w[(size_t)u[b] * np + u[a]];
                }
        }
        std::vector<uint32_t> nib(np, 16), first(np);
        std::vector<uint64_t> meets(np, 0);
        for (uint32_t a = 0; a < np; ++a) {
            first[a] = pairs[a] & 0xFFFFu;
            for (uint32_t b = 0; b < np; ++b) meets[a] += w[(size_t)a * np + b];
        }
        // cost of pair a in nibble n: how often it meets the pairs of other i holding n
        auto cost = [&](uint32_t a, uint32_t n) {
            uint64_t c = 0;
            for (uint32_t b = 0; b < np; ++b)
                if (b != a && nib[b] == n && first[b] != first[a]) c += w[(size_t)a * np + b];
            return c;
        };
        std::vector<uint32_t> order(np);
        for (uint32_t a = 0; a < np; ++a) order[a] = a;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return meets[x] > meets[y]; });
        std::vector<uint32_t> used(16, 0);  // per i: nibbles taken (bitmask)
        for (uint32_t a : order) {
            const uint32_t i = first[a], j = pairs[a] >> 16, pref = (i + j) & 15u;
            uint32_t best = 16;
            uint64_t bc = ~0ull;
            for (uint32_t k = 0; k < 16; ++k) {
                const uint32_t n = (pref + k) & 15u;  // ties keep the fixed slot's nibble first
                if (used[i] >> n & 1u) continue;
                const uint64_t c = cost(a, n);
                if (c < bc) {
                    bc = c;
                    best = n;
                }
            }
            nib[a] = best;
            used[i] |= 1u << best;
        }
        for (int pass = 0; pass < 4; ++pass) {
            bool moved = false;
            for (uint32_t a = 0; a < np; ++a) {
                const uint32_t i = first[a], na = nib[a];
                for (uint32_t n = 0; n < 16; ++n) {
                    if (n == na) continue;
                    uint32_t r = np;  // the pair of the same i holding n, if any
                    if (used[i] >> n & 1u)
                        for (uint32_t b = 0; b < np && r == np; ++b)
                            if (first[b] == i && nib[b] == n) r = b;
                    const int64_t before = (int64_t)cost(a, na) + (r < np ? (int64_t)cost(r, n) : 0);
                    nib[a] = n;
                    if (r < np) nib[r] = na;
                    const int64_t after = (int64_t)cost(a, n) + (r < np ? (int64_t)cost(r, na) : 0);
                    if (after < before) {
                        if (r == np) used[i] = (used[i] & ~(1u << na)) | (1u << n);
                        moved = true;
                        break;
                    }
                    nib[a] = na;
                    if (r < np) nib[r] = n;
                }
            }
            if (!moved) break;
        }
        for (uint32_t a = 0; a < np; ++a) out[(size_t)f * np + a] = (uint8_t)(first[a] << 4 | nib[a]);
    };
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    std::atomic<uint32_t> next{0};
    for (unsigned t = 0; t < std::min<unsigned>(hw, L); ++t)
        th.emplace_back([&] {
            for (uint32_t f; (f = next.fetch_add(1)) < L;) one_part(f);
        });
    for (auto& t : th) t.join();
    return out;
}

void parallel_rows(uint64_t n, const std::function<void(uint64_t, uint64_t)>& fn) {
    unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n < 65536 || hw == 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    const uint64_t chunk = (n + hw - 1) / hw;
    for (unsigned t = 0; t < hw; ++t) {
        const uint64_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        th.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : th) t.join();
}

template <class T>
T* upload(DevIndex& ix, const T* host, uint64_t count) {
    T* d = dev_alloc<T>(ix.allocations, count, &ix.bytes);
    if (count) PQTG_CUDA_CHECK(cudaMemcpy(d, host, count * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

}  // namespace

HostStreams build_streams(const uint32_t* entries, uint32_t table_len, uint32_t W, uint32_t P) {
    HostStreams hs;
    hs.W = W;
    hs.P = P;
    hs.W2 = (uint64_t)W * W;
    if (P == 1) {
        hs.total = W;
        return hs;
    }
    if (hs.W2 * kSlopeTables > (1ull << 28)) unsupported("w*k2 too large to materialize the slope streams");
    hs.pair.reserve(hs.W2 * kSlopeTables);
    for (uint32_t t = 0; t < kSlopeTables; ++t) {
        auto s = pair_stream(entries + (size_t)t * table_len * 2, table_len, W, W);
        // PairCursor re-emits a repeated in-bounds table cell; built tables never repeat one
        // (binorder.cpp:30-47 sorts a duplicate-free grid), so require that here
        if (s.size() != hs.W2) unsupported("slope table repeats grid cells");
        hs.pair.insert(hs.pair.end(), s.begin(), s.end());
    }
    if (P == 2) {
        hs.total = hs.W2;
        return hs;
    }
    // merge cursor over (u, v) in [0, W²)² with the slope-1 table (binorder.cpp:229-240):
    // its in-bounds prefix, then the sweep of the rows that prefix touched; every later row
    // is swept whole and is addressed in closed form (row0 + j / W², j % W²).
    const uint64_t len = hs.W2;
    const uint32_t* e5 = entries + (size_t)kSlopeOne * table_len * 2;
    std::unordered_set<uint64_t> emitted;
    int64_t last_row = -1;
    for (uint32_t e = 0; e < table_len; ++e) {
        const uint64_t a = e5[2 * e], b = e5[2 * e + 1];
        if (a < len && b < len) {
            if (!emitted.insert((a << 32) | b).second) unsupported("slope table repeats grid cells");
            hs.merge.push_back(make_uint2((uint32_t)a, (uint32_t)b));
            last_row = std::max<int64_t>(last_row, (int64_t)a);
        }
    }
    const uint64_t swept_rows = (uint64_t)(last_row + 1);
    if (swept_rows * len > (1ull << 26)) unsupported("slope-1 table too deep to materialize its sweep");
    for (uint64_t a = 0; a < swept_rows; ++a)
        for (uint64_t b = 0; b < len; ++b)
            if (!emitted.count((a << 32) | b)) hs.merge.push_back(make_uint2((uint32_t)a, (uint32_t)b));
    hs.merge_row0 = swept_rows;
    const long double tot = (long double)len * (long double)len;
    hs.total = tot > 4294967294.0L ? 4294967294ull : len * len;
    return hs;
}

// Host twin of the kernel's tuple addressing (kernels.cu tuple_slot): ranks of tuple s.
void HostStreams::tuple_at(uint64_t s, uint32_t ta, uint32_t tb, uint32_t* r) const {
    if (P == 1) {
        r[0] = (uint32_t)s;
        return;
    }
    if (P == 2) {
        const uint32_t e = pair[(size_t)ta * W2 + s];
        r[0] = e & 0xFFFF;
        r[1] = e >> 16;
        return;
    }
    uint64_t u, v;
    if (s < merge.size()) {
        u = merge[s].x;
        v = merge[s].y;
    } else {
        const uint64_t j = s - merge.size();
        u = merge_row0 + j / W2;
        v = j % W2;
    }
    const uint32_t ea = pair[(size_t)ta * W2 + u], eb = pair[(size_t)tb * W2 + v];
    r[0] = ea & 0xFFFF;
    r[1] = ea >> 16;
    r[2] = eb & 0xFFFF;
    r[3] = eb >> 16;
}

DevIndex* build_device_index(const Source& src, int device, uint64_t shard_lo, uint64_t shard_hi) {
    const pqtg_config& c = src.cfg;
    validate_config(c);
    const uint64_t n = src.n;
    const uint32_t P = c.p_tree, k1 = c.k1, k2 = c.k2, L = c.p_line;
    const uint32_t m = c.dim / P, per_part = L / P, fd = m / per_part;
    const uint64_t W64 = (uint64_t)c.w * k2;
    const uint64_t H = c.hash_size;

    // --- GPU-path limits (valid reference configs outside them are reported, not emulated)
    // part counts without a precomputed heuristic, or an index without its slope tables, use
    // the exact order (binorder.cpp:242-244)
    const bool exact_order = !(P == 1 || P == 2 || P == 4) || (P > 1 && src.table_count != kSlopeTables);
    if (P > 8) unsupported("p_tree must be <= 8");
    if (k1 > 65535 || k2 > 65535) unsupported("k1 and k2 must be < 65536");
    if (W64 > 65535) unsupported("w*k2 must be < 65536");
    if (n >= (1ull << 32)) unsupported("n must be < 2^32");
    if (H == 0 || H >= 0xFFFFFFFFull) unsupported("hash_size must be in [1, 2^32-1)");
    const uint32_t W = (uint32_t)W64;
    uint32_t tuple_bits = 1;
    while ((1ull << tuple_bits) < W) ++tuple_bits;
    if (exact_order && (uint64_t)tuple_bits * P > 64) unsupported("exact bin order: P * ceil(log2(w*k2)) > 64");
    const uint32_t npairs = k1 <= 1 ? 1u : k1 * (k1 - 1) / 2;
    const uint32_t pw = npairs <= 256 ? 1u : 2u;  // index_io.cpp:132
    if (npairs > 65536) unsupported("k1 too large for 16-bit pair ids");
    const uint64_t budget = std::min<uint64_t>(c.candidate_budget, n);
    if (budget > 65535) unsupported("candidate budget > 65535");
    if (shard_hi == 0 && shard_lo == 0) shard_hi = n;
    if (shard_lo > shard_hi || shard_hi > n) throw Error{PQTG_ERR_ARG, "bad shard range"};

    // offsets sanity (InvertedLists invariants, pqtree.cpp:40-57)
    if (src.offsets[0] != 0 || src.offsets[H] != n) format("inverted-list offsets do not cover [0, n)");

    int ndev = 0;
    PQTG_CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error{PQTG_ERR_ARG, "bad device ordinal"};
    PQTG_CUDA_CHECK(cudaSetDevice(device));

    auto ix = std::make_unique<DevIndex>();
    ix->cfg = c;
    ix->n = n;
    ix->device = device;
    DevParams& p = ix->prm;
    p.D = c.dim;
    p.P = P;
    p.k1 = k1;
    p.k2 = k2;
    p.w = c.w;
    p.L = L;
    p.m = m;
    p.fd = fd;
    p.per_part = per_part;
    p.W = W;
    p.npairs = npairs;
    p.pw = pw;
    p.row_bytes = (L * (1 + pw) + 15) / 16 * 16;
    p.budget = (uint32_t)budget;
    p.resort = c.resort_bins ? 1u : 0u;
    p.rerank_exact = c.rerank_exact;
    p.db = nullptr;
    p.H = H;
    p.n = n;
    p.shard_lo = shard_lo;
    p.shard_hi = shard_hi;
    p.log108 = std::log(1.08);  // glibc, as in binorder.cpp:62
    p.inv_log108 = 1.0 / p.log108;
    p.h_pow2 = (H & (H - 1)) == 0;
    p.exact_order = exact_order ? 1u : 0u;
    p.tuple_bits = tuple_bits;

    // positional multipliers (pqtree.cpp:12-21) and whether the u64 code can wrap
    const uint64_t base = (uint64_t)k1 * k2;
    uint64_t mult = 1;
    long double span = 1.0L;
    for (uint32_t q = 0; q < P; ++q) {
        p.mult[q] = mult;
        mult *= base;
        span *= (long double)base;
    }
    p.mod_fast = (span < 18446744073709551616.0L || p.h_pow2) ? 1u : 0u;

    // --- level-1 slices [f][t][i] and level-2 codebooks [p][i][t][c]
    {
        std::vector<float> fine_t((size_t)L * fd * k1);
        for (uint32_t f = 0; f < L; ++f) {
            const uint32_t pp = f / per_part, within = f % per_part;
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t t = 0; t < fd; ++t)
                    fine_t[((size_t)f * fd + t) * k1 + i] =
                        src.level1[((size_t)pp * k1 + i) * m + (size_t)within * fd + t];
        }
        p.fine_t = upload(*ix, fine_t.data(), fine_t.size());
        std::vector<float> l2_t((size_t)P * k1 * m * k2);
        for (uint32_t pp = 0; pp < P; ++pp)
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t ch = 0; ch < k2; ++ch)
                    for (uint32_t t = 0; t < m; ++t)
                        l2_t[(((size_t)pp * k1 + i) * m + t) * k2 + ch] =
                            src.level2[(((size_t)pp * k1 + i) * k2 + ch) * m + t];
        p.l2_t = upload(*ix, l2_t.data(), l2_t.size());
    }

    // --- tensor-core level-2 screen (screen.cu). Per part p: mu_p = the mean child; each child
    // c of parent i as c'' = c - mu_i (mu_i = the level-1 centroid), K-major rows [P][nj][kpad]
    // zero-padded; kc = (mu_i - mu_p) . c'' and |c''|^2 (fp64 sums). The screen then uses
    // |y - c|^2 = |y - mu_i|^2 - 2 ((y - mu_p) . c'' - kc) + |c''|^2 with small operands.
    {
        const uint32_t nj0 = k1 * k2;
        const uint32_t nt = nj0 >= 256 ? 256u : 64u;  // screen.cu's N tile
        const uint32_t nj = (nj0 + nt - 1) / nt * nt;
        const uint32_t kpad = (m + 15) / 16 * 16;
        p.scr_nj = nj;
        p.scr_kpad = kpad;
        std::vector<float> crow((size_t)P * nj * kpad, 0.0f), mu((size_t)P * kpad, 0.0f), cn((size_t)P * nj, 0.0f),
            kc((size_t)P * nj, 0.0f);
        for (uint32_t pp = 0; pp < P; ++pp) {
            const float* l2 = src.level2 + (size_t)pp * nj0 * m;  // [k1][k2][m] = [nj0][m]
            const float* l1 = src.level1 + (size_t)pp * k1 * m;   // [k1][m]
            std::vector<double> mup(m, 0.0);
            for (uint32_t t = 0; t < m; ++t) {
                for (uint32_t j = 0; j < nj0; ++j) mup[t] += l2[(size_t)j * m + t];
                mup[t] /= nj0;
                mu[(size_t)pp * kpad + t] = (float)mup[t];
            }
            for (uint32_t j = 0; j < nj0; ++j) {
                const float* par = l1 + (size_t)(j / k2) * m;
                double nrm = 0.0, kk = 0.0;
                for (uint32_t t = 0; t < m; ++t) {
                    const float v = (float)((double)l2[(size_t)j * m + t] - (double)par[t]);
                    crow[((size_t)pp * nj + j) * kpad + t] = v;
                    nrm += (double)v * v;
                    kk += ((double)par[t] - (double)mu[(size_t)pp * kpad + t]) * v;
                }
                cn[(size_t)pp * nj + j] = (float)nrm;
                kc[(size_t)pp * nj + j] = (float)kk;
            }
        }
        p.scr_c = upload(*ix, crow.data(), crow.size());
        p.scr_mu = upload(*ix, mu.data(), mu.size());
        p.scr_cn = upload(*ix, cn.data(), cn.size());
        p.scr_kc = upload(*ix, kc.data(), kc.size());
    }

    // --- pair enumeration and per-pair d2
    {
        std::vector<uint32_t> pairs(npairs);
        std::vector<float> c2((size_t)L * npairs);
        if (k1 <= 1) {
            pairs[0] = 0;
        } else {
            uint32_t q = 0;
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t j = i + 1; j < k1; ++j) pairs[q++] = i | (j << 16);
        }
        for (uint32_t f = 0; f < L; ++f)
            for (uint32_t q = 0; q < npairs; ++q) {
                const uint32_t i = pairs[q] & 0xFFFF, j = pairs[q] >> 16;
                c2[(size_t)f * npairs + q] = src.d2[((size_t)f * k1 + i) * k1 + j];
            }
        p.pairs = upload(*ix, pairs.data(), pairs.size());
        p.c2 = upload(*ix, c2.data(), c2.size());
    }

    // --- static bin-order streams (binorder.cpp:178-283)
    if (exact_order) {  // BinStream::total = the saturating product of the list lengths
        p.W2 = (uint64_t)W * W;
        uint64_t t = 1;
        for (uint32_t q = 0; q < P; ++q) t = t > (1ull << 62) / W ? (1ull << 62) : t * W;
        p.total_tuples = t;
    } else {
        HostStreams hs = build_streams(src.entries, src.table_len, W, P);
        p.W2 = hs.W2;
        p.total_tuples = hs.total;
        p.merge_count = hs.merge.size();
        p.merge_row0 = hs.merge_row0;
        if (!hs.pair.empty()) p.pair_streams = upload(*ix, hs.pair.data(), hs.pair.size());
        if (!hs.merge.empty()) p.merge = upload(*ix, hs.merge.data(), hs.merge.size());
        p.merge_fold_end = 0;
        while (p.merge_fold_end < hs.merge.size() && hs.merge[p.merge_fold_end].x < kPartialFold &&
               hs.merge[p.merge_fold_end].y < kPartialFold)
            ++p.merge_fold_end;
        if (!hs.merge.empty() && hs.W2 <= 65536) {  // the same (u, v) as u | v << 16: half the bytes per probe
            std::vector<uint32_t> m16(hs.merge.size());
            for (size_t i = 0; i < m16.size(); ++i) m16[i] = hs.merge[i].x | (hs.merge[i].y << 16);
            p.merge16 = upload(*ix, m16.data(), m16.size());
        }
    }

    // --- inverted lists: bitmap of non-empty slots, u32 offsets
    {
        std::vector<uint32_t> bitmap((H + 31) / 32, 0u);
        std::vector<uint32_t> off32(H + 1);
        for (uint64_t s = 0; s <= H; ++s) {
            if (s < H && src.offsets[s + 1] < src.offsets[s]) format("inverted-list offsets decrease");
            off32[s] = (uint32_t)src.offsets[s];
            if (s < H && src.offsets[s + 1] > src.offsets[s]) bitmap[s >> 5] |= 1u << (s & 31);
        }
        p.bitmap = upload(*ix, bitmap.data(), bitmap.size());
        p.offsets = upload(*ix, off32.data(), off32.size());
        // a coarse bitmap (1 bit per 2^coarse_shift slots, 2 KB, L1-resident) in front of the
        // fine one when the slots are sparse (< 1.8% occupied, P = 4): most empty probes never
        // reach L2. GIST1M (0.24% occupied) bins: 72 -> 51 us; the table size was swept
        // 128 KB .. 2 KB (71, 60, 54, 53, 52, 51, 51 us) -- a query's probes cluster, so a tiny
        // table stays in L1 and still filters
        uint64_t occupied = 0;
        for (uint32_t w : bitmap) occupied += (uint64_t)__builtin_popcount(w);
        uint32_t g = 4;
        while ((H >> g) > 2 * 1024 * 8) ++g;
        const double occ = H ? (double)occupied / (double)H : 1.0;
        p.coarse_shift = 0;
        p.bitmap_coarse = nullptr;
        // P = 4 only: its streams run thousands of mostly empty probes per query; P <= 2
        // queries probe a few dozen mostly non-empty slots (SIFT1M bins: 58.4 -> 60.6 us with it)
        if (occ < 0.018 && P == 4) {
            std::vector<uint32_t> coarse(((H >> g) + 32) / 32 + 1, 0u);
            for (uint64_t w = 0; w < bitmap.size(); ++w) {
                uint32_t bits = bitmap[w];
                while (bits) {
                    const uint64_t s = w * 32 + (uint64_t)__builtin_ctz(bits);
                    bits &= bits - 1;
                    coarse[(s >> g) >> 5] |= 1u << ((s >> g) & 31);
                }
            }
            p.coarse_shift = g;
            p.bitmap_coarse = upload(*ix, coarse.data(), coarse.size());
        }
    }

    // --- k1 <= 16 with 1-byte pairs: codes carry the pair's centroids as t = i << 4 | ((i + j) & 15)
    // (rerank_ij.cu: the low nibble picks the shared-memory bank pair of the per-query table, and
    // i + j spreads the lines of a part over the banks better than j alone); c2 by that byte
    p.code_ij = (pw == 1 && k1 <= 16) ? 1u : 0u;
    // 16 < k1 <= 32 (2-byte pair ids, <= 496 pairs): the stored u16 also carries the pair's
    // first centroid, v = pid | i << 9, so the re-rank reads fine[f][i] without the pair table
    p.code_pi = (pw == 2 && k1 <= 32 && npairs <= 512) ? 1u : 0u;
    std::vector<uint16_t> pi_of(p.code_pi ? npairs : 0);
    // DIRECT shards (rerank_ij.cu: ~budget/8 candidates per query at 8 shards, no per-query table)
    p.code_j = p.code_pi && shard_hi > shard_lo && (shard_hi - shard_lo) * 4 <= n ? 1u : 0u;
    if (p.code_j) {
        std::vector<float> c2v((size_t)L * 1024, 0.0f);
        uint32_t q = 0;
        for (uint32_t i = 0; i < k1; ++i)
            for (uint32_t j = i + 1; j < k1; ++j, ++q) pi_of[q] = (uint16_t)(i | (j << 5));
        for (uint32_t f = 0; f < L; ++f)
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t j = i + 1; j < k1; ++j)
                    c2v[(size_t)f * 1024 + (i | (j << 5))] = src.d2[((size_t)f * k1 + i) * k1 + j];
        p.c2v = upload(*ix, c2v.data(), c2v.size());
    }
    if (p.code_pi) {
        uint32_t q = 0;
        for (uint32_t i = 0; i < k1 && !p.code_j; ++i)
            for (uint32_t j = i + 1; j < k1; ++j, ++q) pi_of[q] = (uint16_t)(q | (i << 9));
        // c2 rows padded to 512 pairs: the DIRECT re-rank's loads use compile-time row offsets
        std::vector<float> c2p((size_t)L * 512, 0.0f);
        for (uint32_t f = 0; f < L; ++f) {
            uint32_t pq = 0;
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t j = i + 1; j < k1; ++j, ++pq)
                    c2p[(size_t)f * 512 + pq] = src.d2[((size_t)f * k1 + i) * k1 + j];
        }
        if (!p.code_j) p.c2p = upload(*ix, c2p.data(), c2p.size());
    }
    std::vector<uint8_t> ij_of(npairs, 0);
    auto tcode = [](uint32_t i, uint32_t j) { return (uint8_t)((i << 4) | ((i + j) & 15u)); };

    // --- this shard's ids and line codes in slot order
    const uint64_t npos = shard_hi - shard_lo;
    const uint32_t* shard_ids = src.pos_lambda_q ? src.ids : src.ids + shard_lo;  // shard-only ids: from 0
    // a position's stored pair id in part f (the staging loop below reads the same sources)
    auto pid_at = [&](uint64_t pos, uint32_t f) -> uint32_t {
        if (src.pos_lambda_q) return src.pos_pair_id[pos * L + f];
        const uint64_t id = shard_ids[pos];
        if (id >= n) return npairs;
        if (src.records) {
            const uint8_t* rec = src.records + (id * L + f) * (1 + src.record_pw);
            return src.record_pw == 1 ? rec[1] : (uint32_t)rec[1] | ((uint32_t)rec[2] << 8);
        }
        return src.pair_id[id * L + f];
    };
    std::vector<uint8_t> tmap;  // [L][npairs] slot per part (the bank map), empty: fixed slots
    if (p.code_ij) {
        std::vector<uint32_t> pr;
        if (k1 > 1) {
            uint32_t q = 0;
            for (uint32_t i = 0; i < k1; ++i)
                for (uint32_t j = i + 1; j < k1; ++j, ++q) {
                    ij_of[q] = tcode(i, j);
                    pr.push_back(i | (j << 16));
                }
        }
        static const bool no_map = [] {
            const char* e = std::getenv("PQTG_BANK_MAP");
            return e && std::strcmp(e, "0") == 0;
        }();
        if (!no_map && !rerank_needs_fixed_slots()) tmap = bank_map(L, pr, npos, pid_at);
        std::vector<float> c2ij((size_t)L * 256, 0.0f);
        if (tmap.empty()) {
            for (uint32_t f = 0; f < L; ++f)
                for (uint32_t i = 0; i < k1; ++i)
                    for (uint32_t j = 0; j < k1; ++j)
                        c2ij[(size_t)f * 256 + tcode(i, j)] = src.d2[((size_t)f * k1 + i) * k1 + j];
        } else {
            std::vector<uint2> c2slot((size_t)L * npairs);
            std::vector<uint8_t> jt((size_t)L * 256, 0);
            for (uint32_t f = 0; f < L; ++f)
                for (uint32_t q = 0; q < npairs; ++q) {
                    const uint32_t i = pr[q] & 0xFFFFu, j = pr[q] >> 16, t = tmap[(size_t)f * npairs + q];
                    const float d = src.d2[((size_t)f * k1 + i) * k1 + j];
                    c2ij[(size_t)f * 256 + t] = d;
                    uint32_t bits;
                    std::memcpy(&bits, &d, 4);
                    c2slot[(size_t)f * npairs + q] = make_uint2(bits, t);
                    jt[(size_t)f * 256 + t] = (uint8_t)j;
                }
            p.c2slot = upload(*ix, c2slot.data(), c2slot.size());
            p.jt_ij = upload(*ix, jt.data(), jt.size());
        }
        p.c2ij = upload(*ix, c2ij.data(), c2ij.size());
    }
    p.ids = upload(*ix, shard_ids, npos);
    {
        uint8_t* dcodes = dev_alloc<uint8_t>(ix->allocations, npos * p.row_bytes + 16, &ix->bytes);
        p.codes = dcodes;
        const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / p.row_bytes);
        std::vector<uint8_t> stage((size_t)std::min(chunk, std::max<uint64_t>(npos, 1)) * p.row_bytes);
        std::atomic<bool> bad_pid{false}, bad_id{false};
        for (uint64_t b = 0; b < npos; b += chunk) {
            const uint64_t e = std::min(npos, b + chunk);
            parallel_rows(e - b, [&](uint64_t lo, uint64_t hi) {
                for (uint64_t r = lo; r < hi; ++r) {
                    const uint64_t id = shard_ids[b + r];
                    uint8_t* row = stage.data() + r * p.row_bytes;
                    std::memset(row, 0, p.row_bytes);
                    if (id >= n) {
                        bad_id = true;
                        continue;
                    }
                    for (uint32_t f = 0; f < L; ++f) {
                        uint32_t lq, pid;
                        if (src.pos_lambda_q) {  // position-ordered shard codes
                            lq = src.pos_lambda_q[(b + r) * L + f];
                            pid = src.pos_pair_id[(b + r) * L + f];
                        } else if (src.records) {
                            const uint8_t* rec = src.records + (id * L + f) * (1 + src.record_pw);
                            lq = rec[0];
                            pid = src.record_pw == 1 ? rec[1] : (uint32_t)rec[1] | ((uint32_t)rec[2] << 8);
                        } else {
                            lq = src.lambda_q[id * L + f];
                            pid = src.pair_id[id * L + f];
                        }
                        if (pid >= npairs) bad_pid = true;
                        if (pw == 1) {  // interleaved (lambda, pair) per part
                            row[2 * f] = (uint8_t)lq;
                            // k1 <= 16: store the pair as its centroids (i << 4 | j), so the
                            // re-rank indexes the fine row and c2[f][i][j] directly
                            row[2 * f + 1] = (uint8_t)(p.code_ij && pid < npairs
                                                           ? (tmap.empty() ? ij_of[pid] : tmap[(size_t)f * npairs + pid])
                                                           : pid);
                        } else {        // lambda block, then little-endian u16 pair ids (| i << 9)
                            const uint32_t v = p.code_pi && pid < npairs ? pi_of[pid] : pid;
                            row[f] = (uint8_t)lq;
                            row[L + 2 * f] = (uint8_t)(v & 0xFF);
                            row[L + 2 * f + 1] = (uint8_t)(v >> 8);
                        }
                    }
                }
            });
            if (bad_pid) format("line code pair id out of range");
            if (bad_id) format("inverted-list id out of range");
            PQTG_CUDA_CHECK(cudaMemcpy(dcodes + b * p.row_bytes, stage.data(), (e - b) * p.row_bytes,
                                       cudaMemcpyHostToDevice));
        }
    }
    configure_kernels(p, 0);
    return ix.release();
}

}  // namespace pqtg
