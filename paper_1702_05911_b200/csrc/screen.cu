// screen.cu — north-star kernel (1): the level-2 distances of a query batch as a dense
// contraction on the 5th-generation tensor cores, plus the fp32-exact residual check.
//
// K1a tc_screen_kernel: for every part p, G = Y'_p · C''_pᵀ for a tile of 128 queries × NT
//   children (all k1·k2 children of all level-1 parents): Y' = Y − μ_p (the part's mean child),
//   C'' = C − μ_parent (each child minus its level-1 centroid), both small, so the products
//   are too. bf16x3 split (x = hi + lo, hi·hi + hi·lo + lo·hi) into one fp32 TMEM accumulator:
//   tcgen05.mma.cta_group::1.kind::f16, operands in shared memory in the K-major no-swizzle
//   core-matrix layout (coalesced 16-byte global loads, converted in registers), issued by one
//   thread, completion through tcgen05.commit → mbarrier, read back with tcgen05.ld.
//   The screened distance is then |y − c|² = |y − μ_i|² − 2 (G − (μ_i − μ_p)·c'') + |c''|², where
//   |y − μ_i|² is the exact level-1 distance of parent i that the traversal computes anyway.
// K1b traverse_screen_kernel (one CTA per (query, part)): the exact fine LUT and level-1 order
//   (pqtree.cpp:84-100) as in traverse.cu, then the w best parents' W = w·k2 children are ordered
//   by their screened distances. Each d̃ has a certified radius R (tensor-core error + the
//   reference's own fp32 rounding of l2_sq, see screen_radius); children whose intervals
//   [d̃ − R, d̃ + R] overlap form groups whose members get the reference's exact sequential
//   l2_sq (pqtree.cpp:109) and are ordered by (dist, parent, child) (:112-117). Groups are
//   ordered by their disjoint intervals, which the exact values would order identically. The
//   entries at ranks 0 and 1 are always exact (pick_slope_table reads them, binorder.cpp:52-65).
//   So the list's ORDER is the reference's and its first two distances are the reference's
//   bits; the remaining distances are the screened values (bin selection reads only ranks and
//   the first two distances when resort_bins is off; resort_bins uses the exact traversal).
#include <cuda_bf16.h>

#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kScThreads = 128;  // 4 warps = the 128 TMEM lanes (query rows) of the tile
constexpr int kScM = 128;
constexpr int kScKC = 64;        // K elements staged per chunk (4 MMA K-steps of 16)

// ---- tcgen05 / TMEM helpers (PTX ISA 8.6+, sm_100a)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 at 46
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

}  // namespace

// Core-matrix layout of an R × kScKC bf16 operand chunk: element (r, k) at byte
// (k / 8) · (R / 8) · 128 + (r / 8) · 128 + (r % 8) · 16 + (k % 8) · 2, i.e. LBO = R · 16 bytes
// between the two 8-wide K halves of an MMA K-step, SBO = 128 bytes between 8-row groups.
// Stores 4 consecutive k (k % 4 == 0) of row r: 8 bytes of hi, 8 of lo.
__device__ __forceinline__ void stage4(unsigned char* hi_base, unsigned char* lo_base, uint32_t R, uint32_t r,
                                      uint32_t k, const float* x) {
    uint32_t h[2], l[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(x[2 * i]), h1 = __float2bfloat16_rn(x[2 * i + 1]);
        const __nv_bfloat16 l0 = __float2bfloat16_rn(x[2 * i] - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(x[2 * i + 1] - __bfloat162float(h1));
        h[i] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
        l[i] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
    }
    const uint32_t off = (k / 8) * (R / 8) * 128 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<uint2*>(hi_base + off) = make_uint2(h[0], h[1]);
    *reinterpret_cast<uint2*>(lo_base + off) = make_uint2(l[0], l[1]);
}

template <int NT>
__global__ void __launch_bounds__(kScThreads) tc_screen_kernel(DevParams p, const float* __restrict__ Q, uint64_t nq,
                                                               float* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr uint32_t A_BYTES = kScM * kScKC * 2, B_BYTES = NT * kScKC * 2;
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;  // hi/lo A, hi/lo B of one K chunk
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar[2];

    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t part = blockIdx.y, m = p.m, kpad = p.scr_kpad, nj = p.scr_nj, D = p.D;
    const uint64_t q0 = (uint64_t)blockIdx.x * kScM;
    const uint32_t j0 = blockIdx.z * NT;  // first child of the tile
    const float* mu = p.scr_mu + (size_t)part * kpad;
    const float* crow = p.scr_c + ((size_t)part * nj + j0) * kpad;
    const bool vec = (D % 4 == 0) && (m % 4 == 0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                     "r"((uint32_t)NT));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    // idesc: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1, K-major A/B, N>>3 [17,23), M>>4 [24,29)
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                               ((uint32_t)(kScM >> 4) << 24);
    constexpr uint32_t kAIt = kScM * (kScKC / 4) / kScThreads;
    constexpr uint32_t kBIt = NT * (kScKC / 4) / kScThreads;
    float4 av[kAIt], bv[kBIt];
    // global -> registers for chunk k0: consecutive threads on consecutive 16-byte pieces of a row
    auto load = [&](uint32_t k0) {
        const uint32_t kc = kpad - k0 < (uint32_t)kScKC ? kpad - k0 : (uint32_t)kScKC, c4n = kc / 4;
#pragma unroll
        for (uint32_t it = 0; it < kAIt; ++it) {
            const uint32_t idx = it * kScThreads + tid, r = idx / c4n, k = (idx - r * c4n) * 4;
            const uint64_t q = q0 + r;
            av[it] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (idx < kScM * c4n && q < nq) {
                const float* yr = Q + q * D + (uint64_t)part * m + k0 + k;
                if (vec && k0 + k + 4 <= m) {
                    av[it] = __ldg(reinterpret_cast<const float4*>(yr));
                } else {
                    float t[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                    for (uint32_t i = 0; i < 4; ++i)
                        if (k0 + k + i < m) t[i] = __ldg(yr + i);
                    av[it] = make_float4(t[0], t[1], t[2], t[3]);
                }
            }
        }
#pragma unroll
        for (uint32_t it = 0; it < kBIt; ++it) {
            const uint32_t idx = it * kScThreads + tid, r = idx / c4n, k = (idx - r * c4n) * 4;
            bv[it] = idx < NT * c4n ? __ldg(reinterpret_cast<const float4*>(crow + (size_t)r * kpad + k0 + k))
                                    : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
    };
    // registers -> bf16 hi/lo core-matrix tiles of a stage (A centred on the part's mean child)
    auto stage_store = [&](uint32_t k0, unsigned char* st) {
        const uint32_t kc = kpad - k0 < (uint32_t)kScKC ? kpad - k0 : (uint32_t)kScKC, c4n = kc / 4;
#pragma unroll
        for (uint32_t it = 0; it < kAIt; ++it) {
            const uint32_t idx = it * kScThreads + tid, r = idx / c4n, k = (idx - r * c4n) * 4;
            if (idx < kScM * c4n) {
                const bool live = q0 + r < nq;
                float x[4] = {av[it].x, av[it].y, av[it].z, av[it].w};
                for (uint32_t i = 0; i < 4; ++i)
                    x[i] = (live && k0 + k + i < m) ? x[i] - __ldg(mu + k0 + k + i) : 0.0f;
                stage4(st, st + A_BYTES, kScM, r, k, x);
            }
        }
#pragma unroll
        for (uint32_t it = 0; it < kBIt; ++it) {
            const uint32_t idx = it * kScThreads + tid, r = idx / c4n, k = (idx - r * c4n) * 4;
            if (idx < NT * c4n) {
                const float x[4] = {bv[it].x, bv[it].y, bv[it].z, bv[it].w};
                stage4(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, NT, r, k, x);
            }
        }
    };
    // two-stage pipeline: chunk c's global loads are in flight while the tensor core multiplies
    // chunk c − 1; a stage is rewritten only after the MMAs that read it have committed
    const uint32_t nchunk = (kpad + kScKC - 1) / kScKC;
    uint32_t phase[2] = {0u, 0u};
    load(0);
    for (uint32_t c = 0; c < nchunk; ++c) {
        const uint32_t k0 = c * kScKC, st = c & 1u;
        unsigned char* sb = smem + (size_t)st * STAGE;
        if (c >= 2) {  // the MMAs of chunk c − 2 read this stage
            mbar_wait(&s_bar[st], phase[st]);
            phase[st] ^= 1u;
        }
        stage_store(k0, sb);
        if (c + 1 < nchunk) load(k0 + kScKC);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t kc = kpad - k0 < (uint32_t)kScKC ? kpad - k0 : (uint32_t)kScKC;
            for (uint32_t s = 0; s < kc / 16; ++s) {
                const uint32_t aoff = 2 * s * (kScM / 8) * 128, boff = 2 * s * (NT / 8) * 128;
                const uint64_t ah = umma_desc(smem_addr(sb + aoff), kScM * 16, 128);
                const uint64_t al = umma_desc(smem_addr(sb + A_BYTES + aoff), kScM * 16, 128);
                const uint64_t bh = umma_desc(smem_addr(sb + 2 * A_BYTES + boff), NT * 16, 128);
                const uint64_t bl = umma_desc(smem_addr(sb + 2 * A_BYTES + B_BYTES + boff), NT * 16, 128);
                umma_bf16(tmem, ah, bh, idesc, (k0 | s) != 0);
                umma_bf16(tmem, ah, bl, idesc, 1u);
                umma_bf16(tmem, al, bh, idesc, 1u);
            }
            umma_commit(&s_bar[st]);  // arrives when these MMAs (and their smem reads) are done
        }
    }
    // the last chunk's commit covers every earlier MMA (tcgen05 ops complete in issue order)
    {
        const uint32_t st = (nchunk - 1) & 1u;
        mbar_wait(&s_bar[st], phase[st]);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // epilogue: warp w owns TMEM lanes (query rows) 32w..32w+31; G rows to global
    const uint64_t q = q0 + tid;
    float* o = out + (q * p.P + part) * (uint64_t)nj + j0;
    for (uint32_t c0 = 0; c0 < (uint32_t)NT; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + ((warp * 32) << 16) + c0, r);
        if (q < nq) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(o + c0 + i) = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                                                     __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)NT));
}

// Certified radius R of a screened distance d̃: |d̃ − d_ref| <= R, d_ref the reference's sequential
// fp32 l2_sq(y_p, c, m). Tensor-core part: bf16x3 leaves <= 3·2^-18 of each |y'_t c''_t| and the
// fp32 accumulation (one rounding per MMA) <= m/16 · 3 · 2^-24 of their sum, so 2|Ĝ − G| <=
// 2^-14.8 Σ|y' c''| <= 2^-14.8 |y'||c''|; 2^-14 keeps a 1.7x margin. The level-1 distance l1 =
// |y − μ_i|² carries the reference's own rounding, <= (m + L/P + 4)·2^-24·l1; c'' and kc are
// fp32-rounded on the host (<= 2^-22 √(d̃|c''|²)), the combination rounds three times. The
// reference's l2_sq itself is within (m + 4)·2^-24 of the true distance.
__device__ __forceinline__ float screen_radius(float dt, float l1, float g, float kc, float yn, float cn,
                                               uint32_t m) {
    const float u = 5.9604645e-8f;  // 2^-24
    const float e = 6.1035156e-5f * sqrtf(yn * cn) + (float)(m + 16) * u * fabsf(l1) +
                    4.0f * u * (2.0f * fabsf(g) + 2.0f * fabsf(kc) + cn) + 2.3841858e-7f * sqrtf(fabsf(dt) * cn);
    return e + (float)(m + 4) * u * 1.05f * (fabsf(dt) + e) + 1e-30f;
}

template <int K1T, int K2T>
__global__ void __launch_bounds__(128) traverse_screen_kernel(DevParams p, const float* __restrict__ Q,
                                                              const float* __restrict__ scr,
                                                              float* __restrict__ fine_out,
                                                              float* __restrict__ l2d_out,
                                                              uint32_t* __restrict__ l2c_out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t k1 = K1T ? (uint32_t)K1T : p.k1, k2 = K2T ? (uint32_t)K2T : p.k2;
    const uint32_t P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W, nj0 = k1 * k2;
    float* y = reinterpret_cast<float*>(smem);                     // m
    float* fine = y + m;                                           // pp · k1
    float* l1d = fine + pp * k1;                                   // k1
    uint32_t* l1o = reinterpret_cast<uint32_t*>(l1d + k1);         // k1
    float* sg = reinterpret_cast<float*>(l1o + k1);                // nj0: G of every child
    float* skc = sg + nj0;                                         // nj0: kc
    float* scn = skc + nj0;                                        // nj0: |c''|^2
    float* dt = scn + nj0;                                         // W screened
    float* lo = dt + W;                                            // W lower bounds
    float* hi = lo + W;                                            // W upper bounds
    float* dx = hi + W;                                            // W exact distances
    uint32_t* code = reinterpret_cast<uint32_t*>(dx + W);          // W (parent << 16 | child)
    uint32_t* grp = code + W;                                      // W group id
    uint32_t* need = grp + W;                                      // W: exact needed
    uint32_t* ord = need + W;                                      // W: entry at lower-bound rank
    float* sq = reinterpret_cast<float*>(ord + W);                 // 4 warps × m squared terms
    __shared__ uint32_t s_nex, s_ex[128];
    __shared__ float s_yn[4];

    const uint64_t q = blockIdx.x / P;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    const uint32_t part = blockIdx.x - (uint32_t)q * P;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t jobs = pp * k1, f0 = part * pp;
    const float* yq = Q + q * p.D + (uint64_t)part * m;
    const float* mu = p.scr_mu + (size_t)part * p.scr_kpad;
    // every global load that does not depend on the level-1 order is issued first: the query
    // part, the tensor-core dot products and constants of all k1·k2 children
    const float* grow = scr + (q * P + part) * (uint64_t)p.scr_nj;
    const size_t cbase = (size_t)part * p.scr_nj;
    for (uint32_t j = tid; j < nj0; j += blockDim.x) {
        sg[j] = __ldg(grow + j);
        skc[j] = __ldg(p.scr_kc + cbase + j);
        scn[j] = __ldg(p.scr_cn + cbase + j);
    }
    float ynp = 0.0f;  // |y − μ_p|² (for the radius only)
    for (uint32_t t = tid; t < m; t += blockDim.x) {
        const float v = __ldg(yq + t);
        y[t] = v;
        const float c = v - __ldg(mu + t);
        ynp += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ynp += __shfl_xor_sync(0xffffffffu, ynp, o);
    if (lane == 0) s_yn[warp] = ynp;
    if (tid == 0) s_nex = 0;
    __syncthreads();

    // exact fine LUT of the part and level-1 order, as traverse.cu
    for (uint32_t idx = tid; idx < jobs; idx += blockDim.x) {
        const uint32_t lf = idx / k1, i = idx - lf * k1;
        const float* c = p.fine_t + (size_t)(f0 + lf) * fd * k1 + i;
        const float* yf = y + lf * fd;
        float acc = 0.0f;
        uint32_t t = 0;
        for (; t + 16 <= fd; t += 16) {
            float cv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) cv[u] = __ldg(c + (size_t)(t + u) * k1);
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = sq_step(acc, yf[t + u], cv[u]);
        }
        for (; t < fd; ++t) acc = sq_step(acc, yf[t], __ldg(c + (size_t)t * k1));
        fine[idx] = acc;
        fine_out[(q * p.L + f0 + lf) * k1 + i] = acc;
    }
    __syncthreads();
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        float tot = 0.0f;
        for (uint32_t lf = 0; lf < pp; ++lf) tot = __fadd_rn(tot, fine[lf * k1 + i]);
        l1d[i] = tot;
    }
    __syncthreads();
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        const float d = l1d[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[j];
            rank += (dj < d) || (dj == d && j < i);
        }
        l1o[rank] = i;
    }
    __syncthreads();

    // screened distances of the W children, |y − c|² = l1(i) − 2 (G − kc) + |c''|², with radii
    const float yn = s_yn[0] + s_yn[1] + s_yn[2] + s_yn[3];
    for (uint32_t j = tid; j < W; j += blockDim.x) {
        const uint32_t r = j / k2, c = j - r * k2, parent = l1o[r], child = parent * k2 + c;
        const float g = sg[child], kc = skc[child], cn = scn[child];
        const float l1 = l1d[parent];
        const float d = __fadd_rn(__fsub_rn(l1, __fmul_rn(2.0f, __fsub_rn(g, kc))), cn);
        const float rad = screen_radius(d, l1, g, kc, yn, cn, m);
        dt[j] = d;
        lo[j] = d - rad;
        hi[j] = d + rad;
        code[j] = (parent << 16) | c;
    }
    __syncthreads();
    // order by lower bound (ties by code): ord[rank] = entry
    for (uint32_t j = tid; j < W; j += blockDim.x) {
        const float l = lo[j];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < W; ++o) rank += (lo[o] < l) || (lo[o] == l && code[o] < code[j]);
        ord[rank] = j;
    }
    __syncthreads();
    // groups, one warp: in lower-bound order an entry starts a new group when its lower bound
    // exceeds every earlier upper bound (a running max: a warp max-scan with a carry per 32)
    if (warp == 0) {
        float carry_hi = -__int_as_float(0x7f800000);
        uint32_t carry_g = 0;
        for (uint32_t b = 0; b < W; b += 32) {
            const uint32_t r = b + lane;
            const bool live = r < W;
            const uint32_t e = live ? ord[r] : 0u;
            const float h = live ? hi[e] : -__int_as_float(0x7f800000);
            float incl = h;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl = fmaxf(incl, t);
            }
            float excl = __shfl_up_sync(0xffffffffu, incl, 1);
            excl = lane == 0 ? carry_hi : fmaxf(excl, carry_hi);
            const bool start = live && r > 0 && lo[e] > excl;
            uint32_t nstart = start ? 1u : 0u;  // inclusive count of group starts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, nstart, o);
                if (lane >= (uint32_t)o) nstart += t;
            }
            if (live) grp[e] = carry_g + nstart;
            carry_g += __shfl_sync(0xffffffffu, nstart, 31);
            carry_hi = fmaxf(carry_hi, __shfl_sync(0xffffffffu, incl, 31));
        }
    }
    __syncthreads();
    // exact for members of groups of two or more, and for ranks 0 and 1 (pick_slope_table): the
    // first group, and the second when the first is a single entry
    {
        const bool first_single = W < 2 || grp[ord[1]] != 0u;
        for (uint32_t r = tid; r < W; r += blockDim.x) {
            const uint32_t e = ord[r], g = grp[e];
            const bool shared = (r > 0 && grp[ord[r - 1]] == g) || (r + 1 < W && grp[ord[r + 1]] == g);
            need[e] = (shared || g == 0u || (first_single && g == 1u)) ? 1u : 0u;
        }
    }
    __syncthreads();
    if (warp == 0) {  // compact the marked entries
        uint32_t n = 0;
        for (uint32_t b = 0; b < W; b += 32) {
            const bool mk = b + lane < W && need[b + lane];
            const uint32_t bal = __ballot_sync(0xffffffffu, mk);
            if (mk) {
                const uint32_t at = n + __popc(bal & ((1u << lane) - 1u));
                if (at < 128) s_ex[at] = b + lane;
            }
            n += __popc(bal);
        }
        if (lane == 0) s_nex = n;
    }
    __syncthreads();
    const uint32_t nex = s_nex;
    // exact l2_sq(y_p, L2[part][parent][c], m) (pqtree.cpp:109) for the marked children: a warp
    // per child — lanes compute the rounded squares, lane 0 sums them in order
    float* wsq = sq + warp * m;
    for (uint32_t x = warp; x < W; x += blockDim.x / 32) {
        uint32_t j;
        if (nex <= 128) {
            if (x >= nex) break;
            j = s_ex[x];
        } else {  // more than 128 marked: walk all entries (rare)
            j = x;
            if (!need[j]) continue;
        }
        const uint32_t r = j / k2, c = j - r * k2;
        const float* b = p.l2_t + ((size_t)part * k1 + l1o[r]) * m * k2 + c;
        for (uint32_t t = lane; t < m; t += 32) {
            const float d = __fsub_rn(y[t], __ldg(b + (size_t)t * k2));
            wsq[t] = __fmul_rn(d, d);
        }
        __syncwarp();
        if (lane == 0) {
            float acc = 0.0f;
            uint32_t t = 0;
            for (; t + 8 <= m; t += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = wsq[t + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
            }
            for (; t < m; ++t) acc = __fadd_rn(acc, wsq[t]);
            dx[j] = acc;
        }
        __syncwarp();
    }
    __syncthreads();
    // final rank: by group, then (exact dist, code) inside groups; singletons keep d̃
    for (uint32_t j = tid; j < W; j += blockDim.x) {
        const uint32_t g = grp[j];
        const float d = need[j] ? dx[j] : dt[j];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < W; ++o) {
            const uint32_t go = grp[o];
            const float dd = need[o] ? dx[o] : dt[o];
            rank += go < g || (go == g && (dd < d || (dd == d && code[o] < code[j])));
        }
        const size_t out = (q * P + part) * W + rank;
        l2d_out[out] = d;
        l2c_out[out] = code[j];
    }
    qt_end(p, q, 0);
}

namespace {

size_t screen_smem(uint32_t nt) { return 2 * ((size_t)2 * kScM * kScKC * 2 + (size_t)2 * nt * kScKC * 2); }

size_t ts_smem(const DevParams& p) {
    return 4ull * ((size_t)p.m + (size_t)p.per_part * p.k1 + 2ull * p.k1 + 3ull * p.k1 * p.k2 + 8ull * p.W +
                   4ull * p.m) + 16;
}

uint32_t screen_nt(const DevParams& p) { return p.scr_nj >= 256 ? 256u : 64u; }

template <class K>
void allow(K kernel, int optin) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, kernel));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

}  // namespace

bool screen_ok(const DevParams& p) {
    return p.scr_c != nullptr && !p.resort && p.W <= 4096 && p.m <= 4096 && ts_smem(p) <= 96 * 1024;
}

void configure_screen() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    allow(tc_screen_kernel<64>, optin);
    allow(tc_screen_kernel<256>, optin);
    allow(traverse_screen_kernel<16, 8>, optin);
    allow(traverse_screen_kernel<32, 16>, optin);
    allow(traverse_screen_kernel<16, 16>, optin);
    allow(traverse_screen_kernel<0, 0>, optin);
}

void launch_screen_gemm(const DevParams& p, const float* queries, uint64_t nq, float* out, cudaStream_t s) {
    if (nq == 0) return;
    const uint32_t nt = screen_nt(p);
    const dim3 grid((unsigned)((nq + kScM - 1) / kScM), p.P, p.scr_nj / nt);
    if (nt == 256)
        tc_screen_kernel<256><<<grid, kScThreads, screen_smem(256), s>>>(p, queries, nq, out);
    else
        tc_screen_kernel<64><<<grid, kScThreads, screen_smem(64), s>>>(p, queries, nq, out);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_traverse_screen(const DevParams& p, const float* queries, uint64_t nq, const float* scr,
                            const WsSlice& ws, cudaStream_t s) {
    const unsigned grid = (unsigned)(nq * p.P);
    const size_t sm = ts_smem(p);
#define PQTG_TS(A, B) \
    traverse_screen_kernel<A, B><<<grid, 128, sm, s>>>(p, queries, scr, ws.fine, ws.l2_dist, ws.l2_code)
    if (p.k1 == 16 && p.k2 == 8) PQTG_TS(16, 8);
    else if (p.k1 == 32 && p.k2 == 16) PQTG_TS(32, 16);
    else if (p.k1 == 16 && p.k2 == 16) PQTG_TS(16, 16);
    else PQTG_TS(0, 0);
#undef PQTG_TS
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
