// build_kernels.cu — offline index construction on the GPU (SURVEY.md §8f "next" #3):
// per database vector the bin code (assign_bin + global_code, pqtree.cpp:12-38) and the line
// code (encode_line, linequant.cpp:84-152), both in the reference's exact fp32 operation
// order so the codes equal the CPU builder's for the same codebooks.
#include <cstdint>

#include "pqtg_internal.h"

namespace pqtg {

namespace {

__device__ __forceinline__ float dsq(float acc, float a, float b) {
    const float d = __fsub_rn(a, b);
    return __fadd_rn(acc, __fmul_rn(d, d));
}

__device__ __forceinline__ float ddot(float acc, float a, float b) { return __fadd_rn(acc, __fmul_rn(a, b)); }

}  // namespace

// One thread per (vector, part): nearest level-1 centroid (strict <, lowest index on ties,
// codebook.cpp:45-57), then nearest child of that parent; accumulate the positional code.
// l1: [P][k1][m], l2: [P][k1][k2][m] (reference layouts).
__global__ void assign_kernel(uint32_t D, uint32_t P, uint32_t k1, uint32_t k2, const float* __restrict__ l1,
                              const float* __restrict__ l2, const float* __restrict__ x, uint64_t n,
                              uint32_t* __restrict__ part_codes) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * P) return;
    const uint64_t v = t / P;
    const uint32_t p = (uint32_t)(t - v * P);
    const uint32_t m = D / P;
    const float* xp = x + v * D + (uint64_t)p * m;
    uint32_t best = 0;
    float bd = __uint_as_float(0x7F800000u);
    for (uint32_t i = 0; i < k1; ++i) {
        const float* c = l1 + ((uint64_t)p * k1 + i) * m;
        float acc = 0.0f;
        for (uint32_t d = 0; d < m; ++d) acc = dsq(acc, xp[d], c[d]);
        if (acc < bd) {
            bd = acc;
            best = i;
        }
    }
    uint32_t best2 = 0;
    float bd2 = __uint_as_float(0x7F800000u);
    for (uint32_t j = 0; j < k2; ++j) {
        const float* c = l2 + (((uint64_t)p * k1 + best) * k2 + j) * m;
        float acc = 0.0f;
        for (uint32_t d = 0; d < m; ++d) acc = dsq(acc, xp[d], c[d]);
        if (acc < bd2) {
            bd2 = acc;
            best2 = j;
        }
    }
    part_codes[t] = best * k2 + best2;  // flat_part_code (pqtree.hpp:18-21)
}

// global_code (pqtree.cpp:12-21): sum of flat part codes times (k1*k2)^p with u64 wrap.
__global__ void global_code_kernel(uint32_t P, uint64_t base, const uint32_t* __restrict__ part_codes, uint64_t n,
                                   uint64_t hash_size, uint64_t* __restrict__ out) {
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint64_t acc = 0, mult = 1;
    for (uint32_t p = 0; p < P; ++p) {
        acc += (uint64_t)part_codes[v * P + p] * mult;
        mult *= base;
    }
    out[v] = hash_size ? acc % hash_size : acc;
}

// encode_line (linequant.cpp:84-152), one thread per (vector, fine part).
// fine: [L][k1][fd] slices; sq: [L][k1] |slice|^2 (dot order); d2: [L][k1][k1].
__global__ void encode_kernel(uint32_t D, uint32_t L, uint32_t k1, const float* __restrict__ fine,
                              const float* __restrict__ sq, const float* __restrict__ d2, const float* __restrict__ x,
                              uint64_t n, uint8_t* __restrict__ lambda_out, uint16_t* __restrict__ pair_out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * L) return;
    const uint64_t v = t / L;
    const uint32_t f = (uint32_t)(t - v * L);
    const uint32_t fd = D / L;
    const float* xf = x + v * D + (uint64_t)f * fd;
    if (k1 == 1) {
        lambda_out[t] = 0;
        pair_out[t] = 0;
        return;
    }
    float xsq = 0.0f;
    for (uint32_t d = 0; d < fd; ++d) xsq = ddot(xsq, xf[d], xf[d]);
    // t[i] = dot(x_f, c_i): recomputed on demand (k1 up to 256 would not fit registers)
    auto tdot = [&](uint32_t i) {
        const float* c = fine + ((uint64_t)f * k1 + i) * fd;
        float acc = 0.0f;
        for (uint32_t d = 0; d < fd; ++d) acc = ddot(acc, xf[d], c[d]);
        return acc;
    };
    float best_res = __uint_as_float(0x7F800000u);
    uint32_t best_pair = 0, pid = 0;
    float best_lambda = 0.0f;
    bool found = false;
    for (uint32_t i = 0; i < k1; ++i) {
        const float ti = tdot(i);
        const float si = sq[f * k1 + i];
        const float ei = __fadd_rn(__fsub_rn(xsq, __fmul_rn(2.0f, ti)), si);
        for (uint32_t j = i + 1; j < k1; ++j, ++pid) {
            const float c2 = d2[((uint64_t)f * k1 + i) * k1 + j];
            if (c2 <= 0.0f) continue;
            const float tj = tdot(j);
            const float sj = sq[f * k1 + j];
            const float proj = __fadd_rn(__fsub_rn(tj, ti), __fmul_rn(0.5f, __fadd_rn(__fsub_rn(si, sj), c2)));
            float lam = __fdiv_rn(proj, c2);
            lam = lam < 0.0f ? 0.0f : (lam > 1.0f ? 1.0f : lam);  // std::clamp(v, 0, 1)
            const float res = __fadd_rn(__fsub_rn(ei, __fmul_rn(__fmul_rn(2.0f, lam), proj)),
                                        __fmul_rn(__fmul_rn(lam, lam), c2));
            if (res < best_res) {
                best_res = res;
                best_pair = pid;
                best_lambda = lam;
                found = true;
            }
        }
    }
    if (!found) {  // every pair degenerate: nearest single centroid (linequant.cpp:129-146)
        uint32_t bi = 0;
        float be = __uint_as_float(0x7F800000u);
        for (uint32_t i = 0; i < k1; ++i) {
            const float e = __fadd_rn(__fsub_rn(xsq, __fmul_rn(2.0f, tdot(i))), sq[f * k1 + i]);
            if (e < be) {
                be = e;
                bi = i;
            }
        }
        auto pidx = [&](uint32_t i, uint32_t j) { return i * k1 - i * (i + 1) / 2 + (j - i - 1); };
        if (bi + 1 < k1) {
            best_pair = pidx(bi, bi + 1);
            best_lambda = 0.0f;
        } else {
            best_pair = pidx(bi - 1, bi);
            best_lambda = 1.0f;
        }
    }
    // std::lround(255.0f * lambda): float product, round half away from zero
    lambda_out[t] = (uint8_t)lroundf(__fmul_rn(255.0f, best_lambda));
    pair_out[t] = (uint16_t)best_pair;
}

}  // namespace pqtg

using namespace pqtg;

extern "C" int pqtg_build_codes(const pqtg_config* cfg, const float* d_level1, const float* d_level2,
                                const float* d_fine, const float* d_fine_sq, const float* d_d2, const float* d_x,
                                uint64_t n, uint32_t* d_part_codes, uint64_t* d_slots, uint8_t* d_lambda,
                                uint16_t* d_pair, void* stream) {
    try {
        if (!cfg) throw Error{PQTG_ERR_ARG, "null config"};
        validate_config(*cfg);
        if (n == 0) return PQTG_OK;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const uint32_t P = cfg->p_tree, L = cfg->p_line;
        const unsigned tb = 128;
        if (d_part_codes && d_slots) {  // bins (NULL: line codes only)
            assign_kernel<<<(unsigned)((n * P + tb - 1) / tb), tb, 0, s>>>(cfg->dim, P, cfg->k1, cfg->k2, d_level1,
                                                                           d_level2, d_x, n, d_part_codes);
            PQTG_CUDA_CHECK(cudaGetLastError());
            global_code_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
                P, (uint64_t)cfg->k1 * cfg->k2, d_part_codes, n, cfg->hash_size, d_slots);
            PQTG_CUDA_CHECK(cudaGetLastError());
        }
        if (d_lambda && d_pair) {  // line codes (NULL: bins only)
            encode_kernel<<<(unsigned)((n * L + tb - 1) / tb), tb, 0, s>>>(cfg->dim, L, cfg->k1, d_fine, d_fine_sq,
                                                                           d_d2, d_x, n, d_lambda, d_pair);
            PQTG_CUDA_CHECK(cudaGetLastError());
        }
        return PQTG_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.status;
    }
}
