/*
 * pqt_oracle.c — TEST INFRASTRUCTURE ONLY. Plain-C restatement of the reference query path,
 * used as the parity checker for the CUDA kernels (see pqt_oracle.h for who may call it).
 *
 * Arithmetic contract: every fp32 operation rounds separately, in the
 * reference's order; compiled with -ffp-contract=off on x86-64 (SSE, no FMA), exactly as the
 * reference is compiled without -march.
 */
#define _GNU_SOURCE
#include "pqt_oracle.h"

#include <errno.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[512];

static void set_err(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
}

const char* pqto_last_error(void) { return g_err; }

struct pqto_index {
    pqtg_config cfg;
    uint64_t n;
    float* level1;          /* P × k1 × m */
    float* level2;          /* P × k1 × k2 × m */
    float* d2;              /* L × k1 × k1 */
    uint32_t table_count, table_len;
    double* slopes;
    uint32_t* entries;      /* count × len × 2 */
    uint64_t* offsets;      /* H + 1 */
    uint32_t* ids;          /* n */
    uint8_t* lambda_q;      /* n × L */
    uint16_t* pair_id;      /* n × L */
    /* derived */
    uint32_t m, fd, per_part, W;
    float* fine;            /* L × k1 × fd: FineCentroids::slices (linequant.cpp:13-46) */
    uint16_t* pairs;        /* npairs × 2: PairDistanceTable::pairs (linequant.cpp:76-82) */
    uint32_t npairs;
    const float* db;        /* borrowed raw vectors n × dim (PqtIndex::database), or NULL */
    /* a position shard (pqto_from_shard_view): ids and codes hold only positions
     * [shard_lo, shard_hi), codes in POSITION order; offsets/ids/codes are borrowed */
    int is_shard;
    uint64_t shard_lo, shard_hi;
};

/* ---------------------------------------------------------------- small containers */

typedef struct {
    uint64_t* keys;
    uint64_t cap;   /* power of two */
    uint64_t size;
} u64set;

#define SET_EMPTY UINT64_MAX

static int set_init(u64set* s, uint64_t expect) {
    uint64_t cap = 16;
    while (cap < expect * 2) cap <<= 1;
    s->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
    if (!s->keys) return -1;
    memset(s->keys, 0xff, cap * sizeof(uint64_t));
    s->cap = cap;
    s->size = 0;
    return 0;
}

static void set_free(u64set* s) { free(s->keys); s->keys = NULL; }

static uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    return x;
}

static int set_contains(const u64set* s, uint64_t k) {
    uint64_t i = mix64(k) & (s->cap - 1);
    for (;;) {
        if (s->keys[i] == SET_EMPTY) return 0;
        if (s->keys[i] == k) return 1;
        i = (i + 1) & (s->cap - 1);
    }
}

/* returns 1 when inserted, 0 when already present, -1 on OOM */
static int set_insert(u64set* s, uint64_t k) {
    if ((s->size + 1) * 2 > s->cap) {
        u64set t;
        if (set_init(&t, s->cap) != 0) return -1;
        for (uint64_t i = 0; i < s->cap; ++i) {
            if (s->keys[i] != SET_EMPTY) {
                uint64_t j = mix64(s->keys[i]) & (t.cap - 1);
                while (t.keys[j] != SET_EMPTY) j = (j + 1) & (t.cap - 1);
                t.keys[j] = s->keys[i];
                t.size++;
            }
        }
        set_free(s);
        *s = t;
    }
    uint64_t i = mix64(k) & (s->cap - 1);
    for (;;) {
        if (s->keys[i] == SET_EMPTY) {
            s->keys[i] = k;
            s->size++;
            return 1;
        }
        if (s->keys[i] == k) return 0;
        i = (i + 1) & (s->cap - 1);
    }
}

typedef struct {
    uint32_t* a;    /* pairs of u32 */
    uint64_t size, cap;
} pairvec;

static int pv_push(pairvec* v, uint32_t x, uint32_t y) {
    if (v->size == v->cap) {
        uint64_t nc = v->cap ? v->cap * 2 : 1024;
        uint32_t* na = (uint32_t*)realloc(v->a, nc * 2 * sizeof(uint32_t));
        if (!na) return -1;
        v->a = na;
        v->cap = nc;
    }
    v->a[2 * v->size] = x;
    v->a[2 * v->size + 1] = y;
    v->size++;
    return 0;
}

/* ---------------------------------------------------------------- index setup */

/* PqtConfig::validate (src/codebook.cpp:15-35) */
static int validate_cfg(const pqtg_config* c) {
    if (c->dim == 0 || c->p_tree == 0 || c->p_line == 0) { set_err("config: dim, p_tree and p_line must be positive"); return PQTG_ERR_CONFIG; }
    if (c->dim % c->p_tree != 0) { set_err("config: dim must be divisible by p_tree"); return PQTG_ERR_CONFIG; }
    if (c->p_line % c->p_tree != 0) { set_err("config: p_line must be a multiple of p_tree"); return PQTG_ERR_CONFIG; }
    if (c->dim % c->p_line != 0) { set_err("config: dim must be divisible by p_line"); return PQTG_ERR_CONFIG; }
    if (c->k1 < 1 || c->k2 < 1) { set_err("config: k1 and k2 must be at least 1"); return PQTG_ERR_CONFIG; }
    if (c->w < 1 || c->w > c->k1) { set_err("config: w must be in [1, k1]"); return PQTG_ERR_CONFIG; }
    return 0;
}

/* build_fine_centroids (src/linequant.cpp:13-46) and the pair enumeration of build_pair_table
 * (src/linequant.cpp:60-82). d2 itself is the stored table (index_io.cpp:188-190). */
static int derive(pqto_index* ix) {
    const pqtg_config* c = &ix->cfg;
    ix->m = c->dim / c->p_tree;
    ix->per_part = c->p_line / c->p_tree;
    ix->fd = ix->m / ix->per_part;
    ix->W = c->w * c->k2;
    ix->fine = (float*)malloc((size_t)c->p_line * c->k1 * ix->fd * sizeof(float));
    if (!ix->fine) return PQTG_ERR_OOM;
    for (uint32_t f = 0; f < c->p_line; ++f) {
        uint32_t p = f / ix->per_part, within = f % ix->per_part;
        for (uint32_t i = 0; i < c->k1; ++i) {
            const float* src = ix->level1 + ((size_t)p * c->k1 + i) * ix->m + (size_t)within * ix->fd;
            memcpy(ix->fine + ((size_t)f * c->k1 + i) * ix->fd, src, ix->fd * sizeof(float));
        }
    }
    ix->npairs = c->k1 <= 1 ? 1u : c->k1 * (c->k1 - 1) / 2;
    ix->pairs = (uint16_t*)malloc((size_t)ix->npairs * 2 * sizeof(uint16_t));
    if (!ix->pairs) return PQTG_ERR_OOM;
    if (c->k1 <= 1) {
        ix->pairs[0] = 0;
        ix->pairs[1] = 0;
    } else {
        uint32_t q = 0;
        for (uint32_t i = 0; i < c->k1; ++i)
            for (uint32_t j = i + 1; j < c->k1; ++j) {
                ix->pairs[2 * q] = (uint16_t)i;
                ix->pairs[2 * q + 1] = (uint16_t)j;
                ++q;
            }
    }
    return 0;
}

void pqto_free(pqto_index* ix) {
    if (!ix) return;
    free(ix->level1); free(ix->level2); free(ix->d2); free(ix->slopes); free(ix->entries);
    if (!ix->is_shard) { free(ix->offsets); free(ix->ids); free(ix->lambda_q); free(ix->pair_id); }
    free(ix->fine); free(ix->pairs);
    free(ix);
}

static void* dup_bytes(const void* src, size_t bytes) {
    void* p = malloc(bytes ? bytes : 1);
    if (p && bytes) memcpy(p, src, bytes);
    return p;
}

pqto_index* pqto_from_view(const pqtg_index_view* v) {
    if (!v) { set_err("null view"); return NULL; }
    if (validate_cfg(&v->config) != 0) return NULL;
    pqto_index* ix = (pqto_index*)calloc(1, sizeof *ix);
    if (!ix) { set_err("out of memory"); return NULL; }
    const pqtg_config* c = &v->config;
    ix->cfg = *c;
    ix->n = v->n;
    uint32_t m = c->dim / c->p_tree;
    ix->level1 = (float*)dup_bytes(v->level1, (size_t)c->p_tree * c->k1 * m * sizeof(float));
    ix->level2 = (float*)dup_bytes(v->level2, (size_t)c->p_tree * c->k1 * c->k2 * m * sizeof(float));
    ix->d2 = (float*)dup_bytes(v->d2, (size_t)c->p_line * c->k1 * c->k1 * sizeof(float));
    ix->table_count = v->table_count;
    ix->table_len = v->table_len;
    ix->slopes = (double*)dup_bytes(v->table_slopes, (size_t)v->table_count * sizeof(double));
    ix->entries = (uint32_t*)dup_bytes(v->table_entries, (size_t)v->table_count * v->table_len * 2 * sizeof(uint32_t));
    ix->offsets = (uint64_t*)dup_bytes(v->offsets, (size_t)(c->hash_size + 1) * sizeof(uint64_t));
    ix->ids = (uint32_t*)dup_bytes(v->ids, (size_t)v->n * sizeof(uint32_t));
    ix->lambda_q = (uint8_t*)dup_bytes(v->lambda_q, (size_t)v->n * c->p_line);
    ix->pair_id = (uint16_t*)dup_bytes(v->pair_id, (size_t)v->n * c->p_line * sizeof(uint16_t));
    if (!ix->level1 || !ix->level2 || !ix->d2 || !ix->slopes || !ix->entries || !ix->offsets ||
        !ix->ids || !ix->lambda_q || !ix->pair_id || derive(ix) != 0) {
        set_err("out of memory");
        pqto_free(ix);
        return NULL;
    }
    return ix;
}

/* One position shard [v->shard_lo, v->shard_hi) of an n-vector index, as a sharded GPU
 * deployment holds it (pqtg_index_create_shard): v->offsets covers the whole index, v->ids the
 * shard's positions, and lambda_q / pair_id the shard's rows in position order. The big arrays
 * are borrowed (they must outlive the oracle). knn on it re-ranks only the shard's candidates
 * (search.cpp:221-227 restricted to the range) into that shard's local top-k. */
pqto_index* pqto_from_shard_view(const pqtg_index_view* v, const uint8_t* lambda_q, const uint16_t* pair_id) {
    if (!v || !lambda_q || !pair_id) { set_err("null view"); return NULL; }
    if (validate_cfg(&v->config) != 0) return NULL;
    if (v->shard_lo > v->shard_hi || v->shard_hi > v->n) { set_err("bad shard range"); return NULL; }
    pqto_index* ix = (pqto_index*)calloc(1, sizeof *ix);
    if (!ix) { set_err("out of memory"); return NULL; }
    const pqtg_config* c = &v->config;
    ix->cfg = *c;
    ix->n = v->n;
    ix->is_shard = 1;
    ix->shard_lo = v->shard_lo;
    ix->shard_hi = v->shard_hi;
    uint32_t m = c->dim / c->p_tree;
    ix->level1 = (float*)dup_bytes(v->level1, (size_t)c->p_tree * c->k1 * m * sizeof(float));
    ix->level2 = (float*)dup_bytes(v->level2, (size_t)c->p_tree * c->k1 * c->k2 * m * sizeof(float));
    ix->d2 = (float*)dup_bytes(v->d2, (size_t)c->p_line * c->k1 * c->k1 * sizeof(float));
    ix->table_count = v->table_count;
    ix->table_len = v->table_len;
    ix->slopes = (double*)dup_bytes(v->table_slopes, (size_t)v->table_count * sizeof(double));
    ix->entries = (uint32_t*)dup_bytes(v->table_entries, (size_t)v->table_count * v->table_len * 2 * sizeof(uint32_t));
    ix->offsets = (uint64_t*)v->offsets;
    ix->ids = (uint32_t*)v->ids;
    ix->lambda_q = (uint8_t*)lambda_q;
    ix->pair_id = (uint16_t*)pair_id;
    if (!ix->level1 || !ix->level2 || !ix->d2 || !ix->slopes || !ix->entries || derive(ix) != 0) {
        set_err("out of memory");
        pqto_free(ix);
        return NULL;
    }
    return ix;
}

void pqto_view(const pqto_index* ix, pqtg_index_view* v) {
    memset(v, 0, sizeof *v);
    v->config = ix->cfg;
    v->n = ix->n;
    v->level1 = ix->level1;
    v->level2 = ix->level2;
    v->d2 = ix->d2;
    v->table_count = ix->table_count;
    v->table_len = ix->table_len;
    v->table_slopes = ix->slopes;
    v->table_entries = ix->entries;
    v->offsets = ix->offsets;
    v->ids = ix->ids;
    v->lambda_q = ix->lambda_q;
    v->pair_id = ix->pair_id;
}

/* ---------------------------------------------------------------- PQTINDEX v1 */

typedef struct {
    const uint8_t* p;
    size_t left;
    int bad;
} reader;

static void rd(reader* r, void* dst, size_t bytes) {
    if (r->bad || bytes > r->left) { r->bad = 1; return; }
    memcpy(dst, r->p, bytes);
    r->p += bytes;
    r->left -= bytes;
}

/* load_index (src/index_io.cpp:148-229), with the config read as in read_config (:59-76). */
pqto_index* pqto_load(const char* path) {
    FILE* fp = fopen(path, "rb");
    if (!fp) { snprintf(g_err, sizeof g_err, "cannot open %s for reading", path); return NULL; }
    fseek(fp, 0, SEEK_END);
    long sz = ftell(fp);
    fseek(fp, 0, SEEK_SET);
    uint8_t* buf = (uint8_t*)malloc(sz > 0 ? (size_t)sz : 1);
    if (!buf || fread(buf, 1, (size_t)sz, fp) != (size_t)sz) {
        fclose(fp); free(buf);
        snprintf(g_err, sizeof g_err, "%s: read failed", path);
        return NULL;
    }
    fclose(fp);
    reader r = {buf, (size_t)sz, 0};
    pqto_index* ix = NULL;
    char magic[8];
    rd(&r, magic, 8);
    if (r.bad || memcmp(magic, "PQTINDEX", 8) != 0) {
        snprintf(g_err, sizeof g_err, "%s: bad index magic", path);
        goto fail;
    }
    uint32_t version = 0;
    rd(&r, &version, 4);
    if (r.bad) goto trunc;
    if (version != 1) {
        snprintf(g_err, sizeof g_err, "%s: unsupported index version %u, expected 1", path, version);
        goto fail;
    }
    ix = (pqto_index*)calloc(1, sizeof *ix);
    pqtg_config* c = &ix->cfg;
    uint8_t resort = 0;
    rd(&r, &c->dim, 4); rd(&r, &c->p_tree, 4); rd(&r, &c->k1, 4); rd(&r, &c->k2, 4);
    rd(&r, &c->w, 4); rd(&r, &c->p_line, 4); rd(&r, &c->hash_size, 8);
    rd(&r, &c->candidate_budget, 4); rd(&r, &c->rerank_exact, 4); rd(&r, &resort, 1);
    rd(&r, &c->train_iters, 4); rd(&r, &c->seed, 8);
    c->resort_bins = resort != 0;
    if (r.bad) goto trunc;
    if (validate_cfg(c) != 0) goto fail;
    rd(&r, &ix->n, 8);
    if (r.bad) goto trunc;
    uint32_t P = c->p_tree, k1 = c->k1, k2 = c->k2, m = c->dim / c->p_tree;
    ix->level1 = (float*)malloc((size_t)P * k1 * m * sizeof(float));
    ix->level2 = (float*)malloc((size_t)P * k1 * k2 * m * sizeof(float));
    for (uint32_t b = 0; b < P + P * k1; ++b) {
        uint32_t pd = 0, kk = 0;
        rd(&r, &pd, 4);
        rd(&r, &kk, 4);
        if (r.bad) goto trunc;
        int lvl1 = b < P;
        if (pd != m || kk != (lvl1 ? k1 : k2)) {
            snprintf(g_err, sizeof g_err, "%s: codebook shape does not match config", path);
            goto fail;
        }
        float* dst = lvl1 ? ix->level1 + (size_t)b * k1 * m : ix->level2 + (size_t)(b - P) * k2 * m;
        rd(&r, dst, (size_t)pd * kk * sizeof(float));
    }
    size_t nd2 = (size_t)c->p_line * k1 * k1;
    ix->d2 = (float*)malloc(nd2 * sizeof(float));
    rd(&r, ix->d2, nd2 * sizeof(float));
    rd(&r, &ix->table_count, 4);
    rd(&r, &ix->table_len, 4);
    if (r.bad) goto trunc;
    ix->slopes = (double*)malloc((size_t)ix->table_count * sizeof(double) + 8);
    ix->entries = (uint32_t*)malloc((size_t)ix->table_count * ix->table_len * 8 + 8);
    for (uint32_t t = 0; t < ix->table_count; ++t) {
        rd(&r, &ix->slopes[t], 8);
        rd(&r, ix->entries + (size_t)t * ix->table_len * 2, (size_t)ix->table_len * 8);
    }
    ix->offsets = (uint64_t*)malloc((size_t)(c->hash_size + 1) * 8);
    ix->ids = (uint32_t*)malloc((size_t)ix->n * 4 + 4);
    if (!ix->offsets || !ix->ids) { set_err("out of memory"); goto fail; }
    rd(&r, ix->offsets, (size_t)(c->hash_size + 1) * 8);
    rd(&r, ix->ids, (size_t)ix->n * 4);
    uint8_t pw = 0;
    rd(&r, &pw, 1);
    if (r.bad) goto trunc;
    if (pw != 1 && pw != 2) {
        snprintf(g_err, sizeof g_err, "%s: invalid line-code pair width %u", path, pw);
        goto fail;
    }
    size_t records = (size_t)ix->n * c->p_line;
    ix->lambda_q = (uint8_t*)malloc(records + 1);
    ix->pair_id = (uint16_t*)malloc(records * 2 + 2);
    if (!ix->lambda_q || !ix->pair_id) { set_err("out of memory"); goto fail; }
    if (r.left < records * (1 + (size_t)pw)) goto trunc;
    for (size_t i = 0; i < records; ++i) {
        ix->lambda_q[i] = r.p[0];
        if (pw == 1) {
            ix->pair_id[i] = r.p[1];
        } else {
            uint16_t v;
            memcpy(&v, r.p + 1, 2);
            ix->pair_id[i] = v;
        }
        r.p += 1 + pw;
    }
    r.left -= records * (1 + (size_t)pw);
    if (derive(ix) != 0) { set_err("out of memory"); goto fail; }
    free(buf);
    return ix;
trunc:
    snprintf(g_err, sizeof g_err, "%s: truncated index file", path);
fail:
    free(buf);
    pqto_free(ix);
    return NULL;
}

/* save_index (src/index_io.cpp:94-146) */
int pqto_save(const pqto_index* ix, const char* path) {
    FILE* fp = fopen(path, "wb");
    if (!fp) { snprintf(g_err, sizeof g_err, "cannot open %s for writing", path); return PQTG_ERR_FORMAT; }
    const pqtg_config* c = &ix->cfg;
    uint32_t version = 1;
    uint8_t resort = c->resort_bins ? 1 : 0;
    fwrite("PQTINDEX", 1, 8, fp);
    fwrite(&version, 4, 1, fp);
    fwrite(&c->dim, 4, 1, fp); fwrite(&c->p_tree, 4, 1, fp); fwrite(&c->k1, 4, 1, fp);
    fwrite(&c->k2, 4, 1, fp); fwrite(&c->w, 4, 1, fp); fwrite(&c->p_line, 4, 1, fp);
    fwrite(&c->hash_size, 8, 1, fp); fwrite(&c->candidate_budget, 4, 1, fp);
    fwrite(&c->rerank_exact, 4, 1, fp); fwrite(&resort, 1, 1, fp);
    fwrite(&c->train_iters, 4, 1, fp); fwrite(&c->seed, 8, 1, fp);
    fwrite(&ix->n, 8, 1, fp);
    uint32_t P = c->p_tree, k1 = c->k1, k2 = c->k2, m = ix->m;
    for (uint32_t p = 0; p < P; ++p) {
        fwrite(&m, 4, 1, fp); fwrite(&k1, 4, 1, fp);
        fwrite(ix->level1 + (size_t)p * k1 * m, 4, (size_t)k1 * m, fp);
    }
    for (uint32_t b = 0; b < P * k1; ++b) {
        fwrite(&m, 4, 1, fp); fwrite(&k2, 4, 1, fp);
        fwrite(ix->level2 + (size_t)b * k2 * m, 4, (size_t)k2 * m, fp);
    }
    fwrite(ix->d2, 4, (size_t)c->p_line * k1 * k1, fp);
    fwrite(&ix->table_count, 4, 1, fp);
    fwrite(&ix->table_len, 4, 1, fp);
    for (uint32_t t = 0; t < ix->table_count; ++t) {
        fwrite(&ix->slopes[t], 8, 1, fp);
        fwrite(ix->entries + (size_t)t * ix->table_len * 2, 8, ix->table_len, fp);
    }
    fwrite(ix->offsets, 8, (size_t)c->hash_size + 1, fp);
    fwrite(ix->ids, 4, ix->n, fp);
    uint8_t pw = ix->npairs <= 256 ? 1 : 2;
    fwrite(&pw, 1, 1, fp);
    size_t records = (size_t)ix->n * c->p_line;
    for (size_t i = 0; i < records; ++i) {
        fwrite(&ix->lambda_q[i], 1, 1, fp);
        if (pw == 1) {
            uint8_t v = (uint8_t)ix->pair_id[i];
            fwrite(&v, 1, 1, fp);
        } else {
            fwrite(&ix->pair_id[i], 2, 1, fp);
        }
    }
    int bad = ferror(fp);
    fclose(fp);
    if (bad) { snprintf(g_err, sizeof g_err, "write failed for %s", path); return PQTG_ERR_FORMAT; }
    return 0;
}

/* ---------------------------------------------------------------- traversal */

/* l2_sq (include/pqt/distance.hpp:11-18): sequential fp32 accumulation. */
static float l2_sq(const float* a, const float* b, size_t dim) {
    float acc = 0.0f;
    for (size_t i = 0; i < dim; ++i) {
        float d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

typedef struct { uint32_t id; float dist; } l1e;
typedef struct { uint32_t parent, child; float dist; } l2e;

static int cmp_l1(const void* x, const void* y) {
    const l1e* a = (const l1e*)x;
    const l1e* b = (const l1e*)y;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}

static int cmp_l2(const void* x, const void* y) {
    const l2e* a = (const l2e*)x;
    const l2e* b = (const l2e*)y;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    if (a->parent != b->parent) return a->parent < b->parent ? -1 : 1;
    return a->child < b->child ? -1 : (a->child > b->child);
}

/* traverse (src/pqtree.cpp:74-120). l1/l2 are caller buffers P×k1 / P×W. */
static void traverse_impl(const pqto_index* ix, const float* y, float* fine, l1e* l1, l2e* l2) {
    const pqtg_config* c = &ix->cfg;
    const uint32_t k1 = c->k1, k2 = c->k2, fd = ix->fd, m = ix->m, W = ix->W;
    for (uint32_t p = 0; p < c->p_tree; ++p) {
        l1e* L1 = l1 + (size_t)p * k1;
        for (uint32_t i = 0; i < k1; ++i) {
            float total = 0.0f;  /* pqtree.cpp:88-96: fine partials first, summed in f order */
            for (uint32_t f = p * ix->per_part; f < (p + 1) * ix->per_part; ++f) {
                float d = l2_sq(y + (size_t)f * fd, ix->fine + ((size_t)f * k1 + i) * fd, fd);
                fine[(size_t)f * k1 + i] = d;
                total += d;
            }
            L1[i].id = i;
            L1[i].dist = total;
        }
        qsort(L1, k1, sizeof(l1e), cmp_l1);  /* pqtree.cpp:98-100, (dist, id) */
        l2e* L2 = l2 + (size_t)p * W;
        const float* yp = y + (size_t)p * m;
        uint32_t q = 0;
        for (uint32_t r = 0; r < c->w; ++r) {  /* pqtree.cpp:105-111 */
            uint32_t parent = L1[r].id;
            const float* book = ix->level2 + ((size_t)p * k1 + parent) * k2 * m;
            for (uint32_t ch = 0; ch < k2; ++ch) {
                L2[q].parent = parent;
                L2[q].child = ch;
                L2[q].dist = l2_sq(yp, book + (size_t)ch * m, m);
                ++q;
            }
        }
        qsort(L2, W, sizeof(l2e), cmp_l2);  /* pqtree.cpp:112-117, (dist, parent, child) */
    }
}

int pqto_traverse(const pqto_index* ix, const float* y, float* fine, uint32_t* l1_id,
                  float* l1_dist, uint32_t* l2_parent, uint32_t* l2_child, float* l2_dist) {
    const pqtg_config* c = &ix->cfg;
    l1e* l1 = (l1e*)malloc(sizeof(l1e) * c->p_tree * c->k1);
    l2e* l2 = (l2e*)malloc(sizeof(l2e) * c->p_tree * ix->W + 1);
    if (!l1 || !l2) { free(l1); free(l2); set_err("out of memory"); return PQTG_ERR_OOM; }
    traverse_impl(ix, y, fine, l1, l2);
    for (uint32_t i = 0; i < c->p_tree * c->k1; ++i) {
        if (l1_id) l1_id[i] = l1[i].id;
        if (l1_dist) l1_dist[i] = l1[i].dist;
    }
    for (uint32_t i = 0; i < c->p_tree * ix->W; ++i) {
        if (l2_parent) l2_parent[i] = l2[i].parent;
        if (l2_child) l2_child[i] = l2[i].child;
        if (l2_dist) l2_dist[i] = l2[i].dist;
    }
    free(l1);
    free(l2);
    return 0;
}

/* ---------------------------------------------------------------- bin order */

/* pick_slope_table (src/binorder.cpp:52-65) */
uint32_t pqto_pick_slope_table(const float* a, uint64_t na, const float* b, uint64_t nb) {
    if (na < 2 || nb < 2) return 5;
    double gap_a = (double)a[1] - a[0];
    double gap_b = (double)b[1] - b[0];
    if (!(gap_a > 0.0) || !(gap_b > 0.0)) return 5;
    double ratio = gap_b / gap_a;
    long k = lround(log(ratio) / log(1.08));
    if (k < -5) k = -5;
    if (k > 4) k = 4;
    return (uint32_t)(k + 5);
}

/* PairCursor (src/binorder.cpp:69-110): table prefix filtered by bounds, then a row-major
 * sweep of every grid cell the table did not emit. */
typedef struct {
    const uint32_t* entries;
    uint64_t table_len;
    uint64_t len_a, len_b;
    uint64_t tpos, sa, sb;
    u64set emitted;
} pair_cursor;

static int pc_init(pair_cursor* pc, const uint32_t* entries, uint64_t table_len, uint64_t la,
                   uint64_t lb) {
    pc->entries = entries;
    pc->table_len = table_len;
    pc->len_a = la;
    pc->len_b = lb;
    pc->tpos = pc->sa = pc->sb = 0;
    return set_init(&pc->emitted, table_len + 1);
}

static int pc_next(pair_cursor* pc, uint32_t* ra, uint32_t* rb) {
    while (pc->tpos < pc->table_len) {
        uint32_t a = pc->entries[2 * pc->tpos], b = pc->entries[2 * pc->tpos + 1];
        pc->tpos++;
        if (a < pc->len_a && b < pc->len_b) {
            set_insert(&pc->emitted, ((uint64_t)a << 32) | b);
            *ra = a;
            *rb = b;
            return 1;
        }
    }
    while (pc->sa < pc->len_a) {
        while (pc->sb < pc->len_b) {
            uint64_t key = (pc->sa << 32) | pc->sb;
            uint32_t a = (uint32_t)pc->sa, b = (uint32_t)pc->sb;
            pc->sb++;
            if (!set_contains(&pc->emitted, key)) {
                *ra = a;
                *rb = b;
                return 1;
            }
        }
        pc->sb = 0;
        pc->sa++;
    }
    return 0;
}

/* BinStream (src/binorder.cpp:170-283): modes single / pair / quad. */
typedef struct {
    int mode;  /* 1 single, 2 pair, 4 quad */
    uint64_t pos, len;
    pair_cursor pa, pb, merge;
    pairvec sa, sb;
} bin_stream;

static int bs_init(bin_stream* s, const pqto_index* ix, const float* const* lists, uint32_t parts,
                   uint64_t len) {
    memset(s, 0, sizeof *s);
    const uint64_t tl = ix->table_len;
    if (parts == 1) {
        s->mode = 1;
        s->len = len;
        return 0;
    }
    if (parts == 2 && ix->table_count == 10) {
        s->mode = 2;
        uint32_t t = pqto_pick_slope_table(lists[0], len, lists[1], len);
        return pc_init(&s->pa, ix->entries + (size_t)t * tl * 2, tl, len, len);
    }
    if (parts == 4 && ix->table_count == 10) {
        s->mode = 4;
        uint32_t ta = pqto_pick_slope_table(lists[0], len, lists[1], len);
        uint32_t tb = pqto_pick_slope_table(lists[2], len, lists[3], len);
        if (pc_init(&s->pa, ix->entries + (size_t)ta * tl * 2, tl, len, len)) return -1;
        if (pc_init(&s->pb, ix->entries + (size_t)tb * tl * 2, tl, len, len)) return -1;
        /* merge over pair ranks with the slope-1 table (binorder.cpp:237-240) */
        return pc_init(&s->merge, ix->entries + (size_t)5 * tl * 2, tl, len * len, len * len);
    }
    set_err("exact (Dijkstra) bin order is not part of the restated path");
    return PQTG_ERR_UNSUPPORTED;
}

static void bs_free(bin_stream* s) {
    set_free(&s->pa.emitted);
    set_free(&s->pb.emitted);
    set_free(&s->merge.emitted);
    free(s->sa.a);
    free(s->sb.a);
}

static int extend(pair_cursor* pc, pairvec* v, uint64_t needed) {
    uint32_t a, b;
    while (v->size < needed) {
        if (!pc_next(pc, &a, &b)) return 0;
        if (pv_push(v, a, b)) return 0;
    }
    return 1;
}

static int bs_next(bin_stream* s, uint32_t* out) {
    switch (s->mode) {
    case 1:
        if (s->pos >= s->len) return 0;
        out[0] = (uint32_t)s->pos++;
        return 1;
    case 2:
        return pc_next(&s->pa, &out[0], &out[1]);
    case 4: {
        uint32_t u, v;
        if (!pc_next(&s->merge, &u, &v)) return 0;
        if (!extend(&s->pa, &s->sa, (uint64_t)u + 1) || !extend(&s->pb, &s->sb, (uint64_t)v + 1)) return 0;
        out[0] = s->sa.a[2 * (uint64_t)u];
        out[1] = s->sa.a[2 * (uint64_t)u + 1];
        out[2] = s->sb.a[2 * (uint64_t)v];
        out[3] = s->sb.a[2 * (uint64_t)v + 1];
        return 1;
    }
    }
    return 0;
}

int64_t pqto_heuristic_order(const pqto_index* ix, const float* lists, uint32_t parts,
                             uint32_t len, uint64_t max_bins, uint32_t* out) {
    const float* lp[8];
    if (parts == 0) return 0;
    if (parts > 8) { set_err("too many parts"); return PQTG_ERR_UNSUPPORTED; }
    for (uint32_t p = 0; p < parts; ++p) lp[p] = lists + (size_t)p * len;
    bin_stream s;
    int rc = bs_init(&s, ix, lp, parts, len);
    if (rc) { bs_free(&s); return rc < 0 ? rc : PQTG_ERR_OOM; }
    uint64_t n = 0;
    while (n < max_bins && bs_next(&s, out + n * parts)) ++n;
    bs_free(&s);
    return (int64_t)n;
}

/* global_code / encode_slot (src/pqtree.cpp:12-25): base-(k1·k2) positional code, u64 wrap. */
uint64_t pqto_encode_slot(const uint32_t* pc, uint32_t parts, uint32_t k1, uint32_t k2,
                          uint64_t hash_size) {
    const uint64_t base = (uint64_t)k1 * k2;
    uint64_t acc = 0, mult = 1;
    for (uint32_t p = 0; p < parts; ++p) {
        acc += ((uint64_t)pc[2 * p] * k2 + pc[2 * p + 1]) * mult;
        mult *= base;
    }
    return acc % hash_size;
}

/* line_distance (src/linequant.cpp:169-182) with line_part_distance (linequant.hpp:83-85). */
float pqto_line_distance(const pqto_index* ix, const uint8_t* lq, const uint16_t* pid,
                         const float* fine) {
    const uint32_t k1 = ix->cfg.k1;
    float total = 0.0f;
    for (uint32_t f = 0; f < ix->cfg.p_line; ++f) {
        const uint16_t* pr = ix->pairs + 2 * (size_t)pid[f];
        float lambda = (float)lq[f] * (1.0f / 255.0f);
        float b2 = fine[f * k1 + pr[0]];
        float a2 = fine[f * k1 + pr[1]];
        float c2 = ix->d2[((size_t)f * k1 + pr[0]) * k1 + pr[1]];
        total += b2 + lambda * lambda * c2 + lambda * (a2 - b2 - c2);
    }
    return total;
}

/* ---------------------------------------------------------------- gather */

typedef struct { float agg; uint32_t idx; } aggi;

static int cmp_aggi(const void* x, const void* y) {
    const aggi* a = (const aggi*)x;
    const aggi* b = (const aggi*)y;
    if (a->agg != b->agg) return a->agg < b->agg ? -1 : 1;  /* stable_sort by agg ... */
    return a->idx < b->idx ? -1 : (a->idx > b->idx);       /* ... == sort by (agg, position) */
}

/* knn_query steps 2-3 (src/search.cpp:139-217). Returns C, or negative status. */
static int64_t gather(const pqto_index* ix, const l2e* l2, uint32_t* positions, uint64_t cap,
                      uint64_t* bins_out) {
    const pqtg_config* c = &ix->cfg;
    const uint32_t parts = c->p_tree, W = ix->W;
    const uint64_t H = c->hash_size;
    uint64_t budget = c->candidate_budget < ix->n ? c->candidate_budget : ix->n;
    if (budget > cap) budget = cap;
    const uint64_t batch_tuples = c->resort_bins ? (budget > 1 ? budget : 1) : 1024;
    float* lists = (float*)malloc(sizeof(float) * parts * W + 4);
    const float* lp[8];
    for (uint32_t p = 0; p < parts; ++p) {
        for (uint32_t r = 0; r < W; ++r) lists[p * W + r] = l2[p * W + r].dist;
        lp[p] = lists + (size_t)p * W;
    }
    bin_stream s;
    int rc = bs_init(&s, ix, lp, parts, W);
    if (rc) { bs_free(&s); free(lists); return rc < 0 ? rc : PQTG_ERR_OOM; }
    uint32_t* batch = (uint32_t*)malloc(sizeof(uint32_t) * parts * batch_tuples);
    aggi* order = (aggi*)malloc(sizeof(aggi) * batch_tuples);
    u64set seen;
    set_init(&seen, 1024);
    uint64_t C = 0, bins = 0;
    int done = 0;
    while (!done && C < budget) {
        uint64_t count = 0;
        while (count < batch_tuples) {
            if (!bs_next(&s, batch + count * parts)) { done = 1; break; }
            ++count;
        }
        for (uint64_t b = 0; b < count; ++b) {
            order[b].idx = (uint32_t)b;
            order[b].agg = 0.0f;
            if (c->resort_bins) {  /* search.cpp:179-190: fp32 sum in part order from 0.0f */
                float sum = 0.0f;
                for (uint32_t p = 0; p < parts; ++p) sum += lists[p * W + batch[b * parts + p]];
                order[b].agg = sum;
            }
        }
        if (c->resort_bins) qsort(order, count, sizeof(aggi), cmp_aggi);
        for (uint64_t oi = 0; oi < count; ++oi) {
            uint32_t b = order[oi].idx;
            uint32_t code[16];
            for (uint32_t p = 0; p < parts; ++p) {
                const l2e* e = &l2[p * W + batch[b * parts + p]];
                code[2 * p] = e->parent;
                code[2 * p + 1] = e->child;
            }
            uint64_t slot = pqto_encode_slot(code, parts, c->k1, c->k2, H);
            if (set_insert(&seen, slot) != 1) continue;        /* search.cpp:200-202 */
            uint64_t lo = ix->offsets[slot], hi = ix->offsets[slot + 1];
            if (lo == hi) continue;                              /* :203-207 */
            ++bins;                                              /* :208 */
            for (uint64_t i = lo; i < hi && C < budget; ++i) positions[C++] = (uint32_t)i;
            if (C >= budget) break;
        }
    }
    set_free(&seen);
    bs_free(&s);
    free(batch);
    free(order);
    free(lists);
    if (bins_out) *bins_out = bins;
    return (int64_t)C;
}

int64_t pqto_candidates(const pqto_index* ix, const float* y, uint32_t* positions, uint64_t cap,
                        uint64_t* bins_visited) {
    const pqtg_config* c = &ix->cfg;
    if (bins_visited) *bins_visited = 0;
    if (ix->n == 0) return 0;
    float* fine = (float*)malloc(sizeof(float) * c->p_line * c->k1);
    l1e* l1 = (l1e*)malloc(sizeof(l1e) * c->p_tree * c->k1);
    l2e* l2 = (l2e*)malloc(sizeof(l2e) * c->p_tree * ix->W + 1);
    traverse_impl(ix, y, fine, l1, l2);
    int64_t C = gather(ix, l2, positions, cap, bins_visited);
    free(fine);
    free(l1);
    free(l2);
    return C;
}

/* ---------------------------------------------------------------- knn */

typedef struct { float dist; uint32_t id; } cand;

static int cmp_cand(const void* x, const void* y) {  /* candidate_less, search.cpp:39-41 */
    const cand* a = (const cand*)x;
    const cand* b = (const cand*)y;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}

/* knn_query (src/search.cpp:126-260). The exact re-rank (:229-249) runs when raw vectors
 * are attached (pqto_attach_database) and rerank_exact > 0, on unsharded searches only. */
static int knn_one(const pqto_index* ix, const float* y, uint32_t k, uint64_t lo, uint64_t hi,
                   uint32_t* ids, float* dists, uint32_t* count, uint64_t* stats) {
    const pqtg_config* c = &ix->cfg;
    *count = 0;
    if (stats) stats[0] = stats[1] = stats[2] = 0;
    if (k == 0 || ix->n == 0) return 0;  /* search.cpp:130-132 */
    uint64_t budget = c->candidate_budget < ix->n ? c->candidate_budget : ix->n;
    float* fine = (float*)malloc(sizeof(float) * c->p_line * c->k1);
    l1e* l1 = (l1e*)malloc(sizeof(l1e) * c->p_tree * c->k1);
    l2e* l2 = (l2e*)malloc(sizeof(l2e) * c->p_tree * ix->W + 1);
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * (budget + 1));
    cand* ranked = (cand*)malloc(sizeof(cand) * (budget + 1));
    traverse_impl(ix, y, fine, l1, l2);
    uint64_t bins = 0;
    int64_t C = gather(ix, l2, pos, budget, &bins);
    if (C < 0) {
        free(fine); free(l1); free(l2); free(pos); free(ranked);
        return (int)C;
    }
    uint64_t nr = 0;
    if (ix->is_shard) {  /* a shard holds (and re-ranks) only its own positions */
        lo = ix->shard_lo;
        hi = ix->shard_hi;
    }
    for (int64_t i = 0; i < C; ++i) {  /* search.cpp:221-227 */
        uint64_t p = pos[i];
        if ((hi > lo || ix->is_shard) && (p < lo || p >= hi)) continue;
        uint32_t id;
        size_t row;
        if (ix->is_shard) {  /* codes by position */
            id = ix->ids[p - lo];
            row = (size_t)(p - lo);
        } else {
            id = ix->ids[p];
            row = id;
        }
        ranked[nr].id = id;
        ranked[nr].dist = pqto_line_distance(ix, ix->lambda_q + row * c->p_line,
                                             ix->pair_id + row * c->p_line, fine);
        ++nr;
    }
    /* rerank = min(max(rerank_exact, k), C) with raw vectors attached (search.cpp:229-238) */
    uint64_t rerank = 0;
    if (c->rerank_exact > 0 && ix->db && !(hi > lo) && !ix->is_shard) {
        uint64_t r = c->rerank_exact > k ? c->rerank_exact : k;
        rerank = r < nr ? r : nr;
    }
    qsort(ranked, nr, sizeof(cand), cmp_cand);  /* partial_sort prefix == full sort prefix */
    if (rerank > 0) {  /* search.cpp:242-249: exact l2_sq(db.row(id), y), then re-sort */
        for (uint64_t i = 0; i < rerank; ++i)
            ranked[i].dist = l2_sq(ix->db + (size_t)ranked[i].id * c->dim, y, c->dim);
        qsort(ranked, rerank, sizeof(cand), cmp_cand);
    }
    uint64_t out = k < nr ? k : nr;
    for (uint64_t i = 0; i < out; ++i) {
        ids[i] = ranked[i].id;
        dists[i] = ranked[i].dist;
    }
    *count = (uint32_t)out;
    if (stats) {
        stats[0] = bins;
        stats[1] = (uint64_t)C;
        stats[2] = rerank;
    }
    free(fine); free(l1); free(l2); free(pos); free(ranked);
    return 0;
}

void pqto_attach_database(pqto_index* ix, const float* rows) { ix->db = rows; }

typedef struct {
    const pqto_index* ix;
    const float* q;
    uint32_t k;
    uint64_t lo, hi, begin, end;
    uint32_t* ids;
    float* dists;
    uint32_t* counts;
    uint64_t* stats;
    int rc;
} job;

static void* run_job(void* arg) {
    job* j = (job*)arg;
    const uint32_t D = j->ix->cfg.dim;
    for (uint64_t q = j->begin; q < j->end && j->rc == 0; ++q) {
        j->rc = knn_one(j->ix, j->q + q * D, j->k, j->lo, j->hi, j->ids + q * j->k,
                        j->dists + q * j->k, j->counts + q, j->stats ? j->stats + q * 3 : NULL);
    }
    return NULL;
}

/* knn_query_batch (src/search.cpp:262-274) with parallel_for's contiguous chunking
 * (include/pqt/parallel.hpp:21-46). */
int pqto_knn_batch(const pqto_index* ix, const float* queries, uint64_t nq, uint32_t dim,
                   uint32_t k, int threads, uint64_t lo, uint64_t hi, uint32_t* ids,
                   float* dists, uint32_t* counts, uint64_t* stats) {
    if (nq > 0 && dim != ix->cfg.dim) {
        set_err("knn_query_batch: query dimension mismatch");
        return PQTG_ERR_BAD_DIM;
    }
    if (ix->cfg.p_tree != 1 && !((ix->cfg.p_tree == 2 || ix->cfg.p_tree == 4) && ix->table_count == 10)) {
        set_err("exact (Dijkstra) bin order is not part of the restated path");
        return PQTG_ERR_UNSUPPORTED;
    }
    if (nq == 0) return 0;
    if (threads <= 0) {
        long hw = sysconf(_SC_NPROCESSORS_ONLN);
        threads = hw > 0 ? (int)hw : 1;
    }
    uint64_t workers = (uint64_t)threads < nq ? (uint64_t)threads : nq;
    uint64_t chunk = (nq + workers - 1) / workers;
    job* jobs = (job*)calloc(workers, sizeof(job));
    pthread_t* th = (pthread_t*)calloc(workers, sizeof(pthread_t));
    uint64_t used = 0;
    for (uint64_t w = 0; w < workers; ++w) {
        uint64_t b = w * chunk, e = b + chunk < nq ? b + chunk : nq;
        if (b >= e) break;
        jobs[w] = (job){ix, queries, k, lo, hi, b, e, ids, dists, counts, stats, 0};
        if (workers == 1) {
            run_job(&jobs[w]);
        } else {
            pthread_create(&th[w], NULL, run_job, &jobs[w]);
        }
        ++used;
    }
    int rc = 0;
    for (uint64_t w = 0; w < used; ++w) {
        if (workers > 1) pthread_join(th[w], NULL);
        if (jobs[w].rc) rc = jobs[w].rc;
    }
    free(jobs);
    free(th);
    return rc;
}
