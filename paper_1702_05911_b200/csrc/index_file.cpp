// index_file.cpp — PQTINDEX v1 reader (the reference's container, src/index_io.cpp:94-229),
// mmap-based. Fields are packed little-endian and every array starts at an unaligned offset
// (the fixed header is 73 bytes), so arrays are memcpy'd out of the mapping; the line-code
// records stay in the mapping and are permuted straight into device layout.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>

#include "pqtg_internal.h"

namespace pqtg {

MappedFile::~MappedFile() {
    if (base) munmap(const_cast<uint8_t*>(base), size);
    if (fd >= 0) close(fd);
}

namespace {
struct Cursor {
    const uint8_t* p;
    size_t left;
    std::string path;
    const uint8_t* take(size_t n) {
        if (n > left) throw Error{PQTG_ERR_FORMAT, path + ": truncated index file"};
        const uint8_t* r = p;
        p += n;
        left -= n;
        return r;
    }
    template <class T>
    T pod() {
        T v;
        std::memcpy(&v, take(sizeof(T)), sizeof(T));
        return v;
    }
    template <class T>
    void vec(std::vector<T>& v, size_t count) {
        v.resize(count);
        if (count) std::memcpy(v.data(), take(count * sizeof(T)), count * sizeof(T));
    }
};

}  // namespace

void parse_index(const char* path, LoadedFile& lf) {
    lf.map.fd = open(path, O_RDONLY);
    if (lf.map.fd < 0) throw Error{PQTG_ERR_FORMAT, std::string("cannot open ") + path + " for reading"};
    struct stat st {};
    fstat(lf.map.fd, &st);
    lf.map.size = (size_t)st.st_size;
    if (lf.map.size > 0) {
        void* m = mmap(nullptr, lf.map.size, PROT_READ, MAP_PRIVATE, lf.map.fd, 0);
        if (m == MAP_FAILED) throw Error{PQTG_ERR_FORMAT, std::string("mmap failed for ") + path};
        lf.map.base = static_cast<const uint8_t*>(m);
        madvise(m, lf.map.size, MADV_SEQUENTIAL);
    }
    Cursor cur{lf.map.base, lf.map.size, path};
    const uint8_t* magic = lf.map.size >= 8 ? cur.take(8) : nullptr;
    if (!magic || std::memcmp(magic, "PQTINDEX", 8) != 0)
        throw Error{PQTG_ERR_FORMAT, std::string(path) + ": bad index magic, expected \"PQTINDEX\""};
    const uint32_t version = cur.pod<uint32_t>();
    if (version != 1)
        throw Error{PQTG_ERR_FORMAT, std::string(path) + ": unsupported index version " + std::to_string(version) +
                                         ", expected 1"};
    Source& s = lf.src;
    pqtg_config& c = s.cfg;
    c.dim = cur.pod<uint32_t>();
    c.p_tree = cur.pod<uint32_t>();
    c.k1 = cur.pod<uint32_t>();
    c.k2 = cur.pod<uint32_t>();
    c.w = cur.pod<uint32_t>();
    c.p_line = cur.pod<uint32_t>();
    c.hash_size = cur.pod<uint64_t>();
    c.candidate_budget = cur.pod<uint32_t>();
    c.rerank_exact = cur.pod<uint32_t>();
    c.resort_bins = cur.pod<uint8_t>() ? 1u : 0u;
    c.train_iters = cur.pod<uint32_t>();
    c.seed = cur.pod<uint64_t>();
    validate_config(c);
    s.n = cur.pod<uint64_t>();
    const uint32_t P = c.p_tree, k1 = c.k1, k2 = c.k2, m = c.dim / P;
    lf.level1.resize((size_t)P * k1 * m);
    lf.level2.resize((size_t)P * k1 * k2 * m);
    for (uint32_t b = 0; b < P + P * k1; ++b) {
        const uint32_t pd = cur.pod<uint32_t>(), kk = cur.pod<uint32_t>();
        const bool lvl1 = b < P;
        if (pd != m || kk != (lvl1 ? k1 : k2))
            throw Error{PQTG_ERR_FORMAT, std::string(path) + ": codebook shape does not match config"};
        float* dst = lvl1 ? lf.level1.data() + (size_t)b * k1 * m : lf.level2.data() + (size_t)(b - P) * k2 * m;
        std::memcpy(dst, cur.take((size_t)pd * kk * 4), (size_t)pd * kk * 4);
    }
    cur.vec(lf.d2, (size_t)c.p_line * k1 * k1);
    const uint32_t tc = cur.pod<uint32_t>(), tl = cur.pod<uint32_t>();
    lf.slopes.resize(tc);
    lf.entries.resize((size_t)tc * tl * 2);
    for (uint32_t t = 0; t < tc; ++t) {
        lf.slopes[t] = cur.pod<double>();
        if (tl) std::memcpy(lf.entries.data() + (size_t)t * tl * 2, cur.take((size_t)tl * 8), (size_t)tl * 8);
    }
    cur.vec(lf.offsets, c.hash_size + 1);
    cur.vec(lf.ids, s.n);
    const uint8_t pw = cur.pod<uint8_t>();
    if (pw != 1 && pw != 2)
        throw Error{PQTG_ERR_FORMAT, std::string(path) + ": invalid line-code pair width " + std::to_string(pw)};
    s.records = cur.take((size_t)s.n * c.p_line * (1 + pw));
    s.record_pw = pw;
    s.level1 = lf.level1.data();
    s.level2 = lf.level2.data();
    s.d2 = lf.d2.data();
    s.table_count = tc;
    s.table_len = tl;
    s.slopes = lf.slopes.data();
    s.entries = lf.entries.data();
    s.offsets = lf.offsets.data();
    s.ids = lf.ids.data();
}


}  // namespace pqtg
