// BLAKE3 from the published spec; tree hashing parallelised over 1 MiB
// subtrees. See blake3.hpp.
#include "blake3.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>

namespace dimg::b3 {
namespace {

constexpr uint32_t kIV[8] = {0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au,
                             0x510E527Fu, 0x9B05688Cu, 0x1F83D9ABu, 0x5BE0CD19u};
constexpr uint32_t CHUNK_START = 1, CHUNK_END = 2, PARENT = 4, ROOT = 8;
constexpr size_t kChunk = 1024;
constexpr size_t kSubtreeChunks = 1024;  // 1 MiB parallel work unit (power of two)

using CV = std::array<uint32_t, 8>;

inline uint32_t rr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

#define B3G(a, b, c, d, x, y)            \
    a = a + b + (x); d = rr(d ^ a, 16);  \
    c = c + d;       b = rr(b ^ c, 12);  \
    a = a + b + (y); d = rr(d ^ a, 8);   \
    c = c + d;       b = rr(b ^ c, 7);

// Message schedule: index of the word used at position i in round r
// (the spec's permutation applied r times, precomputed).
struct Schedule {
    uint8_t s[7][16];
    constexpr Schedule() : s{} {
        const uint8_t perm[16] = {2, 6, 3, 10, 7, 0, 4, 13, 1, 11, 12, 5, 9, 14, 15, 8};
        for (int i = 0; i < 16; ++i) s[0][i] = uint8_t(i);
        for (int r = 1; r < 7; ++r)
            for (int i = 0; i < 16; ++i) s[r][i] = s[r - 1][perm[i]];
    }
};
constexpr Schedule kSched;

void compress(const uint32_t* cv, const uint32_t* m, uint64_t ctr, uint32_t len, uint32_t flags,
              uint32_t* out16) {
    uint32_t v0 = cv[0], v1 = cv[1], v2 = cv[2], v3 = cv[3], v4 = cv[4], v5 = cv[5], v6 = cv[6],
             v7 = cv[7], v8 = kIV[0], v9 = kIV[1], v10 = kIV[2], v11 = kIV[3],
             v12 = uint32_t(ctr), v13 = uint32_t(ctr >> 32), v14 = len, v15 = flags;
    for (int r = 0; r < 7; ++r) {
        const uint8_t* s = kSched.s[r];
        B3G(v0, v4, v8, v12, m[s[0]], m[s[1]]);
        B3G(v1, v5, v9, v13, m[s[2]], m[s[3]]);
        B3G(v2, v6, v10, v14, m[s[4]], m[s[5]]);
        B3G(v3, v7, v11, v15, m[s[6]], m[s[7]]);
        B3G(v0, v5, v10, v15, m[s[8]], m[s[9]]);
        B3G(v1, v6, v11, v12, m[s[10]], m[s[11]]);
        B3G(v2, v7, v8, v13, m[s[12]], m[s[13]]);
        B3G(v3, v4, v9, v14, m[s[14]], m[s[15]]);
    }
    out16[0] = v0 ^ v8;   out16[1] = v1 ^ v9;   out16[2] = v2 ^ v10;  out16[3] = v3 ^ v11;
    out16[4] = v4 ^ v12;  out16[5] = v5 ^ v13;  out16[6] = v6 ^ v14;  out16[7] = v7 ^ v15;
    out16[8] = v8 ^ cv[0];   out16[9] = v9 ^ cv[1];   out16[10] = v10 ^ cv[2];
    out16[11] = v11 ^ cv[3]; out16[12] = v12 ^ cv[4]; out16[13] = v13 ^ cv[5];
    out16[14] = v14 ^ cv[6]; out16[15] = v15 ^ cv[7];
}

inline void load_block(const uint8_t* p, size_t n, uint32_t* m) {
    uint8_t tmp[64];
    if (n < 64) {
        std::memset(tmp, 0, 64);
        std::memcpy(tmp, p, n);
        p = tmp;
    }
    for (int i = 0; i < 16; ++i)
        m[i] = uint32_t(p[4 * i]) | uint32_t(p[4 * i + 1]) << 8 | uint32_t(p[4 * i + 2]) << 16 |
               uint32_t(p[4 * i + 3]) << 24;
}

// A node that can yield either its chaining value or the root output.
struct Node {
    CV cv;
    uint32_t m[16];
    uint64_t ctr;
    uint32_t len, flags;

    CV chain() const {
        uint32_t o[16];
        compress(cv.data(), m, ctr, len, flags, o);
        CV r;
        std::copy(o, o + 8, r.begin());
        return r;
    }
    Digest root() const {
        uint32_t o[16];
        compress(cv.data(), m, 0, len, flags | ROOT, o);
        Digest d;
        for (int i = 0; i < 8; ++i)
            for (int b = 0; b < 4; ++b) d[4 * i + b] = uint8_t(o[i] >> (8 * b));
        return d;
    }
};

Node parent(const CV& l, const CV& r) {
    Node n;
    std::copy(kIV, kIV + 8, n.cv.begin());
    std::copy(l.begin(), l.end(), n.m);
    std::copy(r.begin(), r.end(), n.m + 8);
    n.ctr = 0;
    n.len = 64;
    n.flags = PARENT;
    return n;
}

// Chunk (<= 1024 bytes) -> its final node (CHUNK_END block not yet compressed).
Node chunk_node(const uint8_t* p, size_t len, uint64_t index) {
    CV cv;
    std::copy(kIV, kIV + 8, cv.begin());
    size_t nblocks = len == 0 ? 1 : (len + 63) / 64;
    uint32_t m[16], o[16];
    for (size_t b = 0; b + 1 < nblocks; ++b) {
        load_block(p + 64 * b, 64, m);
        compress(cv.data(), m, index, 64, b == 0 ? CHUNK_START : 0, o);
        std::copy(o, o + 8, cv.begin());
    }
    Node n;
    n.cv = cv;
    size_t last = len - 64 * (nblocks - 1);
    load_block(p + 64 * (nblocks - 1), last, n.m);
    n.ctr = index;
    n.len = uint32_t(last);
    n.flags = CHUNK_END | (nblocks == 1 ? CHUNK_START : 0);
    return n;
}

// CV of a complete subtree of n (power of two) full chunks starting at chunk `base`.
CV subtree_cv(const uint8_t* p, uint64_t base, size_t n) {
    if (n == 1) return chunk_node(p, kChunk, base).chain();
    CV l = subtree_cv(p, base, n / 2);
    CV r = subtree_cv(p + (n / 2) * kChunk, base + n / 2, n / 2);
    return parent(l, r).chain();
}

void push_cv(std::vector<CV>& stack, CV cv, uint64_t total_units) {
    while ((total_units & 1) == 0) {
        cv = parent(stack.back(), cv).chain();
        stack.pop_back();
        total_units >>= 1;
    }
    stack.push_back(cv);
}

}  // namespace

Digest hash(const void* data, size_t len, int threads) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    const size_t unit = kSubtreeChunks * kChunk;
    // Parallel prefix: full 1 MiB subtrees, leaving >= 1 byte for the tail so
    // the root is always formed by the serial finalisation below.
    size_t n_units = len == 0 ? 0 : (len - 1) / unit;
    std::vector<CV> unit_cv(n_units);
    if (n_units) {
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        unsigned nt = threads > 0 ? unsigned(threads) : hw;
        nt = std::min<unsigned>(nt, unsigned(n_units));
        std::atomic<size_t> next{0};
        auto work = [&] {
            for (size_t i; (i = next.fetch_add(1)) < n_units;)
                unit_cv[i] = subtree_cv(p + i * unit, uint64_t(i) * kSubtreeChunks, kSubtreeChunks);
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    }
    std::vector<CV> stack;
    for (size_t i = 0; i < n_units; ++i) push_cv(stack, unit_cv[i], i + 1);
    // Tail: whole chunks while more input follows, then the final chunk.
    size_t off = n_units * unit;
    uint64_t chunk = uint64_t(n_units) * kSubtreeChunks;
    while (len - off > kChunk) {
        push_cv(stack, chunk_node(p + off, kChunk, chunk).chain(), chunk + 1);
        off += kChunk;
        ++chunk;
    }
    Node node = chunk_node(p + off, len - off, chunk);
    for (size_t i = stack.size(); i-- > 0;) node = parent(stack[i], node.chain());
    return node.root();
}

Hasher::Hasher() = default;
void Hasher::update(const void* data, size_t len) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    buf_.insert(buf_.end(), p, p + len);
}
Digest Hasher::finalize() const { return hash(buf_.data(), buf_.size(), 1); }

}  // namespace dimg::b3
