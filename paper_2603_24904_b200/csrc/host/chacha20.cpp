#include "chacha20.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "blake3.hpp"

namespace dimg::chacha {
namespace {

inline uint32_t rl(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
#define CQR(a, b, c, d)                          \
    a += b; d ^= a; d = rl(d, 16);               \
    c += d; b ^= c; b = rl(b, 12);               \
    a += b; d ^= a; d = rl(d, 8);                \
    c += d; b ^= c; b = rl(b, 7);

constexpr size_t kSegBlocks = 16384;          // 1 MiB of keystream per segment
constexpr size_t kSegBytes = kSegBlocks * 64;

unsigned pick_threads(int threads) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return threads > 0 ? unsigned(threads) : hw;
}

template <class F>
void parallel_for(size_t n, unsigned nt, F&& f) {
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < std::min<size_t>(nt, n); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
}

}  // namespace

void block(const Key& key, uint32_t counter, uint8_t out[64]) {
    const uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                             key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                             counter, 0, 0, 0};
    uint32_t x[16];
    std::memcpy(x, in, sizeof x);
    for (int i = 0; i < 10; ++i) {
        CQR(x[0], x[4], x[8], x[12]);
        CQR(x[1], x[5], x[9], x[13]);
        CQR(x[2], x[6], x[10], x[14]);
        CQR(x[3], x[7], x[11], x[15]);
        CQR(x[0], x[5], x[10], x[15]);
        CQR(x[1], x[6], x[11], x[12]);
        CQR(x[2], x[7], x[8], x[13]);
        CQR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; ++i) {
        uint32_t w = x[i] + in[i];
        std::memcpy(out + 4 * i, &w, 4);  // little-endian host
    }
}

Key key_from_seed(uint64_t seed) {
    uint8_t le[8];
    for (int i = 0; i < 8; ++i) le[i] = uint8_t(seed >> (8 * i));
    b3::Digest d = b3::hash(le, 8, 1);
    Key k;
    for (int i = 0; i < 8; ++i)
        k[i] = uint32_t(d[4 * i]) | uint32_t(d[4 * i + 1]) << 8 | uint32_t(d[4 * i + 2]) << 16 |
               uint32_t(d[4 * i + 3]) << 24;
    return k;
}

uint8_t Stream::u8() {
    if (pos_ == 64) {
        block(key_, ctr_++, buf_);
        pos_ = 0;
    }
    return buf_[pos_++];
}

uint32_t Stream::u32() {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= uint32_t(u8()) << (8 * i);
    return v;
}

void weight_stream(uint64_t seed, const Span* spans, size_t n_spans, int threads) {
    std::vector<uint64_t> span_end(n_spans);
    uint64_t n = 0;
    for (size_t i = 0; i < n_spans; ++i) span_end[i] = (n += spans[i].len);
    if (n == 0) return;
    const Key key = key_from_seed(seed);
    const unsigned nt = pick_threads(threads);
    // Pass 1: accepted-byte count of each 1 MiB keystream segment, in waves
    // until the running total covers n.
    std::vector<uint64_t> accepted;
    uint64_t total = 0;
    size_t nseg = 0;
    while (total < n) {
        size_t want = size_t((n - total) / (kSegBytes - kSegBytes / 128)) + 1;
        want = std::max<size_t>(want, nt);
        accepted.resize(nseg + want);
        parallel_for(want, nt, [&](size_t i) {
            uint8_t buf[64];
            uint64_t cnt = 0;
            uint32_t base = uint32_t((nseg + i) * kSegBlocks);
            for (size_t b = 0; b < kSegBlocks; ++b) {
                block(key, base + uint32_t(b), buf);
                for (int j = 0; j < 64; ++j) cnt += buf[j] != 255;
            }
            accepted[nseg + i] = cnt;
        });
        for (size_t i = nseg; i < nseg + want; ++i) total += accepted[i];
        nseg += want;
    }
    // Exclusive prefix sum = output index of each segment's first accepted byte.
    std::vector<uint64_t> offset(nseg + 1, 0);
    for (size_t i = 0; i < nseg; ++i) offset[i + 1] = offset[i] + accepted[i];
    size_t used = 0;
    while (used < nseg && offset[used] < n) ++used;
    // Pass 2: regenerate and compact into the spans.
    parallel_for(used, nt, [&](size_t i) {
        uint8_t buf[64];
        uint64_t o = offset[i];
        size_t sp = size_t(std::upper_bound(span_end.begin(), span_end.end(), o) - span_end.begin());
        uint64_t sp_begin = span_end[sp] - spans[sp].len;
        int8_t* dst = spans[sp].dst + (o - sp_begin);
        int8_t* dst_end = spans[sp].dst + spans[sp].len;
        uint32_t base = uint32_t(i * kSegBlocks);
        for (size_t b = 0; b < kSegBlocks && o < n; ++b) {
            block(key, base + uint32_t(b), buf);
            for (int j = 0; j < 64 && o < n; ++j) {
                if (buf[j] == 255) continue;
                while (dst == dst_end) {  // next non-empty span
                    ++sp;
                    dst = spans[sp].dst;
                    dst_end = dst + spans[sp].len;
                }
                *dst++ = int8_t(int(buf[j]) - 127);
                ++o;
            }
        }
    });
}

}  // namespace dimg::chacha
