// Toy-model weight synthesis on the GPU: the weight stream
// of gen_toy_model (proj/src/model.cpp:189-215 with ChaCha20Rng,
// proj/src/chacha20.cpp:48-96): the ChaCha20 keystream (RFC 8439 block,
// key = BLAKE3(seed as u64 LE), nonce 0, block counter from 0), every byte
// that is not 0xFF mapped to int8(b - 127), in stream order, n of them.
//
// Three launches over 64-byte keystream blocks, one block per thread:
//   cc_count_kernel    accepted bytes per block (u8) and per CTA (u64)
//   cc_scan_kernel     exclusive scan of the CTA totals (one CTA)
//   cc_compact_kernel  block-local exclusive scan in shared memory + the
//                      CTA offset, the block regenerated, its accepted
//                      bytes written at their global index (< n)
// About 50 integer ops per byte of keystream, run twice: a few ms at 7B.
#pragma once

#include <cstdint>

namespace dimg::dev {

constexpr int CC_THREADS = 1024;

__device__ __forceinline__ uint32_t cc_rotl(uint32_t x, int n) { return __funnelshift_l(x, x, n); }

__device__ __forceinline__ void cc_qr(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    a += b; d = cc_rotl(d ^ a, 16);
    c += d; b = cc_rotl(b ^ c, 12);
    a += b; d = cc_rotl(d ^ a, 8);
    c += d; b = cc_rotl(b ^ c, 7);
}

struct CcKey {
    uint32_t k[8];
};

// RFC 8439 block function, nonce 0: 16 output words (little-endian bytes)
__device__ __forceinline__ void cc_block(const CcKey& key, uint32_t counter, uint32_t (&out)[16]) {
    const uint32_t init[16] = {0x61707865u, 0x3320646Eu, 0x79622D32u, 0x6B206574u, key.k[0], key.k[1],
                               key.k[2],    key.k[3],    key.k[4],    key.k[5],    key.k[6], key.k[7],
                               counter,     0u,          0u,          0u};
    uint32_t s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = init[i];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        cc_qr(s[0], s[4], s[8], s[12]);
        cc_qr(s[1], s[5], s[9], s[13]);
        cc_qr(s[2], s[6], s[10], s[14]);
        cc_qr(s[3], s[7], s[11], s[15]);
        cc_qr(s[0], s[5], s[10], s[15]);
        cc_qr(s[1], s[6], s[11], s[12]);
        cc_qr(s[2], s[7], s[8], s[13]);
        cc_qr(s[3], s[4], s[9], s[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = s[i] + init[i];
}

// bytes of w that are not 0xFF (per-byte compare: exact, unlike the
// borrow-propagating zero-byte trick)
__device__ __forceinline__ uint32_t cc_accepted(uint32_t w) { return 4 - __popc(__vcmpeq4(w, 0xFFFFFFFFu)) / 8; }

__global__ void __launch_bounds__(CC_THREADS) cc_count_kernel(CcKey key, uint64_t n_blocks, uint8_t* cnt,
                                                               uint64_t* cta_tot) {
    __shared__ uint32_t red[32];
    const uint64_t b = uint64_t(blockIdx.x) * CC_THREADS + threadIdx.x;
    uint32_t c = 0;
    if (b < n_blocks) {
        uint32_t w[16];
        cc_block(key, uint32_t(b), w);
#pragma unroll
        for (int i = 0; i < 16; ++i) c += cc_accepted(w[i]);
        cnt[b] = uint8_t(c);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t t = __reduce_add_sync(0xffffffffu, red[threadIdx.x]);
        if (threadIdx.x == 0) cta_tot[blockIdx.x] = t;
    }
}

// in-place exclusive scan of n CTA totals (one CTA, strided chunks)
__global__ void __launch_bounds__(CC_THREADS) cc_scan_kernel(uint64_t* tot, uint64_t n, uint64_t* grand) {
    __shared__ uint64_t part[CC_THREADS];
    const uint64_t per = (n + CC_THREADS - 1) / CC_THREADS;
    const uint64_t i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
    uint64_t s = 0;
    for (uint64_t i = i0; i < i1; ++i) s += tot[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < CC_THREADS; o <<= 1) {
        const uint64_t add = threadIdx.x >= uint32_t(o) ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    uint64_t run = part[threadIdx.x] - s;
    for (uint64_t i = i0; i < i1; ++i) {
        const uint64_t v = tot[i];
        tot[i] = run;
        run += v;
    }
    if (threadIdx.x == CC_THREADS - 1) *grand = part[CC_THREADS - 1];
}

__global__ void __launch_bounds__(CC_THREADS) cc_compact_kernel(CcKey key, uint64_t n_blocks, const uint8_t* cnt,
                                                                 const uint64_t* cta_off, uint64_t n, int8_t* out) {
    __shared__ uint32_t scan[CC_THREADS];
    const uint64_t b = uint64_t(blockIdx.x) * CC_THREADS + threadIdx.x;
    const uint32_t c = b < n_blocks ? cnt[b] : 0;
    scan[threadIdx.x] = c;
    __syncthreads();
    for (int o = 1; o < CC_THREADS; o <<= 1) {
        const uint32_t add = threadIdx.x >= uint32_t(o) ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += add;
        __syncthreads();
    }
    uint64_t o = cta_off[blockIdx.x] + scan[threadIdx.x] - c;  // index of this block's first accepted byte
    if (b >= n_blocks || o >= n) return;
    uint32_t w[16];
    cc_block(key, uint32_t(b), w);
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t byte = (w[i] >> (8 * e)) & 0xFFu;
            if (byte != 0xFFu && o < n) out[o++] = int8_t(int(byte) - 127);
        }
}

}  // namespace dimg::dev
