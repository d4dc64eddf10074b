// BLAKE3 (hash mode, 32-byte output) of a device-resident byte string: the
// model-bytes hash of weight_hash / deserialize (proj/src/model.cpp:310-316)
// and verify_by_reexecution (proj/src/attest.cpp:93), at HBM speed.
//
// The algorithm is the published BLAKE3 (the reference's
// proj/src/blake3.cpp implements the same): 1 KiB chunks of 16 64-byte
// blocks compressed in sequence (CHUNK_START / CHUNK_END, counter = chunk
// index), chunk chaining values merged pairwise by PARENT compressions into
// the left-complete binary tree, the final merge (or a lone chunk's last
// block) flagged ROOT. Level by level the tree is "merge adjacent pairs, an
// odd last node moves up unchanged" -- for n nodes at a level the left
// subtree of the root holds the largest power of two below n, as the
// reference's CV stack builds it -- so any aligned group of 2^k nodes
// reduces independently given the global node count of each level.
//
// Kernels: b3_chunks_kernel hashes 256 chunks per CTA (one per thread, the
// input read with 16-byte non-coherent loads) and folds their 256 chaining
// values in shared memory through 8 levels; b3_fold_kernel folds 256
// chaining values of a higher level per CTA. 6.75 GB (6.6 M chunks) takes
// four launches. Compression: 7 rounds of the G function on 16 words with the
// message schedule fixed at compile time, so the block stays in registers.
#pragma once

#include <cstdint>

namespace dimg::dev {

constexpr uint32_t B3_CHUNK_START = 1, B3_CHUNK_END = 2, B3_PARENT = 4, B3_ROOT = 8;
constexpr int B3_FOLD = 256;  // nodes folded per CTA (8 levels)

__device__ __constant__ uint32_t B3_IV[8] = {0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au,
                                             0x510E527Fu, 0x9B05688Cu, 0x1F83D9ABu, 0x5BE0CD19u};

// message word used at position i of round r: round 0 in order, each next
// round the published permutation {2,6,3,10,7,0,4,13,1,11,12,5,9,14,15,8}
// applied to the previous one
// (a constexpr function of compile-time indices: folds to register names)
__host__ __device__ constexpr int b3_sig(int r, int i) {
    constexpr int P[16] = {2, 6, 3, 10, 7, 0, 4, 13, 1, 11, 12, 5, 9, 14, 15, 8};
    for (; r > 0; --r) i = P[i];
    return i;
}

__device__ __forceinline__ uint32_t b3_rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void b3_g(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, uint32_t mx, uint32_t my) {
    a = a + b + mx;
    d = b3_rotr(d ^ a, 16);
    c = c + d;
    b = b3_rotr(b ^ c, 12);
    a = a + b + my;
    d = b3_rotr(d ^ a, 8);
    c = c + d;
    b = b3_rotr(b ^ c, 7);
}

// The compression function; cv (in/out) = the first 8 output words.
__device__ __forceinline__ void b3_compress(uint32_t (&cv)[8], const uint32_t (&m)[16], uint64_t counter,
                                            uint32_t block_len, uint32_t flags) {
    uint32_t v[16] = {cv[0],    cv[1],    cv[2],    cv[3],    cv[4],    cv[5],          cv[6],
                      cv[7],    B3_IV[0], B3_IV[1], B3_IV[2], B3_IV[3], uint32_t(counter), uint32_t(counter >> 32),
                      block_len, flags};
#pragma unroll
    for (int r = 0; r < 7; ++r) {
        b3_g(v[0], v[4], v[8], v[12], m[b3_sig(r, 0)], m[b3_sig(r, 1)]);
        b3_g(v[1], v[5], v[9], v[13], m[b3_sig(r, 2)], m[b3_sig(r, 3)]);
        b3_g(v[2], v[6], v[10], v[14], m[b3_sig(r, 4)], m[b3_sig(r, 5)]);
        b3_g(v[3], v[7], v[11], v[15], m[b3_sig(r, 6)], m[b3_sig(r, 7)]);
        b3_g(v[0], v[5], v[10], v[15], m[b3_sig(r, 8)], m[b3_sig(r, 9)]);
        b3_g(v[1], v[6], v[11], v[12], m[b3_sig(r, 10)], m[b3_sig(r, 11)]);
        b3_g(v[2], v[7], v[8], v[13], m[b3_sig(r, 12)], m[b3_sig(r, 13)]);
        b3_g(v[3], v[4], v[9], v[14], m[b3_sig(r, 14)], m[b3_sig(r, 15)]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = v[i] ^ v[i + 8];
}

// parent node of two chaining values (key = IV)
__device__ __forceinline__ void b3_parent(const uint32_t* l, const uint32_t* r, uint32_t flags, uint32_t (&out)[8]) {
    uint32_t m[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = l[i], m[i + 8] = r[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = B3_IV[i];
    b3_compress(out, m, 0, 64, B3_PARENT | flags);
}

// Folds the CTA's B3_FOLD nodes of level `lvl0` (cv[i] = node base + i,
// base = blockIdx.x * B3_FOLD; nodes >= cnt absent) through 8 levels in
// shared memory. Returns (thread 0) the node of level lvl0 + 8 in cv[0];
// writes the root hash when the final merge happens in this CTA.
__device__ __forceinline__ void b3_fold(uint32_t (*cv)[9], uint64_t cnt, uint32_t* root_out) {
    uint64_t base = uint64_t(blockIdx.x) * B3_FOLD;
#pragma unroll 1
    for (int w = B3_FOLD / 2; w >= 1; w >>= 1) {
        __syncthreads();
        const uint32_t i = threadIdx.x;
        uint32_t out[8];
        bool write = false;
        if (i < uint32_t(w)) {
            const uint64_t left = base + 2 * i;  // global index of the pair's left node at this level
            if (left + 1 < cnt) {
                b3_parent(cv[2 * i], cv[2 * i + 1], cnt == 2 ? B3_ROOT : 0, out);
                write = true;
                if (cnt == 2 && root_out)
#pragma unroll
                    for (int k = 0; k < 8; ++k) root_out[k] = out[k];
            } else if (left < cnt) {  // odd last node: moves up unchanged
#pragma unroll
                for (int k = 0; k < 8; ++k) out[k] = cv[2 * i][k];
                write = true;
            }
        }
        __syncthreads();
        if (write)
#pragma unroll
            for (int k = 0; k < 8; ++k) cv[i][k] = out[k];
        cnt = (cnt + 1) / 2;
        base /= 2;
    }
    __syncthreads();
}

// Chunk chaining values of chunks [256 b, 256 b + 256), folded to one node
// of level 8 (out[b]). len >= 1 (the empty input is one empty chunk: host).
__global__ void __launch_bounds__(B3_FOLD) b3_chunks_kernel(const uint8_t* __restrict__ data, uint64_t len,
                                                             uint32_t* __restrict__ out, uint32_t* root_out) {
    __shared__ uint32_t cv_s[B3_FOLD][9];  // +1 word: no bank conflicts across threads
    const uint64_t n_chunks = (len + 1023) / 1024;
    const uint64_t c = uint64_t(blockIdx.x) * B3_FOLD + threadIdx.x;
    if (c < n_chunks) {
        uint32_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = B3_IV[i];
        const uint8_t* p = data + c * 1024;
        const uint64_t clen = c + 1 < n_chunks ? 1024 : len - c * 1024;  // 1..1024
        const bool aligned = (reinterpret_cast<uintptr_t>(data) & 15) == 0;
        if (clen == 1024 && aligned) {  // full chunk: 16-byte loads
            const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll 1
            for (int blk = 0; blk < 16; ++blk) {
                uint32_t m[16];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint4 x = __ldg(q + blk * 4 + k);
                    m[4 * k] = x.x, m[4 * k + 1] = x.y, m[4 * k + 2] = x.z, m[4 * k + 3] = x.w;
                }
                const uint32_t fl = (blk == 0 ? B3_CHUNK_START : 0) | (blk == 15 ? B3_CHUNK_END : 0) |
                                    (blk == 15 && n_chunks == 1 ? B3_ROOT : 0);
                b3_compress(h, m, c, 64, fl);
            }
        } else {  // last (partial) chunk or unaligned input: bytes, zero-padded blocks
            const uint32_t nblk = uint32_t((clen + 63) / 64);
#pragma unroll 1
            for (uint32_t blk = 0; blk < nblk; ++blk) {
                uint32_t m[16];
                const uint32_t blen = blk + 1 < nblk ? 64 : uint32_t(clen - 64 * blk);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    uint32_t w = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t off = 4 * k + e;
                        if (off < blen) w |= uint32_t(p[64 * blk + off]) << (8 * e);
                    }
                    m[k] = w;
                }
                const uint32_t fl = (blk == 0 ? B3_CHUNK_START : 0) | (blk + 1 == nblk ? B3_CHUNK_END : 0) |
                                    (blk + 1 == nblk && n_chunks == 1 ? B3_ROOT : 0);
                b3_compress(h, m, c, blen, fl);
            }
        }
        if (n_chunks == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) root_out[i] = h[i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) cv_s[threadIdx.x][i] = h[i];
    }
    b3_fold(cv_s, n_chunks, root_out);
    if (threadIdx.x < 8 && uint64_t(blockIdx.x) * B3_FOLD < n_chunks) out[size_t(blockIdx.x) * 8 + threadIdx.x] = cv_s[0][threadIdx.x];
}

// One more 8-level fold: cnt nodes in (8 words each) -> ceil(cnt / 256) out.
__global__ void __launch_bounds__(B3_FOLD) b3_fold_kernel(const uint32_t* __restrict__ in, uint64_t cnt,
                                                           uint32_t* __restrict__ out, uint32_t* root_out) {
    __shared__ uint32_t cv_s[B3_FOLD][9];
    const uint64_t i = uint64_t(blockIdx.x) * B3_FOLD + threadIdx.x;
    if (i < cnt)
#pragma unroll
        for (int k = 0; k < 8; ++k) cv_s[threadIdx.x][k] = in[i * 8 + k];
    b3_fold(cv_s, cnt, root_out);
    if (threadIdx.x < 8) out[size_t(blockIdx.x) * 8 + threadIdx.x] = cv_s[0][threadIdx.x];
}

}  // namespace dimg::dev
