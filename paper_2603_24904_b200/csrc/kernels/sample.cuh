// Seeded sampling from one logits row, exact: sample_from_logits
// (proj/src/engine.cpp:122-139) as the selection step of generate_sampled
// (:148-163). One 1024-thread CTA per row (the vocabulary in contiguous
// per-thread segments):
//   scaled_i = int64((int128(logit_i) << 16) / T)        (truncating, low 64 bits)
//   p = softmax_q16(scaled)                              (exp LUT, (w << 16) / total)
//   threshold = (draw * sum p) >> 32; token = first i with p_0 + .. + p_i > threshold
// The draw is the step's ChaCha20 u32 (precomputed on the host from the
// BLAKE3(model bytes || prompt) key). The token goes to tokens[pos + 1],
// where the next decode step reads it.
// Reference edge cases kept:
//   * scaled logits spanning more than 2^63: m - s wraps negative and
//     exp_neg_lut throws std::domain_error (q16.cpp:82) -> bit 1 of *err
//     (DIMG_EDOMAIN at the API), no LUT read out of range;
//   * every probability truncated to 0 (vocab > 65536, near-flat): the
//     cumulative walk never passes the threshold and the reference returns
//     V - 1 (engine.cpp:138).
#pragma once

#include <cstdint>

#include "q16.cuh"

namespace dimg::dev {

constexpr int SM_THREADS = 1024;

template <class T, class Op>
__device__ __forceinline__ T sm_block_reduce(T v, T* red, Op op) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        T w = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w = op(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (threadIdx.x == 0) red[0] = w;
    }
    __syncthreads();
    const T r = red[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SM_THREADS) sample_kernel(const int64_t* __restrict__ logits, uint32_t V,
                                                            int64_t temperature, const uint32_t* __restrict__ draws,
                                                            uint32_t step, const int64_t* __restrict__ lut_g,
                                                            int64_t* __restrict__ scratch, uint32_t* tokens,
                                                            uint32_t pos, uint32_t* err) {
    __shared__ int64_t lut[257];
    __shared__ int64_t red[32];
    __shared__ uint64_t scan[SM_THREADS];
    for (int i = threadIdx.x; i < 257; i += SM_THREADS) lut[i] = lut_g[i];
    const uint32_t per = (V + SM_THREADS - 1) / SM_THREADS;
    const uint32_t i0 = min(V, threadIdx.x * per), i1 = min(V, i0 + per);
    // 1. temperature scaling + the maximum
    int64_t mx = INT64_MIN;
    for (uint32_t i = i0; i < i1; ++i) {
        const int64_t v = int64_t((__int128(logits[i]) << 16) / temperature);
        scratch[i] = v;
        mx = v > mx ? v : mx;
    }
    const int64_t m = sm_block_reduce<int64_t>(mx, red, [](int64_t a, int64_t b) { return a > b ? a : b; });
    // 2. softmax_q16 weights (kernels.cpp:90-107) and their total
    int64_t tot = 0;
    int bad = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        int64_t d = wrap_sub(m, scratch[i]);
        bad |= d < 0;
        tot += d < 0 ? 0 : exp_neg(d > 8 * ONE ? 8 * ONE : d, lut);
    }
    if (__syncthreads_or(bad)) {  // exp_neg_lut's domain_error: no token
        if (threadIdx.x == 0) atomicOr(err, 2u);
        return;
    }
    const int64_t total = sm_block_reduce<int64_t>(tot, red, [](int64_t a, int64_t b) { return a + b; });
    // 3. probabilities (truncating division by the total) and this segment's mass
    const uint64_t inv = ~0ull / uint64_t(total);
    uint64_t seg = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        int64_t d = wrap_sub(m, scratch[i]);
        const uint64_t w = uint64_t(exp_neg(d > 8 * ONE ? 8 * ONE : d, lut));
        const uint64_t p = udiv_inv(w << 16, uint64_t(total), inv);
        scratch[i] = int64_t(p);
        seg += p;
    }
    // 4. exclusive scan of the segment masses, then the one segment that
    //    crosses the threshold walks to the token
    scan[threadIdx.x] = seg;
    __syncthreads();
    for (int o = 1; o < SM_THREADS; o <<= 1) {
        const uint64_t add = threadIdx.x >= uint32_t(o) ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += add;
        __syncthreads();
    }
    const uint64_t mass = scan[SM_THREADS - 1];
    const uint64_t start = scan[threadIdx.x] - seg;
    const int64_t threshold = int64_t((uint64_t(draws[step]) * mass) >> 32);
    if (mass == 0) {  // no cumulative mass ever exceeds the threshold (0): the reference's V - 1
        if (threadIdx.x == 0) tokens[pos + 1] = V - 1;
        return;
    }
    if (int64_t(start) <= threshold && threshold < int64_t(start + seg)) {
        int64_t cum = int64_t(start);
        for (uint32_t i = i0; i < i1; ++i) {
            cum += scratch[i];
            if (cum > threshold) {
                tokens[pos + 1] = i;
                break;
            }
        }
    }
}

}  // namespace dimg::dev
