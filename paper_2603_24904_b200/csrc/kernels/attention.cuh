// Decode attention step (proj/src/kernels.cpp:117-177), one CTA per head:
//
//   q', k' = RoPE(q_h, k_h, pos)            rope_apply_inplace (:70-82)
//   K[pos], V[pos] = k', v_h                KV append (:139-142)
//   s_t = mul16((sum_j q'_j K[t]_j)_int128 >> 16, inv_sqrt(dh))   (:143-151)
//   p = softmax_q16(s)                      exact LUT softmax (:90-107)
//   out_j = sum_t mul16(p_t, V[t]_j)        per-product floor (:153-159)
//
// The score dot is int128 (warp per position, lanes over dh); the softmax
// needs the exact max before any exp (no online form), so it is three block
// passes over an L2-resident score strip; PV uses the exact 64-bit split of
// mul16 for probabilities (q16.cuh mul16_prob). Every sum is an integer sum,
// so the parallel order cannot move a bit.
// KV layout: [layer][head][max_ctx][dh] int64 (the reference's LayerKv strips).
#pragma once

#include <cstdint>

#include "gemv.cuh"
#include "q16.cuh"

namespace dimg::dev {

constexpr int ATTN_THREADS = 256;

struct AttnArgs {
    const int64_t* qkv;       // [3*D]: q | k | v (this step's projections)
    int64_t* kc;              // this layer: [H][max_ctx][dh]
    int64_t* vc;
    const int64_t* rope_cos;  // [max_ctx][dh/2]
    const int64_t* rope_sin;
    int64_t* scores;          // [H][max_ctx] scratch
    int64_t* out;             // [D]
    const Ctl* ctl;
    uint32_t H, dh, max_ctx;
    int64_t inv_scale;        // inv_sqrt_q16(dh * ONE)
    const int64_t* exp_lut;
};

__device__ __forceinline__ void rope_pair(int64_t a, int64_t b, int64_t c, int64_t s, int64_t& x0,
                                          int64_t& x1) {
    x0 = wrap_sub(mul16(a, c), mul16(b, s));
    x1 = wrap_add(mul16(a, s), mul16(b, c));
}

// softmax_q16 in place over S[0..n) (proj/src/kernels.cpp:90-107): exact max,
// LUT weights lut(min(m - s, 8)), then p = (w << 16) / sum w (truncating).
// Block-wide; ends with a barrier.
__device__ __forceinline__ void softmax_strip_inl(int64_t* S, uint32_t n, const int64_t* lut, u128* red) {
    int64_t m = INT64_MIN;
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) m = S[t] > m ? S[t] : m;
    m = block_reduce<int64_t>(m, reinterpret_cast<int64_t*>(red),
                              [](int64_t x, int64_t y) { return x > y ? x : y; }, warp_max_i64);
    uint64_t total = 0;
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        int64_t d = wrap_sub(m, S[t]);
        total += uint64_t(exp_neg(d > 8 * ONE ? 8 * ONE : d, lut));
    }
    total = block_reduce<uint64_t>(total, reinterpret_cast<uint64_t*>(red),
                                   [](uint64_t x, uint64_t y) { return x + y; }, warp_sum_u64);
    const uint64_t inv = ~0ull / total;  // total >= 1: the maximum's weight is ONE
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        int64_t d = wrap_sub(m, S[t]);
        int64_t w = exp_neg(d > 8 * ONE ? 8 * ONE : d, lut);
        S[t] = int64_t(udiv_inv(uint64_t(w) << 16, total, inv));
    }
    __syncthreads();
}

// softmax_q16 over S[0..n) in place (proj/src/kernels.cpp:90-107), the same
// arithmetic as softmax_strip with fewer round trips: the int64 max as two
// 32-bit REDUX steps, the weights (<= 2^16 each, n <= 2^19) summed in 32 bits
// per warp, and the per-element division (w << 16) / total as a multiply by
// floor((2^64 - 1) / total) plus one exact correction step.
__device__ __forceinline__ void softmax_strip_fast(int64_t* S, uint32_t n, const int64_t* lut, u128* red) {
    if (n > (1u << 19)) {  // the 32-bit warp sums could overflow: the plain version
        softmax_strip_inl(S, n, lut, red);
        return;
    }
    int64_t* smax = reinterpret_cast<int64_t*>(red);           // [8]
    uint32_t* ssum = reinterpret_cast<uint32_t*>(smax + 8);    // [8]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t m = INT64_MIN;
#pragma unroll 1
    for (uint32_t t = threadIdx.x; t < n; t += ATTN_THREADS) m = S[t] > m ? S[t] : m;
    const int32_t mh = __reduce_max_sync(0xffffffffu, int32_t(uint64_t(m) >> 32));
    const uint32_t ml = __reduce_max_sync(0xffffffffu, int32_t(uint64_t(m) >> 32) == mh ? uint32_t(m) : 0u);
    if (lane == 0) smax[warp] = int64_t((uint64_t(uint32_t(mh)) << 32) | ml);
    __syncthreads();
    m = smax[0];
#pragma unroll
    for (int w = 1; w < ATTN_THREADS / 32; ++w) m = smax[w] > m ? smax[w] : m;
    uint32_t tot = 0;
#pragma unroll 1
    for (uint32_t t = threadIdx.x; t < n; t += ATTN_THREADS) {
        const int64_t d = wrap_sub(m, S[t]);
        const int64_t w = exp_neg(d > 8 * ONE ? 8 * ONE : d, lut);
        S[t] = w;
        tot += uint32_t(w);
    }
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) ssum[warp] = tot;
    __syncthreads();
    uint64_t total = 0;
#pragma unroll
    for (int w = 0; w < ATTN_THREADS / 32; ++w) total += ssum[w];
    if (total < (uint64_t(1) << 30)) {
        // floor(w 2^16 / total), w <= 2^16: a float estimate within one of the
        // quotient (three roundings of 2^-24 on a quotient <= 2^16), fixed by
        // the exact remainder, which lies in (-total, 2 total) and so is an
        // exact int32 although w 2^16 and q total wrap (no 64-bit division)
        const uint32_t tot32 = uint32_t(total);
        const float scale = 65536.0f / float(tot32);
#pragma unroll 1
        for (uint32_t t = threadIdx.x; t < n; t += ATTN_THREADS) {
            const uint32_t w = uint32_t(S[t]);
            uint32_t q = uint32_t(float(w) * scale);
            const int32_t r = int32_t((w << 16) - q * tot32);
            q -= r < 0;
            q += r >= int32_t(tot32);
            S[t] = int64_t(q);
        }
    } else {
        const uint64_t inv = ~0ull / total;
#pragma unroll 1
        for (uint32_t t = threadIdx.x; t < n; t += ATTN_THREADS) {
            const uint64_t a = uint64_t(S[t]) << 16;
            uint64_t q = __umul64hi(a, inv);  // floor(a / total) or one less
            q += (a - q * total) >= total;
            S[t] = int64_t(q);
        }
    }
    __syncthreads();
}

__device__ __noinline__ void softmax_strip(int64_t* S, uint32_t n, const int64_t* lut, u128* red) {
    softmax_strip_inl(S, n, lut, red);
}

// Bytes of shared scratch attn_head needs (score strip in shared memory when
// max_ctx > 0, else in a.scores).
__host__ __device__ constexpr size_t attn_op_scratch_bytes(uint32_t dh) {  // attn_head_part, strip in global
    return (2 * size_t(dh) + 257 + ATTN_THREADS) * sizeof(int64_t);
}
__host__ __device__ constexpr size_t attn_scratch_bytes(uint32_t dh, uint32_t max_ctx = 0) {
    return (6 * size_t(dh) + 257 + 4 * ATTN_THREADS + max_ctx) * sizeof(int64_t);
}

// One head of one attention step at position `pos`, or one of `nparts`
// slices of it: every part computes all scores and the softmax (cheap,
// redundant) and the probability-weighted V sum for its own slice of the
// head's dimensions -- an exact split with no cross-CTA exchange. Part 0
// writes the new K/V row. Block-wide (blockDim.x == ATTN_THREADS); `scratch`
// = attn_scratch_bytes(dh[, max_ctx]) of shared memory; `smem_scores` keeps
// the score strip on chip (required when nparts > 1). When `planes` is set,
// the output is also emitted as 3-limb byte planes for the WO GEMV (plus the
// wide flag), see persistent.cuh.
__device__ __noinline__ void attn_head_part(const AttnArgs& a_in, uint32_t h, uint32_t part_idx,
                                            uint32_t nparts, uint32_t pos, int64_t* scratch, u128* red,
                                            uint8_t* planes, uint32_t pitch, uint32_t* flag, uint32_t tag,
                                            bool smem_scores, unsigned long long* tr) {
    // one copy of the arguments into registers (a_in may live in local memory,
    // whose L1 lines the persistent kernel's grid fences invalidate)
    const AttnArgs a = a_in;
    const uint32_t dh = a.dh, half = dh / 2, D = a.H * dh;
    int64_t* qrot = scratch;                                   // [dh]
    int64_t* krot = scratch + dh;                              // [dh] this position's key
    int64_t* lut = scratch + 2 * dh;                           // [257] (unless a.exp_lut is on chip)
    uint64_t* part = reinterpret_cast<uint64_t*>(lut + 257);   // [ATTN_THREADS]
    if (smem_scores) lut = const_cast<int64_t*>(a.exp_lut);  // persistent kernel: already in smem
    else
        for (int i = threadIdx.x; i < 257; i += blockDim.x) lut[i] = a.exp_lut[i];
    int64_t* S = smem_scores ? reinterpret_cast<int64_t*>(part + ATTN_THREADS)
                             : a.scores + size_t(h) * a.max_ctx;

    const int64_t* q = a.qkv + size_t(h) * dh;
    const int64_t* k = a.qkv + D + size_t(h) * dh;
    const int64_t* v = a.qkv + 2 * size_t(D) + size_t(h) * dh;
    int64_t* K = a.kc + size_t(h) * a.max_ctx * dh;
    int64_t* V = a.vc + size_t(h) * a.max_ctx * dh;
    const int64_t* cr = a.rope_cos + size_t(pos) * half;
    const int64_t* sr = a.rope_sin + size_t(pos) * half;
    // RoPE on q and k (rope_apply_inplace, kernels.cpp:70-82); K/V append
    for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) {
        const int64_t c = cr[i], s = sr[i];
        rope_pair(q[i], q[i + half], c, s, qrot[i], qrot[i + half]);
        rope_pair(k[i], k[i + half], c, s, krot[i], krot[i + half]);
        if (part_idx == 0) {
            K[size_t(pos) * dh + i] = krot[i];
            K[size_t(pos) * dh + i + half] = krot[i + half];
        }
    }
    if (part_idx == 0)
        for (uint32_t j = threadIdx.x; j < dh; j += blockDim.x) V[size_t(pos) * dh + j] = v[j];
    int q_small = 1;
    for (uint32_t j = threadIdx.x; j < dh; j += blockDim.x)
        q_small &= qrot[j] < (int64_t(1) << 27) && qrot[j] > -(int64_t(1) << 27);
    q_small = __syncthreads_and(q_small) && dh <= 512;  // 512 * 2^54 < 2^63
    if (tr) tr[4] = clock64();

    // scores (kernels.cpp:143-151): one warp per cached position, lanes over
    // dh, four positions per warp in flight. The dot is int128 in the
    // reference; when every |q|, |k| < 2^27 and dh <= 512 the int64 sum is
    // exact and a warp-uniform check takes that path.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t t0 = warp; t0 <= pos; t0 += 4 * nw) {
        int small = q_small;
        uint64_t d64[4] = {0, 0, 0, 0};
        u128 dot[4] = {0, 0, 0, 0};
        for (uint32_t j0 = 0; j0 < dh; j0 += 128) {
            int64_t kv[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t t = t0 + u * nw;
                const int64_t* kt = t == pos ? krot : K + size_t(t) * dh;  // newest key: on chip
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t j = j0 + lane + 32 * c;
                    kv[u][c] = (t <= pos && j < dh) ? kt[j] : 0;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    small &= kv[u][c] < (int64_t(1) << 27) && kv[u][c] > -(int64_t(1) << 27);
            small = __all_sync(0xffffffffu, small);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t j = j0 + lane + 32 * c;
                const int64_t qj = j < dh ? qrot[j] : 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (small) d64[u] += uint64_t(qj * kv[u][c]);
                    else dot[u] += mul_full(qj, kv[u][c]);
                }
            }
        }
#pragma unroll 1
        for (int u = 0; u < 4; ++u) {
            const uint32_t t = t0 + u * nw;
            // int64 partial (exact) + 128-bit remainder, then the warp total
            const u128 d = warp_sum_u128(dot[u] + u128(int64_t(d64[u])));
            if (lane == 0 && t <= pos) S[t] = mul16(int64_t(i128(d) >> 16), a.inv_scale);
        }
    }
    __syncthreads();
    if (tr) tr[5] = clock64();
    softmax_strip(S, pos + 1, lut, red);
    if (tr) tr[6] = clock64();

    // out_j = sum_t mul16(p_t, V[t]_j) (kernels.cpp:153-159) over this part's
    // dims; threads = (dim, position slice); the newest V row is read from
    // this step's projection (part 0 may not have stored it yet)
    const uint32_t dpp = (dh + nparts - 1) / nparts;
    const uint32_t d0 = min(dh, part_idx * dpp), d1 = min(dh, d0 + dpp), nd = d1 - d0;
    if (nd > 0 && nd <= ATTN_THREADS) {
        const uint32_t slices = ATTN_THREADS / nd;
        const uint32_t jj = threadIdx.x % nd, sl = threadIdx.x / nd, j = d0 + jj;
        uint64_t acc = 0;
        if (sl < slices) {
            uint32_t t = sl;
            for (; t + 7 * slices < pos; t += 8 * slices) {  // 8 V rows in flight
                int64_t vv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) vv[u] = V[size_t(t + u * slices) * dh + j];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += uint64_t(mul16_prob(S[t + u * slices], vv[u]));
            }
            for (; t <= pos; t += slices)
                acc += uint64_t(mul16_prob(S[t], t == pos ? v[j] : V[size_t(t) * dh + j]));
        }
        part[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < nd) {
            uint64_t sum = 0;
            for (uint32_t s = 0; s < slices; ++s) sum += part[s * nd + threadIdx.x];
            const uint32_t o = h * dh + d0 + threadIdx.x;
            a.out[o] = int64_t(sum);
            if (planes) {
                planes[o] = uint8_t(sum);
                planes[pitch + o] = uint8_t(sum >> 8);
                planes[2 * pitch + o] = uint8_t(sum >> 16);
                const int64_t sv = int64_t(sum);
                if (sv < -(int64_t(1) << 23) || sv >= (int64_t(1) << 23)) *((volatile uint32_t*)flag) = tag;
            }
        }
    } else {
        for (uint32_t j = d0 + threadIdx.x; j < d1; j += blockDim.x) {
            uint64_t acc = 0;
            for (uint32_t t = 0; t <= pos; ++t)
                acc += uint64_t(mul16_prob(S[t], t == pos ? v[j] : V[size_t(t) * dh + j]));
            const uint32_t o = h * dh + j;
            a.out[o] = int64_t(acc);
            if (planes) {
                planes[o] = uint8_t(acc);
                planes[pitch + o] = uint8_t(acc >> 8);
                planes[2 * pitch + o] = uint8_t(acc >> 16);
                const int64_t sv = int64_t(acc);
                if (sv < -(int64_t(1) << 23) || sv >= (int64_t(1) << 23)) *((volatile uint32_t*)flag) = tag;
            }
        }
    }
    __syncthreads();  // scratch may be reused by the caller's next head/stage
    if (tr) tr[7] = clock64();
}

__global__ void __launch_bounds__(ATTN_THREADS) attn_decode_kernel(AttnArgs a) {
    extern __shared__ __align__(16) int64_t attn_smem[];
    __shared__ u128 red[32];
    attn_head_part(a, blockIdx.x, 0, 1, a.ctl->pos, attn_smem, red, nullptr, 0, nullptr, 0, false, nullptr);
}

}  // namespace dimg::dev
