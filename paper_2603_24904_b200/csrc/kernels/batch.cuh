// Batched steps over many independent sequences (C5: 64 sequences, one per
// slot of a batch): every token of a step is (sequence, position, token id),
// the dense products of all of them are one tensor-core limb GEMM per matrix
// (tc_gemm.cuh), and attention / RoPE / the KV append are per token against
// that token's own sequence cache. The same step function serves the prompt
// phase (all prompt positions but the last of every sequence, no logits) and
// the decode steps (one token per sequence, logits + greedy argmax), so a
// sequence sees exactly the forward passes of run_generation
// (proj/src/engine.cpp:31-54).
//
// The batch keeps only the int32 KV mirror; any value outside the fast
// representations (3 byte limbs, int32 K/V and scores, |q| < 2^23) sets
// *wide and the engine regenerates every sequence on the exact single-
// sequence path instead.
#pragma once

#include <cstdint>

#include "attention.cuh"
#include "prefill.cuh"
#include "q16.cuh"

namespace dimg::dev {

struct BatchTok {  // device arrays, one entry per token of the step
    const uint32_t* tok;
    const uint32_t* seq;
    const uint32_t* pos;
};

__global__ void bd_embed_kernel(BatchTok bt, uint32_t n, const int8_t* __restrict__ E,
                                const int64_t* __restrict__ Es, uint32_t D, int32_t* __restrict__ x, uint32_t* wide) {
    pdl_launch_dependents();
    pdl_wait();
    int bad = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < size_t(n) * D;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(i / D), j = uint32_t(i % D);
        const uint32_t tk = bt.tok[t];
        const int64_t v = int64_t(uint64_t(int64_t(E[size_t(tk) * D + j])) * uint64_t(Es[tk]));
        bad |= !fits_i32(v);  // the int32 residual stream (pf_embed_kernel)
        x[i] = int32_t(v);
    }
    if (bad) *wide = 1;
}

// RoPE (proj/src/kernels.cpp:70-82) and the KV append (:139-142) of token t
// at its own (sequence, position); q' overwrites q. grid (n, H), dh/2 threads.
// cache layout: [seq][layer][head][ctx][dh] int32; this layer's base given.
__global__ void bd_rope_kv_kernel(int64_t* __restrict__ qkv, BatchTok bt, uint32_t D, uint32_t dh,
                                  const int64_t* __restrict__ rc, const int64_t* __restrict__ rs, int32_t* K32,
                                  int32_t* V32, size_t seq_stride, uint32_t ctx, uint32_t* wide) {
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x, h = blockIdx.y, half = dh / 2, i = threadIdx.x;
    const uint32_t b = bt.seq[t], p = bt.pos[t];
    int64_t* q = qkv + size_t(t) * 3 * D + size_t(h) * dh;
    const int64_t* k = q + D;
    const int64_t* v = q + 2 * D;
    const size_t kv = size_t(b) * seq_stride + (size_t(h) * ctx + p) * dh;
    const int64_t c = rc[size_t(p) * half + i], s = rs[size_t(p) * half + i];
    int64_t q0, q1, k0, k1;
    rope_pair(q[i], q[i + half], c, s, q0, q1);
    rope_pair(k[i], k[i + half], c, s, k0, k1);
    const int64_t v0 = v[i], v1 = v[i + half];
    __syncthreads();
    q[i] = q0;
    q[i + half] = q1;
    K32[kv + i] = int32_t(k0);
    K32[kv + i + half] = int32_t(k1);
    V32[kv + i] = int32_t(v0);
    V32[kv + i + half] = int32_t(v1);
    const auto b23 = [](int64_t a) { return a >= -(int64_t(1) << 23) && a < (int64_t(1) << 23); };
    if (!fits_i32(k0) || !fits_i32(k1) || !fits_i32(v0) || !fits_i32(v1) || !b23(q0) || !b23(q1)) *wide = 1;
}

// rmsnorm (proj/src/kernels.cpp:56-68) of each token row into the next
// GEMM's digit planes, for the few tokens of a decode batch: ONE 1024-thread
// CTA per token (no cluster barriers; round 1's 4-CTA cluster with a
// distributed-shared-memory exchange was 2% slower per C5 step): 4 elements
// per thread for K <= 4096, x^2 summed in 21-bit chunks with REDUX
// (per-warp totals < 2^29), one shared-memory pass for the block total.
__global__ void __launch_bounds__(1024) bd_norm1k_kernel(const int32_t* __restrict__ x, uint32_t K,
                                                         const int64_t* __restrict__ gamma, int gamma_unit,
                                                         const int64_t* __restrict__ seeds, uint8_t* planes,
                                                         uint32_t rows_pad, uint32_t ldp, uint32_t* wide) {
    __shared__ uint32_t s_c[32][3];
    __shared__ int64_t s_r;
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x;
    const int32_t* xr = x + size_t(t) * K;
    constexpr int PER = 4;
    int64_t v[PER];
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    const auto add_sq = [&](int64_t xv) {
        const uint64_t q2 = uint64_t(xv * xv);  // < 2^62
        c0 += uint32_t(q2) & 0x1FFFFFu;
        c1 += uint32_t(q2 >> 21) & 0x1FFFFFu;
        c2 += uint32_t(q2 >> 42);
    };
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const uint32_t j = threadIdx.x + u * 1024;
        v[u] = j < K ? xr[j] : 0;
        add_sq(v[u]);
    }
    for (uint32_t j = threadIdx.x + PER * 1024; j < K; j += 1024) add_sq(int64_t(xr[j]));  // K <= 8192
    c0 = __reduce_add_sync(0xffffffffu, c0);
    c1 = __reduce_add_sync(0xffffffffu, c1);
    c2 = __reduce_add_sync(0xffffffffu, c2);
    if ((threadIdx.x & 31) == 0) {
        s_c[threadIdx.x >> 5][0] = c0;
        s_c[threadIdx.x >> 5][1] = c1;
        s_c[threadIdx.x >> 5][2] = c2;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // warp 0 adds the 32 warp totals (< 2^29 each) as 16-bit halves, so
        // every 32-bit REDUX sum stays exact
        const auto add32 = [](uint32_t v) {
            return uint64_t(__reduce_add_sync(0xffffffffu, v & 0xFFFFu)) +
                   (uint64_t(__reduce_add_sync(0xffffffffu, v >> 16)) << 16);
        };
        const uint64_t t0 = add32(s_c[threadIdx.x][0]);
        const uint64_t t1 = add32(s_c[threadIdx.x][1]);
        const uint64_t t2 = add32(s_c[threadIdx.x][2]);
        const u128 tot = u128(t0) + (u128(t1) << 21) + (u128(t2) << 42);
        const int64_t ms = (tot >> 63) != 0          ? int64_t((i128(tot) / i128(K)) >> 16)
                           : (K & (K - 1)) == 0       ? int64_t((uint64_t(tot) >> (__ffs(K) - 1)) >> 16)
                                                      : int64_t((uint64_t(tot) / K) >> 16);
        if (threadIdx.x == 0) {
            s_r = ms + 1 > 0 ? inv_sqrt_q16(ms + 1, seeds) : 0;
            if (ms + 1 <= 0) *wide = 1;
        }
    }
    __syncthreads();
    const int64_t r = s_r;
    const size_t plane = size_t(rows_pad) * ldp;
    uint8_t* pr = planes + size_t(t) * ldp;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const uint32_t j = threadIdx.x + u * 1024;
        if (j < K) {
            int64_t o = mul16(v[u], r);
            if (!gamma_unit) o = mul16(o, gamma[j]);
            pf_put_limbs(pr + j, plane, o, wide);
        }
    }
    for (uint32_t j = threadIdx.x + PER * 1024; j < K; j += 1024) {
        int64_t o = mul16(int64_t(xr[j]), r);
        if (!gamma_unit) o = mul16(o, gamma[j]);
        pf_put_limbs(pr + j, plane, o, wide);
    }
}

constexpr int BD_THREADS = 256;

__host__ __device__ constexpr size_t bd_attn_smem(uint32_t dh, uint32_t ctx) {
    return size_t(ctx) * 8 + size_t(dh) * 4 + size_t(BD_THREADS) * 8 * 4;
}

// attention_step (proj/src/kernels.cpp:117-177) of token t against positions
// 0..pos[t] of its sequence, exact: int64 score sums of int32 products (one
// warp per position, lanes over 4-dim quads), the softmax of softmax_q16 over
// the strip in shared memory, the per-product floor of mul16(p, v).
// grid (H, n); writes the limb planes of the attention vector, row t.
// rc != nullptr (decode steps: one token per sequence, so no other CTA
// reads this (sequence, head) row): the CTA also does bd_rope_kv_kernel's
// work for its head first -- RoPE of q and k, the K/V append -- one launch
// per layer fewer.
// KDB (decode steps of <= 16 sequences): the next pass's K rows load while
// this pass's products run (+1% at 8 sequences; its registers cost the
// 64-sequence steps occupancy, so those use the plain loop).
template <bool KDB>
__global__ void __launch_bounds__(BD_THREADS) bd_attn_kernel(const int64_t* __restrict__ qkv, BatchTok bt,
                                                             uint32_t D, uint32_t dh, int32_t* K32, int32_t* V32,
                                                             size_t seq_stride, uint32_t ctx, int64_t inv_scale,
                                                             const int64_t* __restrict__ lut_g, uint8_t* planes,
                                                             uint32_t rows_pad, uint32_t ldp, uint32_t* wide,
                                                             const int64_t* __restrict__ rc,
                                                             const int64_t* __restrict__ rs) {
    extern __shared__ __align__(16) uint8_t bd_smem[];
    __shared__ int64_t lut[257];
    __shared__ u128 red[32];
    pdl_launch_dependents();
    for (int i = threadIdx.x; i < 257; i += BD_THREADS) lut[i] = lut_g[i];  // constant: before the wait
    pdl_wait();
    const uint32_t h = blockIdx.x, t = blockIdx.y;
    const uint32_t b = bt.seq[t], T = bt.pos[t] + 1;
    int64_t* S = reinterpret_cast<int64_t*>(bd_smem);              // [ctx]
    int32_t* q = reinterpret_cast<int32_t*>(S + ctx);              // [dh]
    uint64_t* part = reinterpret_cast<uint64_t*>(q + dh + (dh & 1));  // [4 * BD_THREADS]
    const int32_t* Kh = K32 + size_t(b) * seq_stride + size_t(h) * ctx * dh;
    const int32_t* Vh = V32 + size_t(b) * seq_stride + size_t(h) * ctx * dh;
    const int64_t* qr = qkv + size_t(t) * 3 * D + size_t(h) * dh;
    if (rc) {
        // RoPE (kernels.cpp:70-82) of q and k at position T - 1, the K/V append
        // (:139-142); the same values and range checks as bd_rope_kv_kernel
        const uint32_t half = dh / 2, p = T - 1;
        const int64_t* kr = qr + D;
        const int64_t* vr = qr + 2 * D;
        int32_t* Kw = K32 + size_t(b) * seq_stride + (size_t(h) * ctx + p) * dh;
        int32_t* Vw = V32 + size_t(b) * seq_stride + (size_t(h) * ctx + p) * dh;
        const auto b23 = [](int64_t a) { return a >= -(int64_t(1) << 23) && a < (int64_t(1) << 23); };
        int bad = 0;
        for (uint32_t i = threadIdx.x; i < half; i += BD_THREADS) {
            const int64_t c = rc[size_t(p) * half + i], sn = rs[size_t(p) * half + i];
            int64_t q0, q1, k0, k1;
            rope_pair(qr[i], qr[i + half], c, sn, q0, q1);
            rope_pair(kr[i], kr[i + half], c, sn, k0, k1);
            q[i] = int32_t(q0);
            q[i + half] = int32_t(q1);
            Kw[i] = int32_t(k0);
            Kw[i + half] = int32_t(k1);
            bad |= !fits_i32(k0) || !fits_i32(k1) || !b23(q0) || !b23(q1);
        }
        for (uint32_t j = threadIdx.x; j < dh; j += BD_THREADS) {
            const int64_t v = vr[j];
            Vw[j] = int32_t(v);
            bad |= !fits_i32(v);
        }
        if (bad) *wide = 1;
    } else {
        for (uint32_t j = threadIdx.x; j < dh; j += BD_THREADS) q[j] = int32_t(qr[j]);
    }
    __syncthreads();  // q, and this CTA's appended K/V row, before they are read
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int big = 0;
    const size_t plane = size_t(rows_pad) * ldp;
    if ((dh & 3) == 0 && dh <= 512) {
        // The decode kernel's layout (persistent.cuh attn_split), so a step
        // costs a few memory round trips instead of one per position group:
        // scores -- an octet of lanes per position, 64 positions' K rows in
        // flight per pass, each lane 4 dims of every 32; the int64 sums are
        // exact (|q| < 2^23, |k| < 2^31, dh <= 512).
        const uint32_t oc = threadIdx.x >> 3, e = threadIdx.x & 7;
        constexpr uint32_t NOCT = BD_THREADS / 8;
        if (KDB && dh <= 128) {
            // one 128-dim pass per position: the next pass's K rows are loaded
            // while this pass's products run
            int4 ka[4], kb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = 4 * e + 32 * u;
                ka[u] = (j < dh && oc < T) ? *reinterpret_cast<const int4*>(Kh + size_t(oc) * dh + j) : make_int4(0, 0, 0, 0);
                kb[u] = (j < dh && oc + NOCT < T) ? *reinterpret_cast<const int4*>(Kh + size_t(oc + NOCT) * dh + j) : make_int4(0, 0, 0, 0);
            }
            for (uint32_t b0 = 0; b0 < T; b0 += 2 * NOCT) {
                const uint32_t ta = b0 + oc, tb = ta + NOCT, na = ta + 2 * NOCT, nb = tb + 2 * NOCT;
                int4 ka2[4], kb2[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = 4 * e + 32 * u;
                    ka2[u] = (j < dh && na < T) ? *reinterpret_cast<const int4*>(Kh + size_t(na) * dh + j) : make_int4(0, 0, 0, 0);
                    kb2[u] = (j < dh && nb < T) ? *reinterpret_cast<const int4*>(Kh + size_t(nb) * dh + j) : make_int4(0, 0, 0, 0);
                }
                int64_t da = 0, db = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = 4 * e + 32 * u;
                    const int4 qq = j < dh ? *reinterpret_cast<const int4*>(q + j) : make_int4(0, 0, 0, 0);
                    da += mulw(qq.x, ka[u].x) + mulw(qq.y, ka[u].y) + mulw(qq.z, ka[u].z) + mulw(qq.w, ka[u].w);
                    db += mulw(qq.x, kb[u].x) + mulw(qq.y, kb[u].y) + mulw(qq.z, kb[u].z) + mulw(qq.w, kb[u].w);
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    da += __shfl_xor_sync(0xffffffffu, da, o);
                    db += __shfl_xor_sync(0xffffffffu, db, o);
                }
                if (e == 0) {
                    if (ta < T) S[ta] = mul16(da >> 16, inv_scale);
                    if (tb < T) S[tb] = mul16(db >> 16, inv_scale);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) ka[u] = ka2[u], kb[u] = kb2[u];
            }
        } else
        for (uint32_t b0 = 0; b0 < T; b0 += 2 * NOCT) {
            const uint32_t ta = b0 + oc, tb = ta + NOCT;
            int64_t da = 0, db = 0;
            for (uint32_t c0 = 0; c0 < dh; c0 += 128) {
                int4 ka[4], kb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = c0 + 4 * e + 32 * u;
                    ka[u] = (j < dh && ta < T) ? *reinterpret_cast<const int4*>(Kh + size_t(ta) * dh + j) : make_int4(0, 0, 0, 0);
                    kb[u] = (j < dh && tb < T) ? *reinterpret_cast<const int4*>(Kh + size_t(tb) * dh + j) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = c0 + 4 * e + 32 * u;
                    const int4 qq = j < dh ? *reinterpret_cast<const int4*>(q + j) : make_int4(0, 0, 0, 0);
                    da += mulw(qq.x, ka[u].x) + mulw(qq.y, ka[u].y) + mulw(qq.z, ka[u].z) +
                          mulw(qq.w, ka[u].w);
                    db += mulw(qq.x, kb[u].x) + mulw(qq.y, kb[u].y) + mulw(qq.z, kb[u].z) +
                          mulw(qq.w, kb[u].w);
                }
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                da += __shfl_xor_sync(0xffffffffu, da, o);
                db += __shfl_xor_sync(0xffffffffu, db, o);
            }
            if (e == 0) {
                if (ta < T) S[ta] = mul16(da >> 16, inv_scale);
                if (tb < T) S[tb] = mul16(db >> 16, inv_scale);
            }
        }
        __syncthreads();
        softmax_strip_fast(S, T, lut, red);  // ends with a barrier
        // PV: thread = (4-dim quad, position slice), 8 V rows in flight;
        // p <= 2^16 and |v| < 2^31: floor(p v / 2^16) is one exact 64-bit
        // product (mul16_prob's int32 case)
        const uint32_t nq = dh / 4, slices = BD_THREADS / nq;
        const uint32_t jq = threadIdx.x % nq, sl = threadIdx.x / nq;
        int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        if (sl < slices) {
            constexpr int U = 8;
            for (uint32_t p = sl; p < T; p += U * slices) {
                int4 vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t tt = p + u * slices;
                    vv[u] = tt < T ? *reinterpret_cast<const int4*>(Vh + size_t(tt) * dh + 4 * jq) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t tt = p + u * slices;
                    const int64_t pr = tt < T ? S[tt] : 0;
                    a0 += mulw(int32_t(pr), vv[u].x) >> 16;  // pr <= 2^16
                    a1 += mulw(int32_t(pr), vv[u].y) >> 16;
                    a2 += mulw(int32_t(pr), vv[u].z) >> 16;
                    a3 += mulw(int32_t(pr), vv[u].w) >> 16;
                }
            }
        }
        part[4 * threadIdx.x + 0] = uint64_t(a0);
        part[4 * threadIdx.x + 1] = uint64_t(a1);
        part[4 * threadIdx.x + 2] = uint64_t(a2);
        part[4 * threadIdx.x + 3] = uint64_t(a3);
        __syncthreads();
        for (uint32_t jj = threadIdx.x; jj < dh; jj += BD_THREADS) {
            const uint32_t qd = jj >> 2, z = jj & 3;
            uint64_t sum = 0;
            for (uint32_t s2 = 0; s2 < slices; ++s2) sum += part[4 * (s2 * nq + qd) + z];
            if (!put_sdigits(planes + size_t(t) * ldp + h * dh + jj, plane, int64_t(sum))) big = 1;
        }
        if (big) *wide = 1;
        return;
    }
    // four positions per warp per pass, their row loads in flight together
    for (uint32_t p0 = 4 * warp; p0 < T; p0 += 4 * (BD_THREADS / 32)) {
        int64_t d[4] = {0, 0, 0, 0};
        for (uint32_t j = 4 * lane; j < dh; j += 128) {
            int4 kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                kk[u] = p0 + u < T ? *reinterpret_cast<const int4*>(Kh + size_t(p0 + u) * dh + j) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                d[u] += int64_t(q[j]) * kk[u].x + int64_t(q[j + 1]) * kk[u].y + int64_t(q[j + 2]) * kk[u].z +
                        int64_t(q[j + 3]) * kk[u].w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
        if (lane == 0)
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (p0 + u < T) S[p0 + u] = mul16(d[u] >> 16, inv_scale);
    }
    __syncthreads();
    softmax_strip_inl(S, T, lut, red);  // ends with a barrier
    // out_j = sum_p mul16(p_p, V[p]_j): threads = (dim, position slice)
    const uint32_t slices = dh <= BD_THREADS ? BD_THREADS / dh : 1;
    const uint32_t j = threadIdx.x % dh, sl = threadIdx.x / dh;
    uint64_t acc = 0;
    if (sl < slices && j < dh) {
        uint32_t p = sl;
        for (; p + 3 * slices < T; p += 4 * slices) {  // four V rows in flight
            int32_t vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) vv[u] = Vh[size_t(p + u * slices) * dh + j];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += uint64_t(mul16_prob(S[p + u * slices], vv[u]));
        }
        for (; p < T; p += slices) acc += uint64_t(mul16_prob(S[p], Vh[size_t(p) * dh + j]));
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    for (uint32_t jj = threadIdx.x; jj < dh; jj += BD_THREADS) {
        uint64_t sum = 0;
        if (dh <= BD_THREADS) {
            for (uint32_t s2 = 0; s2 < slices; ++s2) sum += part[s2 * dh + jj];
        } else {  // dh > BD_THREADS: this thread sums dimension jj itself
            for (uint32_t p = 0; p < T; ++p) sum += uint64_t(mul16_prob(S[p], Vh[size_t(p) * dh + jj]));
        }
        const int64_t v = int64_t(sum);
        if (!put_sdigits(planes + size_t(t) * ldp + h * dh + jj, plane, v)) big = 1;
    }
    if (big) *wide = 1;
}

// Greedy selection per token row of the logits (proj/src/engine.cpp:113-120:
// largest value, lowest index on ties); feeds the next step: tok[t] = the
// choice, pos[t] += 1, and the choice is recorded at out[seq][step].
__global__ void __launch_bounds__(1024) bd_argmax_kernel(const int64_t* __restrict__ logits, uint32_t V,
                                                         uint32_t* tok, uint32_t* pos, const uint32_t* seq,
                                                         uint32_t* out, uint32_t max_new, uint32_t* step) {
    __shared__ int64_t sv[32];
    __shared__ uint32_t si[32];
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x;
    const int64_t* row = logits + size_t(t) * V;
    int64_t bv = INT64_MIN;
    uint32_t bi = 0xFFFFFFFFu;
    // 8 loads in flight per thread: the row (256 KB at 32000 vocab) is a few
    // memory round trips, not one per element
    constexpr int U = 8;
    for (uint32_t i0 = threadIdx.x; i0 < V; i0 += U * blockDim.x) {
        int64_t vals[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * blockDim.x;
            vals[u] = i < V ? row[i] : INT64_MIN;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * blockDim.x;
            if (i < V && better(vals[u], i, bv, bi)) {
                bv = vals[u];
                bi = i;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ov, oi, bv, bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < blockDim.x / 32; ++w)
            if (better(sv[w], si[w], bv, bi)) {
                bv = sv[w];
                bi = si[w];
            }
        const uint32_t s = *step;
        out[size_t(seq[t]) * max_new + s] = bi;
        tok[t] = bi;
        pos[t] += 1;
    }
}

__global__ void bd_step_kernel(uint32_t* step) {
    pdl_wait();
    *step += 1;
}

}  // namespace dimg::dev
