// Prefill of a prompt's first n tokens with the tensor-core limb GEMM
// (tc_gemm.cuh): all n tokens go through each layer together instead of one
// forward step at a time. The arithmetic is the reference's, element for
// element (proj/src/engine.cpp:80-102 per token): embedding, rmsnorm, the
// dense products, RoPE, the causal attention with the exact LUT softmax, the
// residual clamps. Only the KV cache is kept: the decode kernel then runs the
// last prompt token and the continuation.
//
// Every kernel here flags (*wide = 1) any value outside the range its fast
// representation covers (3 byte limbs, int32 K/V and scores, |q| < 2^23);
// the engine then discards the result and prefills with the decode kernel,
// which is exact for every input.
#pragma once

#include <cstdint>

#include "attention.cuh"
#include "q16.cuh"

namespace dimg::dev {

// x[t] = embed_token(tok[t]) (proj/src/engine.cpp:10-19)
// The residual stream is int32 in the prefill and batch paths: every residual
// epilogue clamps it to +-2^24; an embedding value outside int32 (a model
// with huge embedding scales) sets *wide and the exact path takes over.
__global__ void pf_embed_kernel(const uint32_t* __restrict__ tok, uint32_t n, const int8_t* __restrict__ E,
                                const int64_t* __restrict__ Es, uint32_t D, int32_t* __restrict__ x, uint32_t* wide) {
    pdl_launch_dependents();
    pdl_wait();
    int bad = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < size_t(n) * D;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(i / D), j = uint32_t(i % D);
        const uint32_t tk = tok[t];
        const int64_t v = int64_t(uint64_t(int64_t(E[size_t(tk) * D + j])) * uint64_t(Es[tk]));
        bad |= !fits_i32(v);
        x[i] = int32_t(v);
    }
    if (bad) *wide = 1;
}

__device__ __forceinline__ void pf_put_limbs(uint8_t* p, size_t plane, int64_t v, uint32_t* wide) {
    if (!put_sdigits(p, plane, v)) *wide = 1;
}

// rmsnorm (proj/src/kernels.cpp:56-68) of every token row, written as the
// three limb planes of the next GEMM's B operand. One CTA per token; the row
// is loaded once into registers (all loads in flight together).
constexpr int PN_PER = 16;  // elements per thread held in registers (K <= 4096 with 256 threads)

__global__ void __launch_bounds__(256) pf_norm_limbs_kernel(const int32_t* __restrict__ x, uint32_t K,
                                                            const int64_t* __restrict__ gamma, int gamma_unit,
                                                            const int64_t* __restrict__ seeds, uint8_t* planes,
                                                            uint32_t rows_pad, uint32_t ldp, uint32_t* wide) {
    __shared__ u128 red[32];
    __shared__ int64_t s_r;
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x;
    const int32_t* xr = x + size_t(t) * K;
    int64_t v[PN_PER];
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) {
        const uint32_t j = threadIdx.x + u * 256;
        v[u] = j < K ? xr[j] : 0;
    }
    // |x| <= 2^24 (every row after a residual clamp): x^2 < 2^48 summed in
    // 21-bit chunks with REDUX, as bd_norm1k_kernel; otherwise (an embedding
    // row beyond 2^24) the 128-bit sums
    int small = 1;
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) small &= v[u] >= -(int64_t(1) << 24) && v[u] <= (int64_t(1) << 24);
    small = __syncthreads_and(small && K <= PN_PER * 256);
    u128 ss = 0;
    if (small) {
        uint32_t c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
        for (int u = 0; u < PN_PER; ++u) {
            const uint64_t q2 = uint64_t(mulw(int32_t(v[u]), int32_t(v[u])));
            c0 += uint32_t(q2) & 0x1FFFFFu;
            c1 += uint32_t(q2 >> 21) & 0x1FFFFFu;
            c2 += uint32_t(q2 >> 42);
        }
        // per-warp sums < 32 * 16 * 2^21 = 2^30: exact 32-bit REDUX
        c0 = __reduce_add_sync(0xffffffffu, c0);
        c1 = __reduce_add_sync(0xffffffffu, c1);
        c2 = __reduce_add_sync(0xffffffffu, c2);
        uint64_t* sw = reinterpret_cast<uint64_t*>(red);  // [8 warps][3]
        if ((threadIdx.x & 31) == 0) {
            sw[3 * (threadIdx.x >> 5)] = c0;
            sw[3 * (threadIdx.x >> 5) + 1] = c1;
            sw[3 * (threadIdx.x >> 5) + 2] = c2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t0 += sw[3 * w], t1 += sw[3 * w + 1], t2 += sw[3 * w + 2];
            ss = u128(t0) + (u128(t1) << 21) + (u128(t2) << 42);
        }
    } else {
#pragma unroll
        for (int u = 0; u < PN_PER; ++u) ss += mul_full(v[u], v[u]);
        for (uint32_t j = threadIdx.x + PN_PER * 256; j < K; j += 256) ss += mul_full(int64_t(xr[j]), int64_t(xr[j]));
        ss = block_sum_u128(ss, red);
    }
    if (threadIdx.x == 0) {
        // usual case: the sum fits 63 bits and one u64 division is exact
        const int64_t ms = (ss >> 63) != 0       ? int64_t((i128(ss) / i128(K)) >> 16)
                           : (K & (K - 1)) == 0 ? int64_t((uint64_t(ss) >> (__ffs(K) - 1)) >> 16)
                                                : int64_t((uint64_t(ss) / K) >> 16);
        s_r = ms + 1 > 0 ? inv_sqrt_q16(ms + 1, seeds) : 0;
        if (ms + 1 <= 0) *wide = 1;  // the reference throws (domain_error): the exact path reports it
    }
    __syncthreads();
    const int64_t r = s_r;
    const size_t plane = size_t(rows_pad) * ldp;
    uint8_t* pr = planes + size_t(t) * ldp;
    const bool r32 = small && r >= 0 && r <= (int64_t(1) << 24);  // mul16(x, r) as one IMAD.WIDE
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) {
        const uint32_t j = threadIdx.x + u * 256;
        if (j < K) {
            int64_t o = r32 ? mulw(int32_t(v[u]), int32_t(r)) >> 16 : mul16(v[u], r);
            if (!gamma_unit) o = mul16(o, gamma[j]);
            pf_put_limbs(pr + j, plane, o, wide);
        }
    }
    for (uint32_t j = threadIdx.x + PN_PER * 256; j < K; j += 256) {
        int64_t o = mul16(int64_t(xr[j]), r);
        if (!gamma_unit) o = mul16(o, gamma[j]);
        pf_put_limbs(pr + j, plane, o, wide);
    }
}

// RoPE of q and k (proj/src/kernels.cpp:70-82, 137-138) for every token and
// head; the KV append (:139-142) at position t: int64 cache, int32 mirror.
// q' overwrites q in place. grid = (n, H), block = dh / 2 threads (<= 1024).
__global__ void pf_rope_kv_kernel(int64_t* __restrict__ qkv, uint32_t D, uint32_t dh,
                                  const int64_t* __restrict__ rc, const int64_t* __restrict__ rs,
                                  int64_t* K64, int64_t* V64, int32_t* K32, int32_t* V32, size_t head_stride,
                                  uint32_t* wide, int8_t* kdig, uint32_t n_pad, uint32_t* kd4) {
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x, h = blockIdx.y, half = dh / 2, i = threadIdx.x;
    int64_t* q = qkv + size_t(t) * 3 * D + size_t(h) * dh;
    const int64_t* k = q + D;
    const int64_t* v = q + 2 * D;
    const size_t kv = size_t(h) * head_stride + size_t(t) * dh;
    const int64_t c = rc[size_t(t) * half + i], s = rs[size_t(t) * half + i];
    int64_t q0, q1, k0, k1;
    rope_pair(q[i], q[i + half], c, s, q0, q1);
    rope_pair(k[i], k[i + half], c, s, k0, k1);
    const int64_t v0 = v[i], v1 = v[i + half];
    __syncthreads();  // q is rewritten in place
    q[i] = q0;
    q[i + half] = q1;
    K64[kv + i] = k0;
    K64[kv + i + half] = k1;
    V64[kv + i] = v0;
    V64[kv + i + half] = v1;
    K32[kv + i] = int32_t(k0);
    K32[kv + i + half] = int32_t(k1);
    V32[kv + i] = int32_t(v0);
    V32[kv + i + half] = int32_t(v1);
    const auto b23 = [](int64_t a) { return a >= -(int64_t(1) << 23) && a < (int64_t(1) << 23); };
    bool bad = !fits_i32(k0) || !fits_i32(k1) || !fits_i32(v0) || !fits_i32(v1) || !b23(q0) || !b23(q1);
    if (kdig) {  // the key's 4 signed digit planes for the tensor-core scores (pf_scores.cuh)
        const int64_t kk[2] = {k0, k1};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            int64_t r = kk[e];
            int8_t* dst = kdig + (size_t(h) * 4 * n_pad + t) * dh + i + e * half;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int64_t dg = int8_t(r);
                dst[size_t(d) * n_pad * dh] = int8_t(dg);
                r = (r - dg) >> 8;
            }
            dst[size_t(3) * n_pad * dh] = int8_t(r);
            bad |= r < -128 || r > 127;
            if (r != 0) atomicOr(kd4, 1u);  // this layer's keys need the 4th digit plane
        }
    }
    if (bad) *wide = 1;
}

constexpr int PA_Q = 32;        // queries per CTA
constexpr int PA_QW = 4;        // queries per warp
constexpr int PA_CH = 64;       // cached positions per K / V chunk
constexpr int PA_THREADS = 256;
static_assert(PA_Q == PA_QW * PA_THREADS / 32, "every warp owns PA_QW queries");

// shared memory: K/V chunk double buffer + the CTA's queries + a double
// buffer of probability chunks ([query][position])
__host__ __device__ constexpr size_t pf_attn_smem(uint32_t dh) {
    return 2 * size_t(PA_CH) * dh * 4 + size_t(PA_Q) * dh * 4 + 2 * size_t(PA_CH) * PA_Q * 4;
}
// global score / probability strips, [H][n rounded to PA_Q][ld] int32
__host__ __device__ constexpr size_t pf_attn_strip_elems(uint32_t H, uint32_t n) {
    return size_t(H) * ((n + PA_Q - 1) / PA_Q * PA_Q) * ((n + 3) & ~3u);
}

__device__ __forceinline__ void pa_cp16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(
                     __cvta_generic_to_shared(dst))),
                 "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void pa_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void pa_cp_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void pa_cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Causal attention (proj/src/kernels.cpp:117-177) of n queries against the
// cache of positions <= each query, exact:
//   scores: int64 sums of int32 products (|q| < 2^23, |k| < 2^31, dh <= 512
//           keep every partial sum below 2^63), then mul16(dot >> 16, inv);
//   softmax: the LUT weights and truncating division of softmax_q16;
//   PV: sum_p floor(p_p v_pj / 2^16) computed as
//       (sum_p p v - sum_p (p v mod 2^16)) / 2^16 -- both sums exact (int64,
//       and 16-bit remainders in 32 bits), the difference divisible by 2^16.
// grid = (H, ceil(n / PA_Q)); each warp owns PA_QW consecutive queries, so
// every K / V value read from shared memory feeds PA_QW queries. The score
// (then probability) strips live in a global scratch that stays in L2: a
// lane writes and re-reads the same positions (p mod 32 = lane), and the PV
// pass stages one chunk of them in shared memory after a CTA barrier. K / V
// chunks are double-buffered with cp.async (K as 4-dim quads [dh/4][PA_CH]
// so a lane reads 16 bytes per position; V row-major). DPL = dims per lane in
// PV (dh <= 32 DPL). Output: digit planes of the attention vector (WO's B
// operand); values outside the fast representation set *wide.
// TCPV: only the per-product half here, and only modulo 2^16: fl_out
// [H][n][dh] gets U = sum_p ((P v_p mod 2^32) >> 16) = sum_p ((P vh_p +
// floor(P vl_p / 2^16)) mod 2^16) -- one IMAD + one LEA.HI per product, no
// vl mask. pf_pv_kernel (pf_pv.cuh) computes the linear half T = sum_p P vh_p
// on the tensor cores; F = sum_p floor(P vl_p / 2^16) < sum_p P <= 2^16, so
// F = (U - T) mod 2^16 exactly, and the output is T + F.
template <int DPL, bool TCPV>
__global__ void __launch_bounds__(PA_THREADS, 2) pf_attn_kernel(const int64_t* __restrict__ qkv, uint32_t n,
                                                                uint32_t D, uint32_t dh,
                                                                const int32_t* __restrict__ K32,
                                                                const int32_t* __restrict__ V32,
                                                                size_t head_stride, int64_t inv_scale,
                                                                const int64_t* __restrict__ lut_g, int32_t* strips,
                                                                uint8_t* planes, uint32_t rows_pad, uint32_t ldp,
                                                                uint32_t* wide, bool scores_ready, int32_t* fl_out) {
    extern __shared__ __align__(16) uint8_t pa_smem[];
    __shared__ int64_t lut[257];
    __shared__ int32_t lut32[258];  // [0] = e[0] (the cell-256 end), [1 + i] = e[i]
    const uint32_t h = blockIdx.x, q0 = blockIdx.y * PA_Q;
    const uint32_t npos = min(n, q0 + PA_Q);  // positions any query of this CTA sees
    const uint32_t ld = (n + 3) & ~3u, nq = dh / 4, chunk_q = PA_CH * nq;
    int4* KV = reinterpret_cast<int4*>(pa_smem);          // 2 x chunk: K [nq][PA_CH] quads / V [PA_CH][nq]
    int4* Q = KV + 2 * size_t(chunk_q);                     // [PA_Q][nq]
    int32_t* Ps = reinterpret_cast<int32_t*>(Q + size_t(PA_Q) * nq);  // [PA_Q][PA_CH]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_launch_dependents();
    for (int i = threadIdx.x; i < 257; i += PA_THREADS) {  // constant: before the wait
        lut[i] = lut_g[i];
        lut32[i + 1] = int32_t(lut_g[i]);
    }
    if (threadIdx.x == 0) lut32[0] = int32_t(lut_g[0]);
    pdl_wait();
    for (uint32_t i = threadIdx.x; i < PA_Q * nq && !scores_ready; i += PA_THREADS) {
        const uint32_t qi = i / nq, j = 4 * (i % nq);
        int4 v = make_int4(0, 0, 0, 0);
        if (q0 + qi < n) {
            const int64_t* qr = qkv + size_t(q0 + qi) * 3 * D + size_t(h) * dh + j;
            v = make_int4(int32_t(qr[0]), int32_t(qr[1]), int32_t(qr[2]), int32_t(qr[3]));
        }
        Q[i] = v;
    }
    const int4* Kh = reinterpret_cast<const int4*>(K32 + size_t(h) * head_stride);
    const int4* Vh = reinterpret_cast<const int4*>(V32 + size_t(h) * head_stride);
    const uint32_t tw = q0 + PA_QW * warp;  // this warp's first query
    int32_t* Sw = strips + ((size_t(h) * gridDim.y + blockIdx.y) * PA_Q + PA_QW * warp) * ld;  // its rows
    const uint32_t nch = (npos + PA_CH - 1) / PA_CH;
    int big = 0;

    // ---- scores (kernels.cpp:143-151): lane = positions c0 + lane, c0 + lane + 32
    auto load_k = [&](uint32_t c, int4* dst) {
        const uint32_t c0 = c * PA_CH;
        for (uint32_t i = threadIdx.x; i < chunk_q; i += PA_THREADS) {
            const uint32_t p = i / nq, jq = i % nq;
            const bool ok = c0 + p < npos;
            pa_cp16(dst + jq * PA_CH + p, Kh + size_t(ok ? c0 + p : 0) * nq + jq, ok);
        }
        pa_cp_commit();
    };
    int32_t mx[PA_QW];
#pragma unroll
    for (int u = 0; u < PA_QW; ++u) mx[u] = INT32_MIN;
    if (scores_ready) {  // pf_scores_kernel wrote the strips: only the row maxima
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PA_QW; ++u) {
            const uint32_t t = tw + u;
            if (t < n)
                for (uint32_t p = lane; p <= t; p += 32) mx[u] = Sw[size_t(u) * ld + p] > mx[u] ? Sw[size_t(u) * ld + p] : mx[u];
        }
    }
    if (!scores_ready) load_k(0, KV);
    for (uint32_t c = 0; c < nch && !scores_ready; ++c) {
        int4* cur = KV + (c & 1) * chunk_q;
        if (c + 1 < nch) {
            load_k(c + 1, KV + ((c + 1) & 1) * chunk_q);
            pa_cp_wait_prev();
        } else {
            pa_cp_wait_all();
        }
        __syncthreads();  // chunk c visible to every warp
        const uint32_t c0 = c * PA_CH;
        if (tw < n && c0 <= tw + PA_QW - 1) {  // warp-uniform: part of this chunk is visible
            int64_t acc[PA_QW][2];
#pragma unroll
            for (int u = 0; u < PA_QW; ++u) acc[u][0] = acc[u][1] = 0;
            const int4* qw = Q + size_t(PA_QW * warp) * nq;
#pragma unroll 2
            for (uint32_t jq = 0; jq < nq; ++jq) {
                const int4 k0 = cur[jq * PA_CH + lane], k1 = cur[jq * PA_CH + lane + 32];
#pragma unroll
                for (int u = 0; u < PA_QW; ++u) {
                    const int4 x = qw[u * nq + jq];
                    acc[u][0] += int64_t(x.x) * k0.x + int64_t(x.y) * k0.y + int64_t(x.z) * k0.z + int64_t(x.w) * k0.w;
                    acc[u][1] += int64_t(x.x) * k1.x + int64_t(x.y) * k1.y + int64_t(x.z) * k1.z + int64_t(x.w) * k1.w;
                }
            }
#pragma unroll
            for (int u = 0; u < PA_QW; ++u) {
                const uint32_t t = tw + u;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t p = c0 + lane + 32 * e;
                    if (t < n && p <= t) {
                        const int64_t v = mul16(acc[u][e] >> 16, inv_scale);
                        big |= !fits_i32(v);
                        const int32_t v32 = int32_t(v);
                        Sw[size_t(u) * ld + p] = v32;
                        mx[u] = v32 > mx[u] ? v32 : mx[u];
                    }
                }
            }
        }
        __syncthreads();  // everyone done with chunk c before it is overwritten
    }

    // ---- softmax_q16 (kernels.cpp:90-107) over each of the warp's rows; a lane
    // re-reads only positions it wrote (p = lane mod 32)
#pragma unroll 1
    for (int u = 0; u < PA_QW; ++u) {
        const uint32_t t = tw + u;
        if (t >= n) break;
        int32_t* R = Sw + size_t(u) * ld;
        const int32_t m = __reduce_max_sync(0xffffffffu, mx[u]);
        // all in 32 bits: m - score < 2^32 (int32 scores), and the LUT
        // weights and their interpolation (< 2^16 x 2^11) fit
        uint32_t tot = 0;  // <= 2^16 per weight, n <= 2560 positions
        for (uint32_t p = lane; p <= t; p += 32) tot += exp_neg32(min(uint32_t(m - R[p]), uint32_t(8 * ONE)), lut32);
        const uint32_t total = __reduce_add_sync(0xffffffffu, tot);
        // floor(w 2^16 / total) <= 2^16: a float estimate within one of the
        // quotient (three roundings of 2^-24), fixed by the exact remainder,
        // which lies in (-total, 2 total) and so is exact as an int32 even
        // though w 2^16 and q total wrap mod 2^32
        const float scale = 65536.0f / float(total);
        for (uint32_t p = lane; p <= t; p += 32) {
            const uint32_t w = exp_neg32(min(uint32_t(m - R[p]), uint32_t(8 * ONE)), lut32);
            uint32_t q = uint32_t(float(w) * scale);
            const int32_t r = int32_t((w << 16) - q * total);
            q -= r < 0;
            q += r >= int32_t(total);
            R[p] = int32_t(q);
        }
        // the positions after t that the warp's PV loop reads for this row
        // (up to its last query) must hold probability 0: the probability
        // chunks are copied into shared memory unmasked
        const uint32_t pe = min(npos, tw + PA_QW);
        if (t + 1 + lane < pe) R[t + 1 + lane] = 0;
    }

    // ---- PV (kernels.cpp:153-159): lane owns dims lane * DPL ... + DPL - 1
    // floor(p v / 2^16) = p vh + floor(p vl / 2^16) with v = vh 2^16 + vl,
    // vl in [0, 2^16): p <= 2^16 makes p vl < 2^32 (one 32-bit product), and
    // sum_t p_t vh_t is within int32 (sum p <= 2^16, |vh| <= 2^15). Two 32-bit
    // multiplies per product, no 64-bit arithmetic.
    int32_t fh[PA_QW][DPL];
    uint32_t fl[PA_QW][DPL];
#pragma unroll
    for (int u = 0; u < PA_QW; ++u)
#pragma unroll
        for (int z = 0; z < DPL; ++z) fh[u][z] = 0, fl[u][z] = 0;
    const uint32_t jl = lane * DPL;  // first dim of this lane
    const bool lane_on = jl < dh;
    const int32_t* Sc = strips + (size_t(h) * gridDim.y + blockIdx.y) * PA_Q * ld;  // the CTA's rows
    auto load_v = [&](uint32_t c, int4* dst) {
        const uint32_t c0 = c * PA_CH;
        for (uint32_t i = threadIdx.x; i < chunk_q; i += PA_THREADS) {
            const uint32_t p = i / nq, jq = i % nq;
            const bool ok = c0 + p < npos;
            pa_cp16(dst + p * nq + jq, Vh + size_t(ok ? c0 + p : 0) * nq + jq, ok);
        }
        pa_cp_commit();
    };
    // this chunk's probabilities, [query][position], copied with V: every
    // position a warp reads is <= its last query and < npos, and holds 0
    // past each row's own query (softmax pass); rows of queries >= n are
    // never used
    auto load_p = [&](uint32_t c, int32_t* dst) {
        const uint32_t c0 = c * PA_CH;
        for (uint32_t i = threadIdx.x; i < PA_Q * (PA_CH / 4); i += PA_THREADS) {
            const uint32_t qi = i / (PA_CH / 4), p = c0 + 4 * (i % (PA_CH / 4));
            const bool ok = p < ld;  // ld % 4 == 0: the 16 bytes lie inside the row
            pa_cp16(dst + qi * PA_CH + (p - c0), Sc + size_t(qi) * ld + (ok ? p : 0), ok);
        }
    };
    __syncthreads();  // every row's probabilities written (global, same CTA)
    load_p(0, Ps);
    load_v(0, KV);
    for (uint32_t c = 0; c < nch; ++c) {
        const int4* cur = KV + (c & 1) * chunk_q;
        const int32_t* Pc = Ps + (c & 1) * (PA_Q * PA_CH);
        const uint32_t c0 = c * PA_CH;
        if (c + 1 < nch) {
            load_p(c + 1, Ps + ((c + 1) & 1) * (PA_Q * PA_CH));
            load_v(c + 1, KV + ((c + 1) & 1) * chunk_q);
            pa_cp_wait_prev();
        } else {
            pa_cp_wait_all();
        }
        __syncthreads();
        if (tw < n && c0 <= tw + PA_QW - 1 && lane_on) {
            const uint32_t pend = min(uint32_t(PA_CH), min(npos, tw + PA_QW) - c0);
            const int32_t* Vs = reinterpret_cast<const int32_t*>(cur);
#pragma unroll 2
            for (uint32_t pp = 0; pp < pend; ++pp) {
                int32_t pq[PA_QW];
#pragma unroll
                for (int u = 0; u < PA_QW; ++u) pq[u] = Pc[(PA_QW * warp + u) * PA_CH + pp];  // broadcast
                int32_t vv[DPL];
                if constexpr (DPL >= 4) {
#pragma unroll
                    for (int z = 0; z < DPL; z += 4) {
                        const int4 q4 = *reinterpret_cast<const int4*>(Vs + pp * dh + jl + z);
                        vv[z] = q4.x, vv[z + 1] = q4.y, vv[z + 2] = q4.z, vv[z + 3] = q4.w;
                    }
                } else {
#pragma unroll
                    for (int z = 0; z < DPL; ++z) vv[z] = Vs[pp * dh + jl + z];
                }
#pragma unroll
                for (int z = 0; z < DPL; ++z) {
                    if constexpr (TCPV) {
                        // (P v mod 2^32) >> 16 = (P vh + floor(P vl / 2^16)) mod 2^16
                        const uint32_t vu = uint32_t(vv[z]);
#pragma unroll
                        for (int u = 0; u < PA_QW; ++u) fl[u][z] += (uint32_t(pq[u]) * vu) >> 16;
                    } else {
                        const int32_t vh = vv[z] >> 16;
                        const uint32_t vl = uint32_t(vv[z]) & 0xFFFFu;
#pragma unroll
                        for (int u = 0; u < PA_QW; ++u) {
                            fh[u][z] += pq[u] * vh;
                            fl[u][z] += (uint32_t(pq[u]) * vl) >> 16;
                        }
                    }
                }
            }
        }
        __syncthreads();  // chunk c and Ps consumed
    }
    if constexpr (TCPV) {
        if (lane_on) {
#pragma unroll
            for (int u = 0; u < PA_QW; ++u) {
                const uint32_t t = tw + u;
                if (t >= n) break;
                int32_t* dst = fl_out + (size_t(h) * n + t) * dh + jl;
#pragma unroll
                for (int z = 0; z < DPL; ++z)
                    if (jl + z < dh) dst[z] = int32_t(fl[u][z]);
            }
        }
        if (big) *wide = 1;
        return;
    }
    if (lane_on) {
        const size_t plane = size_t(rows_pad) * ldp;
#pragma unroll
        for (int u = 0; u < PA_QW; ++u) {
            const uint32_t t = tw + u;
            if (t >= n) break;
#pragma unroll
            for (int z = 0; z < DPL; ++z) {
                const uint32_t j = jl + z;
                if (j < dh) pf_put_limbs(planes + size_t(t) * ldp + h * dh + j, plane, int64_t(fh[u][z]) + fl[u][z], wide);
            }
        }
    }
    if (big) *wide = 1;
}

}  // namespace dimg::dev
