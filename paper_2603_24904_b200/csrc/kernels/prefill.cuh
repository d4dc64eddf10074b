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
__global__ void pf_embed_kernel(const uint32_t* __restrict__ tok, uint32_t n, const int8_t* __restrict__ E,
                                const int64_t* __restrict__ Es, uint32_t D, int64_t* __restrict__ x) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < size_t(n) * D;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(i / D), j = uint32_t(i % D);
        const uint32_t tk = tok[t];
        x[i] = int64_t(uint64_t(int64_t(E[size_t(tk) * D + j])) * uint64_t(Es[tk]));
    }
}

__device__ __forceinline__ void pf_put_limbs(uint8_t* p, size_t plane, int64_t v, uint32_t* wide) {
    if (!put_sdigits(p, plane, v)) *wide = 1;
}

// rmsnorm (proj/src/kernels.cpp:56-68) of every token row, written as the
// three limb planes of the next GEMM's B operand. One CTA per token; the row
// is loaded once into registers (all loads in flight together).
constexpr int PN_PER = 16;  // elements per thread held in registers (K <= 4096 with 256 threads)

__global__ void __launch_bounds__(256) pf_norm_limbs_kernel(const int64_t* __restrict__ x, uint32_t K,
                                                            const int64_t* __restrict__ gamma, int gamma_unit,
                                                            const int64_t* __restrict__ seeds, uint8_t* planes,
                                                            uint32_t rows_pad, uint32_t ldp, uint32_t* wide) {
    __shared__ u128 red[32];
    __shared__ int64_t s_r;
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t t = blockIdx.x;
    const int64_t* xr = x + size_t(t) * K;
    int64_t v[PN_PER];
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) {
        const uint32_t j = threadIdx.x + u * 256;
        v[u] = j < K ? xr[j] : 0;
    }
    u128 ss = 0;
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) ss += mul_full(v[u], v[u]);
    for (uint32_t j = threadIdx.x + PN_PER * 256; j < K; j += 256) ss += mul_full(xr[j], xr[j]);
    ss = block_sum_u128(ss, red);
    if (threadIdx.x == 0) {
        // usual case: the sum fits 63 bits and one u64 division is exact
        const int64_t ms = (ss >> 63) == 0 ? int64_t((uint64_t(ss) / K) >> 16) : int64_t((i128(ss) / i128(K)) >> 16);
        s_r = ms + 1 > 0 ? inv_sqrt_q16(ms + 1, seeds) : 0;
        if (ms + 1 <= 0) *wide = 1;  // the reference throws (domain_error): the exact path reports it
    }
    __syncthreads();
    const int64_t r = s_r;
    const size_t plane = size_t(rows_pad) * ldp;
    uint8_t* pr = planes + size_t(t) * ldp;
#pragma unroll
    for (int u = 0; u < PN_PER; ++u) {
        const uint32_t j = threadIdx.x + u * 256;
        if (j < K) {
            int64_t o = mul16(v[u], r);
            if (!gamma_unit) o = mul16(o, gamma[j]);
            pf_put_limbs(pr + j, plane, o, wide);
        }
    }
    for (uint32_t j = threadIdx.x + PN_PER * 256; j < K; j += 256) {
        int64_t o = mul16(xr[j], r);
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
                                  uint32_t* wide) {
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
    if (!fits_i32(k0) || !fits_i32(k1) || !fits_i32(v0) || !fits_i32(v1) || !b23(q0) || !b23(q1)) *wide = 1;
}

constexpr int PA_Q = 16;        // queries per CTA (two per warp)
constexpr int PA_CH = 64;       // cached positions per K / V chunk
constexpr int PA_THREADS = 256;

__host__ __device__ constexpr size_t pf_attn_smem(uint32_t dh, uint32_t n) {
    return size_t(PA_Q) * ((n + 3) & ~3u) * 4 + size_t(PA_CH) * dh * 4 + size_t(PA_Q) * dh * 4;
}

// Causal attention (proj/src/kernels.cpp:117-177) of n queries against the
// cache of positions <= each query, exact:
//   scores: int64 sums of int32 products (|q| < 2^23, |k| < 2^31, dh <= 512
//           keep every partial sum below 2^63), then mul16(dot >> 16, inv);
//   softmax: the LUT weights and truncating division of softmax_q16;
//   PV: sum_p floor(p_p v_pj / 2^16) computed as
//       (sum_p p v - sum_p (p v mod 2^16)) / 2^16 -- both sums exact (int64,
//       and 16-bit remainders in 32 bits), the difference divisible by 2^16.
// grid = (H, ceil(n / PA_Q)); each warp owns two queries. Scores, then
// probabilities, live in shared memory as int32 (flagged if one does not
// fit). K chunks are stored as 4-dim quads [dh/4][PA_CH] so a lane reads
// 16 bytes per position; V chunks row-major. DPL = dims per lane in PV
// (dh <= 32 DPL). Output: limb planes of the attention vector (WO's B operand).
template <int DPL>
__global__ void __launch_bounds__(PA_THREADS) pf_attn_kernel(const int64_t* __restrict__ qkv, uint32_t n,
                                                             uint32_t D, uint32_t dh,
                                                             const int32_t* __restrict__ K32,
                                                             const int32_t* __restrict__ V32,
                                                             size_t head_stride, int64_t inv_scale,
                                                             const int64_t* __restrict__ lut_g, uint8_t* planes,
                                                             uint32_t rows_pad, uint32_t ldp, uint32_t* wide) {
    extern __shared__ __align__(16) uint8_t pa_smem[];
    __shared__ int64_t lut[257];
    const uint32_t h = blockIdx.x, q0 = blockIdx.y * PA_Q;
    const uint32_t npos = min(n, q0 + PA_Q);  // positions any query of this CTA sees
    const uint32_t ld = (n + 3) & ~3u, nq = dh / 4;
    int32_t* S = reinterpret_cast<int32_t*>(pa_smem);   // [PA_Q][ld]
    int4* KV = reinterpret_cast<int4*>(S + size_t(PA_Q) * ld);  // K: [nq][PA_CH] quads; V: [PA_CH][nq]
    int4* Q = KV + size_t(PA_CH) * nq;                   // [PA_Q][nq]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 257; i += PA_THREADS) lut[i] = lut_g[i];
    for (uint32_t i = threadIdx.x; i < PA_Q * nq; i += PA_THREADS) {
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
    const uint32_t ta = q0 + 2 * warp, tb = ta + 1;  // this warp's two queries
    const int4* qa = Q + (2 * warp) * nq;
    const int4* qb = qa + nq;
    int32_t* Sa = S + size_t(2 * warp) * ld;
    int32_t* Sb = Sa + ld;
    int big = 0;

    // scores (kernels.cpp:143-151): lane = positions c0 + lane, c0 + lane + 32
    for (uint32_t c0 = 0; c0 < npos; c0 += PA_CH) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < PA_CH * nq; i += PA_THREADS) {
            const uint32_t p = i / nq, jq = i % nq;
            KV[jq * PA_CH + p] = c0 + p < npos ? Kh[size_t(c0 + p) * nq + jq] : make_int4(0, 0, 0, 0);
        }
        __syncthreads();
        if (ta >= n || c0 > tb) continue;  // warp-uniform: nothing of this chunk is visible
        int64_t a0 = 0, a1 = 0, b0 = 0, b1 = 0;
#pragma unroll 4
        for (uint32_t jq = 0; jq < nq; ++jq) {
            const int4 x = qa[jq], y = qb[jq];
            const int4 k0 = KV[jq * PA_CH + lane], k1 = KV[jq * PA_CH + lane + 32];
            a0 += int64_t(x.x) * k0.x + int64_t(x.y) * k0.y + int64_t(x.z) * k0.z + int64_t(x.w) * k0.w;
            a1 += int64_t(x.x) * k1.x + int64_t(x.y) * k1.y + int64_t(x.z) * k1.z + int64_t(x.w) * k1.w;
            b0 += int64_t(y.x) * k0.x + int64_t(y.y) * k0.y + int64_t(y.z) * k0.z + int64_t(y.w) * k0.w;
            b1 += int64_t(y.x) * k1.x + int64_t(y.y) * k1.y + int64_t(y.z) * k1.z + int64_t(y.w) * k1.w;
        }
        const uint32_t p0 = c0 + lane, p1 = p0 + 32;
        if (p0 <= ta) {
            const int64_t v = mul16(a0 >> 16, inv_scale);
            big |= !fits_i32(v);
            Sa[p0] = int32_t(v);
        }
        if (p1 <= ta) {
            const int64_t v = mul16(a1 >> 16, inv_scale);
            big |= !fits_i32(v);
            Sa[p1] = int32_t(v);
        }
        if (tb < n && p0 <= tb) {
            const int64_t v = mul16(b0 >> 16, inv_scale);
            big |= !fits_i32(v);
            Sb[p0] = int32_t(v);
        }
        if (tb < n && p1 <= tb) {
            const int64_t v = mul16(b1 >> 16, inv_scale);
            big |= !fits_i32(v);
            Sb[p1] = int32_t(v);
        }
    }
    // softmax_q16 (kernels.cpp:90-107), one warp per query row
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
        const uint32_t t = u ? tb : ta;
        int32_t* R = u ? Sb : Sa;
        if (t >= n) continue;
        int32_t m = INT32_MIN;
        for (uint32_t p = lane; p <= t; p += 32) m = R[p] > m ? R[p] : m;
        m = __reduce_max_sync(0xffffffffu, m);
        uint32_t tot = 0;  // <= 2^16 per weight, n <= 2560 positions
        for (uint32_t p = lane; p <= t; p += 32) {
            const int64_t d = int64_t(m) - R[p];
            const int64_t w = exp_neg(d > 8 * ONE ? 8 * ONE : d, lut);
            R[p] = int32_t(w);
            tot += uint32_t(w);
        }
        const uint64_t total = __reduce_add_sync(0xffffffffu, tot);
        const uint64_t inv = ~0ull / total;
        for (uint32_t p = lane; p <= t; p += 32) {
            const uint64_t a = uint64_t(R[p]) << 16;
            uint64_t qv = __umul64hi(a, inv);
            qv += (a - qv * total) >= total;
            R[p] = int32_t(qv);  // <= 2^16
        }
    }
    // PV (kernels.cpp:153-159): lane owns dims lane * DPL ... + DPL - 1
    int64_t fa[DPL], fb[DPL];
    uint32_t ra[DPL], rb[DPL];
#pragma unroll
    for (int z = 0; z < DPL; ++z) fa[z] = fb[z] = 0, ra[z] = rb[z] = 0;
    const uint32_t jl = lane * DPL;  // first dim of this lane
    const bool lane_on = jl < dh;
    for (uint32_t c0 = 0; c0 < npos; c0 += PA_CH) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < PA_CH * nq; i += PA_THREADS) {
            const uint32_t p = i / nq, jq = i % nq;
            KV[p * nq + jq] = c0 + p < npos ? Vh[size_t(c0 + p) * nq + jq] : make_int4(0, 0, 0, 0);
        }
        __syncthreads();
        if (ta >= n || c0 > tb || !lane_on) continue;
        const uint32_t pend = min(uint32_t(PA_CH), min(npos, tb + 1) - c0);
        const int32_t* Vs = reinterpret_cast<const int32_t*>(KV);
#pragma unroll 2
        for (uint32_t pp = 0; pp < pend; ++pp) {
            const uint32_t p = c0 + pp;
            const int32_t pa = p <= ta ? Sa[p] : 0, pb = p <= tb && tb < n ? Sb[p] : 0;
            const int32_t* vr = Vs + pp * dh + jl;
#pragma unroll
            for (int z = 0; z < DPL; ++z) {
                const int32_t v = vr[z];
                fa[z] += int64_t(pa) * v;
                fb[z] += int64_t(pb) * v;
                ra[z] += (uint32_t(pa) * uint32_t(v)) & 0xFFFFu;  // low bits of the exact product
                rb[z] += (uint32_t(pb) * uint32_t(v)) & 0xFFFFu;
            }
        }
    }
    if (lane_on) {
        const size_t plane = size_t(rows_pad) * ldp;
#pragma unroll
        for (int z = 0; z < DPL; ++z) {
            const uint32_t j = jl + z;
            if (j >= dh) break;
            if (ta < n) pf_put_limbs(planes + size_t(ta) * ldp + h * dh + j, plane, (fa[z] - int64_t(ra[z])) >> 16, wide);
            if (tb < n) pf_put_limbs(planes + size_t(tb) * ldp + h * dh + j, plane, (fb[z] - int64_t(rb[z])) >> 16, wide);
        }
    }
    if (big) *wide = 1;
}

}  // namespace dimg::dev
