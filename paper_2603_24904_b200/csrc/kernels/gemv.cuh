// Decode GEMV for the reference's dense layers (proj/src/kernels.cpp:18-30):
//
//     out[r] = (int128(sum_j w[r,j] * x[j]) * s[r]) >> 16
//
// with w int8 and x int64 Q16. The int64 activations are split EXACTLY into
// byte limbs, x = sum_k l_k 2^(8k) (l_k unsigned bytes, the top limb signed),
// so each limb is a plain int8 operand: DP4A (s8 x u8 / s8 x s8) accumulates
// per-limb int32 partial sums, which are recombined in int64 with the limb
// shifts. Integer addition is associative, so the result is bit-identical to
// the reference's sequential int64 loop, wrap-around included.
//   * 3 limbs when every |x| < 2^23 (all real activations: max measured
//     2^18.3 at 7B);
//   * 8 limbs otherwise (any int64; still exact mod 2^64 like the reference).
// The choice is made per CTA from the vector it just built, so it is uniform
// and needs no host round trip.
//
// The input vector is built in the prologue straight into shared memory:
//   MODE_PLAIN  x as given (attention output, FFN hidden)
//   MODE_NORM   rmsnorm(x, gamma) (proj/src/kernels.cpp:56-68), recomputed per
//               CTA from the L2-resident residual stream: no separate norm
//               kernel, no round trip through HBM
//   MODE_EMBED  embed_token (proj/src/engine.cpp:10-19) then rmsnorm; CTA 0
//               also writes the embedding to the residual stream
// Weights stream from HBM once, 16 B per lane per row (LDG.128, no L1
// allocate); each CTA owns a contiguous, balanced row range (grid = SMs x k)
// and its warps take R-row groups so one shared-memory limb read feeds R rows.
//
// Epilogues fuse the reference's next elementwise step:
//   EPI_STORE   y[r] = scaled                       (q/k/v projections)
//   EPI_RESID   x[r] = clamp(x[r] + scaled)         (wo, w_down + residual_add_clamp)
//   EPI_SILU    h[i] = mul16(silu(g_i), u_i)        (gate/up rows interleaved, ffn_silu)
//   EPI_ARGMAX  logits + greedy argmax (lowest index on ties), the last CTA
//               appends the selected token on the device (select_greedy)
//   EPI_RAW     y[r] = pre-scale int64 accumulator  (tensor-parallel partials)
#pragma once

#include <cstdint>

#include "q16.cuh"

namespace dimg::dev {

enum { EPI_STORE = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_ARGMAX = 3, EPI_RAW = 4 };
enum { MODE_PLAIN = 0, MODE_NORM = 1, MODE_EMBED = 2 };

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;

// Device control block of a session (one per sequence).
struct Ctl {
    uint32_t pos;           // position processed by the next step
    uint32_t logit_base;    // first position whose logits are kept
    uint32_t keep_cap;      // capacity of the kept-logits buffer (vectors)
    uint32_t argmax_count;  // CTAs of the lm_head that finished this step
    uint32_t err;           // bit 0: inv_sqrt domain error (ms + 1 <= 0)
    uint32_t serr;          // bit 1: sampling's exp_neg_lut domain error (kept across steps)
    uint32_t pad[2];
    unsigned long long stats[4];  // [0] CTAs on the 8-limb path, [1] attention parts on the int64 KV path
};

struct ArgPart {
    int64_t v;
    uint32_t idx;
    uint32_t pad;
};

struct GemvArgs {
    const int8_t* W;          // [rows][Kp]
    const int64_t* scales;    // [rows]
    uint32_t rows, K, Kp;
    const int64_t* x;         // [K] input (MODE_PLAIN / MODE_NORM)
    const int64_t* gamma;     // [K] (MODE_NORM / MODE_EMBED)
    const int8_t* embd;       // [V][K] (MODE_EMBED)
    const int64_t* embd_scales;
    const uint32_t* tokens;   // token ring (MODE_EMBED reads tokens[pos])
    int64_t* x_out;           // MODE_EMBED: CTA 0 writes the embedding here
    int64_t* y;               // epilogue output
    int64_t* logits;          // EPI_ARGMAX: [keep_cap + 1][rows] (last row = scratch)
    ArgPart* parts;           // EPI_ARGMAX: one per CTA
    uint32_t* tokens_out;     // EPI_ARGMAX: tokens[pos + 1] = argmax
    Ctl* ctl;
    const int64_t* exp_lut;   // [257]
    const int64_t* seeds;     // [64]
};

__device__ __forceinline__ int4 ldg_stream(const int8_t* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// d += dot4(a as s8x4, b as u8x4) / dot4(a s8x4, b s8x4)
__device__ __forceinline__ int32_t dp4a_su(int32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int32_t dp4a_ss(int32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Contiguous balanced row range of this CTA, in units of `unit` rows.
__device__ __forceinline__ void cta_rows(uint32_t rows, uint32_t unit, uint32_t& lo, uint32_t& hi) {
    uint32_t units = (rows + unit - 1) / unit;
    uint64_t a = uint64_t(units) * blockIdx.x / gridDim.x;
    uint64_t b = uint64_t(units) * (blockIdx.x + 1) / gridDim.x;
    lo = uint32_t(a) * unit;
    hi = min(uint32_t(b) * unit, rows);
}

// ---- prologue: build the input vector's limb planes in shared memory -------

// Element j of the input vector (after embedding / normalisation).
template <int MODE>
__device__ __forceinline__ int64_t input_elem(const GemvArgs& a, uint32_t j, int64_t r_inv,
                                              int64_t es, const int8_t* erow) {
    int64_t x;
    if (MODE == MODE_EMBED) x = int64_t(uint64_t(int64_t(erow[j])) * uint64_t(es));
    else x = a.x[j];
    if (MODE == MODE_PLAIN) return x;
    return mul16(mul16(x, r_inv), a.gamma[j]);
}

// rmsnorm's r = inv_sqrt(((sum x^2) / n >> 16) + 1) with the sum in int128
// (proj/src/kernels.cpp:56-68). Block-wide; every thread gets r.
template <int MODE>
__device__ int64_t norm_factor(const GemvArgs& a, int64_t es, const int8_t* erow, void* scratch) {
    const uint32_t K = a.K;
    u128 ss = 0;
    for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
        int64_t x = MODE == MODE_EMBED ? int64_t(uint64_t(int64_t(erow[j])) * uint64_t(es)) : a.x[j];
        ss += u128(i128(x) * i128(x));
    }
    ss = block_reduce<u128>(ss, static_cast<u128*>(scratch), [](u128 p, u128 q) { return p + q; },
                            warp_sum_u128);
    int64_t ms = int64_t((i128(ss) / i128(K)) >> 16);
    if (ms + 1 <= 0) {  // the reference throws std::domain_error from inv_sqrt_q16
        if (threadIdx.x == 0) atomicOr(&a.ctl->err, 1u);
        return 0;
    }
    return inv_sqrt_q16(ms + 1, a.seeds);
}

// Writes the limb planes; returns the limb count (3 or 8).
template <int MODE>
__device__ int build_limbs(const GemvArgs& a, uint32_t* planes /* [8][Kp/4] */, void* scratch) {
    const uint32_t K = a.K, Kw = a.Kp / 4;
    int64_t es = 0;
    const int8_t* erow = nullptr;
    if (MODE == MODE_EMBED) {
        uint32_t tok = a.tokens[a.ctl->pos];
        es = a.embd_scales[tok];
        erow = a.embd + size_t(tok) * K;
        if (blockIdx.x == 0)
            for (uint32_t j = threadIdx.x; j < K; j += blockDim.x)
                a.x_out[j] = int64_t(uint64_t(int64_t(erow[j])) * uint64_t(es));
    }
    const int64_t r_inv = MODE == MODE_PLAIN ? 0 : norm_factor<MODE>(a, es, erow, scratch);
    // pass 1: does every element fit the 3-limb range [-2^23, 2^23)?
    int fits = 1;
    for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
        int64_t v = input_elem<MODE>(a, j, r_inv, es, erow);
        fits &= (v >= -(int64_t(1) << 23)) & (v < (int64_t(1) << 23));
    }
    fits = __syncthreads_and(fits);
    const int L = fits ? 3 : 8;
    // pass 2: 4 consecutive elements -> one 32-bit word per plane
    for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
        uint32_t word[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint32_t j = 4 * w + e;
            uint64_t v = j < K ? uint64_t(input_elem<MODE>(a, j, r_inv, es, erow)) : 0;
            if (L == 3) {
                word[0] |= uint32_t(v & 0xFF) << (8 * e);
                word[1] |= uint32_t((v >> 8) & 0xFF) << (8 * e);
                word[2] |= uint32_t((v >> 16) & 0xFF) << (8 * e);  // == (x >> 16) as s8
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) word[k] |= uint32_t((v >> (8 * k)) & 0xFF) << (8 * e);
            }
        }
        for (int k = 0; k < L; ++k) planes[k * Kw + w] = word[k];
    }
    if (L == 8 && threadIdx.x == 0) atomicAdd(&a.ctl->stats[0], 1ull);
    __syncthreads();
    return L;
}

// ---- main loop --------------------------------------------------------------

// acc[r] (int64, wrapping) of R rows starting at r0 for this warp's lane
// slice; returns the full row sums in every lane after the warp reduction.
template <int L, int R, int U>
__device__ __forceinline__ void row_group_dot(const GemvArgs& a, const uint32_t* planes,
                                              uint32_t r0, uint32_t hi, int64_t (&out)[R]) {
    const int lane = threadIdx.x & 31;
    const uint32_t Kp = a.Kp, Kw = Kp / 4;
    int32_t acc[R][L];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < L; ++k) acc[r][k] = 0;
    const int8_t* wbase = a.W + size_t(r0) * Kp;
    bool valid[R];
#pragma unroll
    for (int r = 0; r < R; ++r) valid[r] = r0 + r < hi;

    for (uint32_t c0 = lane * 16; c0 < Kp; c0 += 512 * U) {
        int4 w[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t c = c0 + u * 512;
#pragma unroll
            for (int r = 0; r < R; ++r)
                w[u][r] = (c < Kp && valid[r]) ? ldg_stream(wbase + size_t(r) * Kp + c)
                                               : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t c = c0 + u * 512;
            if (c >= Kp) break;
            uint4 xl[L];
#pragma unroll
            for (int k = 0; k < L; ++k) xl[k] = *reinterpret_cast<const uint4*>(planes + k * Kw + c / 4);
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int k = 0; k < L - 1; ++k) {
                    acc[r][k] = dp4a_su(w[u][r].x, xl[k].x, acc[r][k]);
                    acc[r][k] = dp4a_su(w[u][r].y, xl[k].y, acc[r][k]);
                    acc[r][k] = dp4a_su(w[u][r].z, xl[k].z, acc[r][k]);
                    acc[r][k] = dp4a_su(w[u][r].w, xl[k].w, acc[r][k]);
                }
                acc[r][L - 1] = dp4a_ss(w[u][r].x, xl[L - 1].x, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(w[u][r].y, xl[L - 1].y, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(w[u][r].z, xl[L - 1].z, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(w[u][r].w, xl[L - 1].w, acc[r][L - 1]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint64_t v = 0;
#pragma unroll
        for (int k = 0; k < L; ++k) v += uint64_t(int64_t(acc[r][k])) << (8 * k);
        out[r] = int64_t(warp_sum_u64(v));
    }
}

template <int R>
__device__ __forceinline__ int64_t pick(const int64_t (&v)[R], int i) {
    int64_t r = v[0];
#pragma unroll
    for (int k = 1; k < R; ++k) r = i == k ? v[k] : r;
    return r;
}

template <int EPI, int L, int R, int U>
__device__ void gemv_rows(const GemvArgs& a, const uint32_t* planes, uint32_t lo, uint32_t hi,
                          int64_t& best_v, uint32_t& best_i) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* logit_row = nullptr;
    if (EPI == EPI_ARGMAX) {
        // kept slot, or the scratch row after the kept ones
        uint32_t slot = a.ctl->pos - a.ctl->logit_base;
        slot = slot < a.ctl->keep_cap ? slot : a.ctl->keep_cap;
        logit_row = a.logits + size_t(slot) * a.rows;
    }
    for (uint32_t r0 = lo + warp * R; r0 < hi; r0 += GEMV_WARPS * R) {
        int64_t v[R];
        row_group_dot<L, R, U>(a, planes, r0, hi, v);
        if (EPI == EPI_SILU) {
            // rows (2i, 2i+1) = (gate_i, up_i); lane j finishes pair j
            if (lane < R / 2 && r0 + 2 * lane + 1 < hi) {
                uint32_t row = r0 + 2 * lane;
                int64_t g = scale_row(pick<R>(v, 2 * lane), a.scales[row]);
                int64_t u = scale_row(pick<R>(v, 2 * lane + 1), a.scales[row + 1]);
                a.y[row / 2] = mul16(silu_q16(g, a.exp_lut), u);
            }
        } else {
            const uint32_t row = r0 + lane;
            int64_t val = 0;
            if (lane < R && row < hi) {
                int64_t acc = pick<R>(v, lane);
                if (EPI == EPI_RAW) {
                    a.y[row] = acc;
                } else {
                    val = scale_row(acc, a.scales[row]);
                    if (EPI == EPI_STORE) a.y[row] = val;
                    if (EPI == EPI_RESID) a.y[row] = add_clamp(a.y[row], val);
                    if (EPI == EPI_ARGMAX) logit_row[row] = val;
                }
            }
            if (EPI == EPI_ARGMAX && lane < R && row < hi && better(val, row, best_v, best_i)) {
                best_v = val;
                best_i = row;
            }
        }
    }
}

template <int EPI, int MODE, int R, int U>
__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(GemvArgs a) {
    extern __shared__ __align__(16) uint32_t planes[];  // [8][Kp/4]
    __shared__ u128 scratch[32];
    uint32_t lo, hi;
    cta_rows(a.rows, EPI == EPI_SILU ? 2 : 1, lo, hi);
    {
        // Warm L2 with this warp's first row group while the prologue runs.
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t r0 = lo + warp * R;
        for (int r = 0; r < R; ++r)
            if (r0 + r < hi)
                for (uint32_t c = lane * 128; c < a.Kp; c += 32 * 128)
                    prefetch_l2(a.W + size_t(r0 + r) * a.Kp + c);
    }
    const int L = build_limbs<MODE>(a, planes, scratch);
    int64_t best_v = INT64_MIN;
    uint32_t best_i = 0xFFFFFFFFu;
    if (L == 3) gemv_rows<EPI, 3, R, U>(a, planes, lo, hi, best_v, best_i);
    else gemv_rows<EPI, 8, R, 2>(a, planes, lo, hi, best_v, best_i);

    if (EPI == EPI_ARGMAX) {
        // CTA best -> parts[blockIdx]; the last CTA reduces all parts and
        // appends the token (deterministic: the (max, min index) order is total).
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int64_t ov = __shfl_xor_sync(0xffffffffu, best_v, o);
            uint32_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (better(ov, oi, best_v, best_i)) { best_v = ov; best_i = oi; }
        }
        __shared__ int64_t sv[GEMV_WARPS];
        __shared__ uint32_t si[GEMV_WARPS];
        __shared__ bool last;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) { sv[warp] = best_v; si[warp] = best_i; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < GEMV_WARPS; ++w)
                if (better(sv[w], si[w], best_v, best_i)) { best_v = sv[w]; best_i = si[w]; }
            a.parts[blockIdx.x].v = best_v;
            a.parts[blockIdx.x].idx = best_i;
            __threadfence();
            last = atomicAdd(&a.ctl->argmax_count, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            int64_t bv = INT64_MIN;
            uint32_t bi = 0xFFFFFFFFu;
            for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
                int64_t v = *((volatile int64_t*)&a.parts[b].v);
                uint32_t i = *((volatile uint32_t*)&a.parts[b].idx);
                if (better(v, i, bv, bi)) { bv = v; bi = i; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
                uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < GEMV_WARPS; ++w)
                    if (better(sv[w], si[w], bv, bi)) { bv = sv[w]; bi = si[w]; }
                uint32_t pos = a.ctl->pos;
                a.tokens_out[pos + 1] = bi;
                a.ctl->pos = pos + 1;
                a.ctl->argmax_count = 0;
            }
        }
    }
}

// Advances the position after a prompt step that has no lm_head.
__global__ void advance_pos_kernel(Ctl* ctl) { ctl->pos += 1; }

}  // namespace dimg::dev
