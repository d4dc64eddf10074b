// Device-side Q16 integer primitives (proj/src/q16.cpp, proj/include/dim/q16.hpp).
//
// Every rescale is the reference's floor shift; every place the reference
// widens to int128 widens here too (__int128 is native in sm_100a device
// code: mul.lo/mul.hi pairs). Sums the reference keeps in int64/int128 are
// carried in unsigned types so the two's-complement wrap it relies on is
// reproduced without C++ undefined behaviour. No floating point anywhere.
#pragma once

#include <cstdint>

namespace dimg::dev {

typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr int64_t ONE = int64_t(1) << 16;
constexpr int64_t ACT_CLAMP = 256 * ONE;  // proj/include/dim/kernels.hpp:16

__device__ __forceinline__ bool fits_i32(int64_t v) {
    return ((uint64_t(v) + 0x80000000ull) >> 32) == 0;
}

// Programmatic dependent launch (the batch step's kernels are launched with
// programmatic stream serialization): a kernel may start while its
// predecessor still runs; pdl_wait() returns once every prerequisite grid has
// completed and its writes are visible, so everything before it may touch
// only constant data (weights, tables). launch_dependents lets the next
// kernel start launching. Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// The tensor-core operand form of an activation: three balanced signed byte
// digits, v = d0 + 2^8 d1 + 2^16 d2 with every d in [-128, 127], exact for
// -0x808080 <= v <= 0x7F7F7F. All three limbs are s8, so one kind::i8 MMA
// covers them together (tc_gemm.cuh). Writes the digits to p[0], p[plane],
// p[2 plane]; returns false (digits meaningless) outside that range.
__device__ __forceinline__ bool put_sdigits(uint8_t* p, size_t plane, int64_t v) {
    const int64_t d0 = int8_t(v);
    const int64_t r1 = (v - d0) >> 8;
    const int64_t d1 = int8_t(r1);
    p[0] = uint8_t(d0);
    p[plane] = uint8_t(d1);
    p[2 * plane] = uint8_t((r1 - d1) >> 8);
    return uint64_t(v + 0x808080) <= 0xFFFFFFu;
}

// int64((int128(a) * b) >> k) for 0 < k < 64, exact for every input: the
// 128-bit product is (hi, lo) = (mul.hi.s64, mul.lo.s64), and the low 64 bits
// of the arithmetic shift are (lo >>> k) | (hi << (64 - k)). Two multiplies,
// no branches -- compact code matters in this kernel (see persistent.cuh).
template <int k>
__device__ __forceinline__ int64_t mul_shr(int64_t a, int64_t b) {
    const uint64_t lo = uint64_t(a) * uint64_t(b);
    const uint64_t hi = uint64_t(__mul64hi(a, b));
    return int64_t((lo >> k) | (hi << (64 - k)));
}

// int64(a) * b for int32 operands as one IMAD.WIDE (in some contexts the
// compiler emits a 64 x 64-bit multiply for the C++ expression).
__device__ __forceinline__ int64_t mulw(int32_t a, int32_t b) {
    int64_t p;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    return p;
}

// Full signed 64x64 -> 128-bit product.
__device__ __forceinline__ u128 mul_full(int64_t a, int64_t b) {
    return (u128(uint64_t(__mul64hi(a, b))) << 64) | uint64_t(a * b);
}

// q16_mul: (int128(a) * b) >> 16, truncated to int64 (q16.hpp:28-30).
__device__ __forceinline__ int64_t mul16(int64_t a, int64_t b) { return mul_shr<16>(a, b); }

// Same value when both factors fit 32 bits (one IMAD.WIDE); callers check.
__device__ __forceinline__ int64_t mul16_small(int64_t a, int64_t b) {
    return (int64_t(int32_t(a)) * int32_t(b)) >> 16;
}

// floor(p * v / 2^16) for 0 <= p <= 2^16 (softmax probabilities) with 64-bit
// ops only: v = vh*2^16 + vl, vl in [0, 2^16) => p*vh + (p*vl >> 16) exactly.
__device__ __forceinline__ int64_t mul16_prob(int64_t p, int64_t v) {
    if (fits_i32(v)) return (p * int64_t(int32_t(v))) >> 16;  // |p*v| < 2^48: exact
    int64_t vh = v >> 16;
    uint64_t vl = uint64_t(v) & 0xFFFFu;
    return int64_t(uint64_t(p) * uint64_t(vh) + ((uint64_t(p) * vl) >> 16));
}

__device__ __forceinline__ int64_t wrap_add(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) + uint64_t(b));
}
__device__ __forceinline__ int64_t wrap_sub(int64_t a, int64_t b) {
    return int64_t(uint64_t(a) - uint64_t(b));
}

// Dense epilogue: (int128(acc) * scale) >> 16 (proj/src/kernels.cpp:27).
__device__ __forceinline__ int64_t scale_row(int64_t acc, int64_t s) { return mul_shr<16>(acc, s); }

// residual_add_clamp (proj/src/kernels.cpp:192-200).
__device__ __forceinline__ int64_t add_clamp(int64_t a, int64_t b) {
    int64_t s = wrap_add(a, b);
    return s > ACT_CLAMP ? ACT_CLAMP : (s < -ACT_CLAMP ? -ACT_CLAMP : s);
}

// floor(a b / 2^s) for 0 < s < 64; *ok cleared if the quotient needs more
// than 64 bits.
__host__ __device__ __forceinline__ uint64_t mul_shr_u64(uint64_t a, uint64_t b, int s, bool* ok) {
#ifdef __CUDA_ARCH__
    const uint64_t lo = a * b, hi = __umul64hi(a, b);
#else
    const unsigned __int128 p = (unsigned __int128)a * b;
    const uint64_t lo = uint64_t(p), hi = uint64_t(p >> 64);
#endif
    if (hi >> s) *ok = false;
    return (lo >> s) | (hi << (64 - s));
}

// The same three Newton steps on 64-bit words: for x >= 16 every quantity
// is non-negative and bounded -- the octave seed y0 = 2^(56 - b/2 - 1/4) is
// within 2^(+-1/4) of 2^56 / sqrt(x), so y <= 2^54.3, t = y^2 >> 48 < 2^61,
// u = x t >> 16 < 2^48.6 < 3 * 2^48, and y (3 * 2^48 - u) < 2^105 -- so each
// int128 product of the reference is one exact 64 x 64 -> 128-bit product
// whose shifted quotient fits 64 bits, and the floors agree (no negative
// values). Returns -1 where that does not hold (x < 16, u >= 3 * 2^48, a
// quotient above 2^64), and the caller takes the int128 path. tests/test_host.py checks it against
// the oracle's int128 routine over every octave.
__host__ __device__ __forceinline__ int64_t inv_sqrt_q16_u64(int64_t x, int b, int64_t seed) {
    if (b < 4 || seed <= 0) return -1;
    const uint64_t three = uint64_t(3) << 48;
    uint64_t y = uint64_t(seed);
    bool ok = true;
    for (int it = 0; it < 3; ++it) {
        const uint64_t t = mul_shr_u64(y, y, 48, &ok);
        const uint64_t u = mul_shr_u64(uint64_t(x), t, 16, &ok);
        if (u >= three) return -1;
        y = mul_shr_u64(y, three - u, 49, &ok);
    }
    if (!ok || (y >> 62)) return -1;
    return int64_t((y + (uint64_t(1) << 31)) >> 32);
}

// inv_sqrt_q16: octave seed (host-built Q48 table) + three Newton steps at
// Q48 in int128, rounded to Q16 (proj/src/q16.cpp:56-68). x > 0.
__device__ __noinline__ int64_t inv_sqrt_q16(int64_t x, const int64_t* seeds) {
    int b = 63 - __clzll(x);
    const int64_t f = inv_sqrt_q16_u64(x, b, seeds[b]);
    if (f >= 0) return f;
    i128 y = seeds[b];
    const i128 three = i128(3) << 48;
#pragma unroll
    for (int it = 0; it < 3; ++it) {
        i128 t = (y * y) >> 48;
        i128 u = (i128(x) * t) >> 16;
        y = (y * (three - u)) >> 49;
    }
    return int64_t((y + (i128(1) << 31)) >> 32);
}

// exp_neg_lut: 257-entry table, 2048 raw units per cell, round-half-up
// linear interpolation (proj/src/q16.cpp:81-92). 0 <= t <= 8*ONE.
__device__ __forceinline__ int64_t exp_neg(int64_t t, const int64_t* e) {
    int64_t cell = t >> 11, frac = t & 2047;
    if (cell == 256) return e[0];
    int64_t hi = e[256 - cell], lo = e[255 - cell];
    return hi - (((hi - lo) * frac + 1024) >> 11);
}

// exp_neg on 32 bits for 0 <= t <= 8*ONE, with the table L[0] = e[0],
// L[1 + i] = e[i] (e <= 2^16): cell 256 (t = 8*ONE) reads L[1] - L[0] = 0.
__device__ __forceinline__ uint32_t exp_neg32(uint32_t t, const int32_t* L) {
    const uint32_t cell = t >> 11, frac = t & 2047;
    const int32_t hi = L[257 - cell], lo = L[256 - cell];
    return uint32_t(hi - ((uint32_t(hi - lo) * frac + 1024) >> 11));
}

// floor(a / d) for a < 2^63, d >= 1, given inv = ~0ull / d (one division
// shared by many quotients): umulhi(a, inv) is floor(a / d) or one less.
__device__ __forceinline__ uint64_t udiv_inv(uint64_t a, uint64_t d, uint64_t inv) {
    const uint64_t q = __umul64hi(a, inv);
    return q + ((a - q * d) >= d);
}

// floor(a / d) for 0 <= a, 1 <= d < 2^24 and a quotient below 2^22, without
// a 64-bit division and branch-free: the float estimate a * rcp(d) carries a
// relative error below 3 * 2^-24 (three roundings), so it is within 0.75 of
// the quotient and truncates to q - 1, q or q + 1; the exact remainder then
// fixes the one step.
__device__ __forceinline__ int64_t div_rcp(int64_t a, int64_t d) {
    int64_t q = int64_t(float(a) * __frcp_rn(float(d)));
    const int64_t r = a - q * d;
    q -= r < 0;
    q += r >= d;
    return q;
}

// sigmoid_q16 with exact symmetry (proj/src/q16.cpp:94-101).
__device__ __forceinline__ int64_t sigmoid_q16(int64_t x, const int64_t* e) {
    bool pos = x > 0;
    int64_t xn = pos ? -x : x;  // x > 0 => -x is representable
    int64_t t = xn <= -8 * ONE ? 8 * ONE : -xn;
    int64_t ev = exp_neg(t, e);   // [0, ONE]
    int64_t den = ONE + ev;       // [2^16, 2^17]
    int64_t s = div_rcp((ev << 16) + den / 2, den);
    return pos ? ONE - s : s;
}

// silu_q16 = mul16(x, sigmoid(x)) (proj/src/q16.cpp:103-105).
__device__ __forceinline__ int64_t silu_q16(int64_t x, const int64_t* e) {
    return mul16(x, sigmoid_q16(x, e));
}

// ---- warp / block reductions ------------------------------------------------

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ u128 warp_sum_u128(u128 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t lo = __shfl_xor_sync(0xffffffffu, uint64_t(v), o);
        uint64_t hi = __shfl_xor_sync(0xffffffffu, uint64_t(v >> 64), o);
        v += (u128(hi) << 64) | lo;
    }
    return v;
}

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// Block-wide reductions through `scratch` (>= 32 entries of the type).
template <class T, class Op>
__device__ __forceinline__ T block_reduce(T v, T* scratch, Op op, T (*warp_op)(T)) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_op(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    T r = scratch[0];
    for (int i = 1; i < nw; ++i) r = op(r, scratch[i]);
    return r;
}

// Block-wide u128 sum (all threads get it); kept out of line.
__device__ __noinline__ u128 block_sum_u128(u128 v, u128* scratch) {
    return block_reduce<u128>(v, scratch, [](u128 p, u128 q) { return p + q; }, warp_sum_u128);
}

// Argmax key: larger value wins, lower index on ties (engine.cpp:113-120).
__device__ __forceinline__ bool better(int64_t v1, uint32_t i1, int64_t v2, uint32_t i2) {
    return v1 > v2 || (v1 == v2 && i1 < i2);
}

}  // namespace dimg::dev
