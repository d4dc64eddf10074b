// Prefill attention scores on the tensor cores (tcgen05.mma kind::i8), exact:
//   score(t, p) = mul16(dot(q_t, k_p) >> 16, inv_scale)   (proj/src/kernels.cpp:143-151)
// for every query t of a 32-query block and every cached position p <= t.
//
// dot(q, k) is an int64 sum of int32 products. With balanced signed byte
// digits -- k = sum_i 2^(8i) k_i (4 digits, |k| within int32's 4-digit range)
// and q = sum_d 2^(8d) q_d (3 digits) -- it is the exact int64 combination
// sum_{i,d} 2^(8(i+d)) (sum_j k_i,j q_d,j) of 12 int8 x int8 dot products,
// each an exact int32 MMA accumulation for dh <= 128 (|sum| <= 2^21). One
// MMA (M = 128 positions, N = 3 x 32 query digits, K = 32 dims) per key
// digit plane and K step: 16 MMAs per 128-position tile. Key digit i's MMA
// starts at TMEM column 32 i, so the tensor core itself adds the digit pairs
// of equal weight: six 32-column groups per tile, double-buffered (the MMAs
// of the next tile overlap this tile's epilogue).
//
// Key digit planes come precomputed per layer (pf_rope_kv_kernel, plain
// [H][4][n_pad][128 B]) and stream in by TMA with the 128B swizzle, two tiles
// in flight; the query digits are built once per CTA straight into the
// swizzled layout. The epilogue reads the six groups of 16 queries, combines
// them into the int64 scores, and writes the int32 score strips pf_attn_kernel's
// softmax / PV passes consume. Values outside the digit ranges set *wide
// (the engine reruns on the exact path).
#pragma once

#include <cstdint>

#include "q16.cuh"
#include "tc_gemm.cuh"

namespace dimg::dev {

constexpr int PS_M = 128;       // positions per tile (MMA M)
constexpr int PS_Q = 32;        // queries per CTA (= PA_Q)
constexpr int PS_KD = 4;        // key digits
constexpr int PS_QD = 3;        // query digits
constexpr int PS_DH = 128;      // head dim (one 128-byte K block)
constexpr int PS_THREADS = 256;  // 8 warps: warps w and w + 4 share TMEM lane quarter w, 16 queries each
constexpr int PS_A_BYTES = PS_KD * PS_M * PS_DH;   // one tile: 4 planes x 128 rows x 128 B
constexpr int PS_B_BYTES = PS_QD * PS_Q * PS_DH;   // 96 rows x 128 B
constexpr int PS_N = PS_QD * PS_Q;                 // MMA N
constexpr int PS_G = PS_KD + PS_QD - 1;            // digit-pair weight groups 2^(8k), k = i + d
constexpr uint32_t PS_ACC_STRIDE = 256;            // TMEM columns between the two accumulator sets
constexpr uint32_t PS_TMEM_COLS = 512;             // 2 x 6 x 32 = 384 used

__host__ __device__ constexpr size_t pf_scores_smem() { return 2 * size_t(PS_A_BYTES) + PS_B_BYTES + 1024; }

// byte offset of (row, byte) in a [rows][128 B] tile with the 128B swizzle
__device__ __forceinline__ uint32_t ps_sw128(uint32_t row, uint32_t byte) {
    return row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}

// balanced signed byte digits of v into packed[0..n): byte e of packed[i] is
// digit i of value e; false if v is outside the n-digit range
template <int N>
__device__ __forceinline__ bool ps_digits(int64_t v, int e, uint32_t (&packed)[N]) {
    int64_t r = v;
#pragma unroll
    for (int i = 0; i < N - 1; ++i) {
        const int64_t d = int8_t(r);
        packed[i] |= uint32_t(uint8_t(d)) << (8 * e);
        r = (r - d) >> 8;
    }
    packed[N - 1] |= uint32_t(uint8_t(int8_t(r))) << (8 * e);
    return r >= -128 && r <= 127;
}

// grid (H, ceil(n / 32)); kmap: the key digit planes [H * 4 * n_pad rows][128 B]
__global__ void __launch_bounds__(PS_THREADS, 1) pf_scores_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                  const int64_t* __restrict__ qkv, uint32_t n,
                                                                  uint32_t n_pad, uint32_t D, int64_t inv_scale,
                                                                  int32_t* strips, uint32_t* wide, const uint32_t* kd4) {
    extern __shared__ uint8_t ps_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ps_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                    // 2 x tile
    uint8_t* B = smem + 2 * PS_A_BYTES;   // query digits, row d * 32 + q
    __shared__ __align__(8) uint64_t full[2], mma_done[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t h = blockIdx.x, q0 = blockIdx.y * PS_Q;
    const uint32_t last_q = min(n, q0 + PS_Q) - 1;
    const uint32_t n_tiles = last_q / PS_M + 1;   // tiles of positions 0 .. last_q
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ld = (n + 3) & ~3u;
    // keys within 3 digits (|k| <= 0x7F7F7F, the usual case) leave the 4th
    // plane zero: 9 digit pairs instead of 12
    int n_kd = PS_KD;
    int big = 0;

    if (threadIdx.x == 0) {
        tg_mbar_init(&full[0], 1);
        tg_mbar_init(&full[1], 1);
        tg_mbar_init(&mma_done[0], 1);
        tg_mbar_init(&mma_done[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tg_smem_u32(&tmem_slot)), "n"(PS_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    pdl_launch_dependents();
    pdl_wait();  // q (QKV GEMM) and the key digits (RoPE/KV kernel) come from the previous kernels
    // query digits: thread = (query, 4-dim group) pairs, one u32 per digit plane
    for (uint32_t i = threadIdx.x; i < PS_Q * (PS_DH / 4); i += PS_THREADS) {
        const uint32_t qi = i / (PS_DH / 4), j = 4 * (i % (PS_DH / 4));
        uint32_t pk[PS_QD] = {0, 0, 0};
        if (q0 + qi < n) {
            const int64_t* qr = qkv + size_t(q0 + qi) * 3 * D + size_t(h) * PS_DH + j;
#pragma unroll
            for (int e = 0; e < 4; ++e) big |= !ps_digits<PS_QD>(qr[e], e, pk);
        }
#pragma unroll
        for (int d = 0; d < PS_QD; ++d)
            *reinterpret_cast<uint32_t*>(B + ps_sw128(d * PS_Q + qi, j)) = pk[d];
    }
    n_kd = *kd4 ? PS_KD : PS_KD - 1;  // set by the RoPE/KV kernel: after the wait
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> MMA operand reads
    tg_fence_before();
    __syncthreads();
    tg_fence_after();
    const uint32_t tmem = tmem_slot;
    // warp 0 issues the TMA loads and MMAs (converged, one elected lane)
    auto load_tile = [&](uint32_t t) {  // the 4 key digit planes of positions [128 t, 128 t + 128)
        uint8_t* dst = A + (t & 1) * PS_A_BYTES;
        tg_expect_tx_w(&full[t & 1], n_kd * PS_M * PS_DH);
#pragma unroll
        for (int i = 0; i < PS_KD; ++i)
            if (i < n_kd)
                tg_tma_2d_w(dst + i * PS_M * PS_DH, &kmap, 0, int32_t((h * PS_KD + i) * n_pad + t * PS_M),
                            &full[t & 1]);
    };
    // Key digit i's MMA (N = 96: the three query digits d) writes TMEM
    // columns 32 i + 32 d + q: each digit pair lands in the accumulator of its
    // weight 2^(8(i + d)) -- six groups of 32 columns, summed by the tensor
    // core (|group| <= 3 x 2^21: int32). The first K step of digits 0 and 3
    // initialises all six groups (digit 3's plane is zero when unused), so a
    // tile takes 192 columns and two tiles' accumulators fit: the MMAs of
    // tile t + 1 run while the epilogue drains tile t.
    if (n_kd < PS_KD) {
        for (uint32_t i = threadIdx.x; i < 2 * PS_M * PS_DH / 16; i += PS_THREADS) {
            const uint32_t b = i / (PS_M * PS_DH / 16), o = i % (PS_M * PS_DH / 16);
            reinterpret_cast<int4*>(A + b * PS_A_BYTES + (PS_KD - 1) * PS_M * PS_DH)[o] = make_int4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tg_fence_before();
        __syncthreads();
        tg_fence_after();
    }
    auto issue_mma = [&](uint32_t t) {  // warp 0
        const uint32_t b = t & 1;
        tg_mbar_wait(&full[b], (t >> 1) & 1);
        tg_fence_after();
        const uint32_t sa = tg_smem_u32(A + b * PS_A_BYTES), sb = tg_smem_u32(B);
        const uint32_t dacc = tmem + b * PS_ACC_STRIDE;
#pragma unroll
        for (int kk = 0; kk < PS_DH / 32; ++kk) {
            tg_mma_w(dacc, tg_desc(sa + 32 * kk), tg_desc(sb + 32 * kk), tg_idesc(PS_N), kk != 0);
            if (kk == 0 || n_kd == PS_KD)
                tg_mma_w(dacc + 32 * (PS_KD - 1), tg_desc(sa + (PS_KD - 1) * PS_M * PS_DH + 32 * kk),
                         tg_desc(sb + 32 * kk), tg_idesc(PS_N), kk != 0);
#pragma unroll
            for (int i = 1; i < PS_KD - 1; ++i)
                tg_mma_w(dacc + 32 * i, tg_desc(sa + i * PS_M * PS_DH + 32 * kk), tg_desc(sb + 32 * kk),
                         tg_idesc(PS_N), 1);
        }
        tg_commit_w(&mma_done[b]);
    };
    if (warp == 0) {
        load_tile(0);
        if (n_tiles > 1) load_tile(1);
        issue_mma(0);
    }
    int32_t* Sc = strips + (size_t(h) * gridDim.y + blockIdx.y) * PS_Q * ld;  // the CTA's rows
    for (uint32_t t = 0; t < n_tiles; ++t) {
        const uint32_t b = t & 1;
        tg_mbar_wait(&mma_done[b], (t >> 1) & 1);
        tg_fence_after();
        if (warp == 0) {
            if (t + 2 < n_tiles) load_tile(t + 2);  // its buffer is free: tile t's MMAs read it
            if (t + 1 < n_tiles) issue_mma(t + 1);  // accumulators of tile t - 1: drained (barrier below)
        }
        // epilogue: thread = position p (TMEM lane of quarter warp % 4), the
        // warp's half of the 32 queries
        const uint32_t p = t * PS_M + 32 * (warp & 3) + lane;
        const uint32_t tb = tmem + b * PS_ACC_STRIDE + ((32 * (warp & 3)) << 16);
        {
            const int half = warp >> 2;
            int32_t g[PS_G][16];
#pragma unroll
            for (int k = 0; k < PS_G; ++k) tg_ld16(tb + 32 * k + 16 * half, g[k]);
            tg_ld_wait();
            // mul16(a, inv) with |a| = |dot >> 16| < 2^47 and 0 <= inv < 2^16
            // (the usual dh): the product fits int64, one multiply
            const bool small_inv = uint64_t(inv_scale) < (uint64_t(1) << 16);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const uint32_t qi = 16 * half + e, tq = q0 + qi;
                if (tq < n && p <= tq) {
                    int64_t s = 0;
#pragma unroll
                    for (int k = 0; k < PS_G; ++k) s += int64_t(g[k][e]) << (8 * k);
                    const int64_t a = s >> 16;
                    const int64_t val = small_inv ? (a * inv_scale) >> 16 : mul16(a, inv_scale);
                    big |= !fits_i32(val);
                    Sc[size_t(qi) * ld + p] = int32_t(val);
                }
            }
        }
        tg_fence_before();
        __syncthreads();  // every lane's TMEM reads done before tile t + 2's MMAs overwrite them
        tg_fence_after();
    }
    if (big) *wide = 1;
    tg_fence_before();
    __syncthreads();
    if (warp == 0) {
        tg_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(PS_TMEM_COLS)
                     : "memory");
    }
}

}  // namespace dimg::dev
