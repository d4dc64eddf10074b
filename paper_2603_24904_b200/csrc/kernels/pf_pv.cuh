// Prefill attention output (proj/src/kernels.cpp:153-159) with its linear
// half on the tensor cores, exact:
//   out(t, j) = sum_p floor(P(t, p) V(p, j) / 2^16)
//             = sum_p P vh  +  sum_p floor(P vl / 2^16),   V = vh 2^16 + vl, vl in [0, 2^16).
// The second sum F is per-product arithmetic and stays on the CUDA cores:
// pf_attn_kernel<_, true> writes only U = sum_p ((P V mod 2^32) >> 16), which
// is congruent to T + F modulo 2^16 (T = the first sum); as 0 <= F < sum_p P
// <= 2^16, F = (U - T) mod 2^16 exactly (epilogue). The first is a plain
// integer GEMM over the positions, done here with tcgen05.mma kind::i8:
//   A = vh as ONE signed byte digit per (dim, position) -- exact while
//       |V| < 2^23, else *wide and the engine reruns on the exact path;
//       [H][128 dims][n_pad positions] planes built by pf_vh_kernel and
//       streamed by TMA (128B swizzle, K-major in positions);
//   B = P as TWO unsigned byte digits (P < 2^16 for every query but the
//       first, whose single P = 2^16 at position 0 makes its output V(0)
//       exactly: handled in the epilogue), rows d * 32 + q, built per
//       128-position tile from the probability strips;
// D (128 dims x 64) accumulates in TMEM over all position tiles: four MMAs
// (K = 32 positions) per tile. |digit sums| <= 2048 * 255 * 128 < 2^26 and
// |sum P vh| <= 2^16 * 2^7 (sum P <= 2^16): int32 throughout.
#pragma once

#include <cstdint>

#include "q16.cuh"
#include "tc_gemm.cuh"

namespace dimg::dev {

constexpr int PV_M = 128;        // head dims (MMA M)
constexpr int PV_Q = 32;         // queries per CTA (= PA_Q)
constexpr int PV_KB = 128;       // positions per tile
constexpr int PV_N = 2 * PV_Q;   // MMA N: two digits x 32 queries
constexpr int PV_THREADS = 256;
constexpr int PV_A_BYTES = PV_M * PV_KB;   // 16 KB
constexpr int PV_B_BYTES = PV_N * PV_KB;   // 8 KB
constexpr uint32_t PV_TMEM_COLS = 64;

__host__ __device__ constexpr size_t pf_pv_smem() { return 2 * size_t(PV_A_BYTES) + 2 * size_t(PV_B_BYTES) + 1024; }

// kind::i8, D s32, A s8 (vh digits), B u8 (probability digits), K-major, M 128
__host__ __device__ constexpr uint32_t pv_idesc() {
    return (2u << 4) | (1u << 7) | (0u << 10) | (uint32_t(PV_N >> 3) << 17) | (uint32_t(PV_M >> 4) << 24);
}

// byte offset of (row, byte) in a [rows][128 B] tile with the 128B swizzle
__device__ __forceinline__ uint32_t pv_sw128(uint32_t row, uint32_t byte) {
    return row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}

// vh = V >> 16 of every cached position < n, transposed to the A planes
// [H][128 dims][n_pad positions] (zero past n); *wide if some |V| >= 2^23.
// grid (H, n_pad / 128), 256 threads: one 128 x 128 tile per CTA.
__global__ void __launch_bounds__(256) pf_vh_kernel(const int32_t* __restrict__ V32, size_t head_stride, uint32_t n,
                                                    uint32_t n_pad, int8_t* __restrict__ vh, uint32_t* wide) {
    __shared__ __align__(16) uint8_t T[PV_M][PV_KB + 16];  // [dim][position], padded rows
    pdl_launch_dependents();
    pdl_wait();
    const uint32_t h = blockIdx.x, p0 = blockIdx.y * PV_KB;
    const int32_t* Vh = V32 + size_t(h) * head_stride;
    int bad = 0;
    for (uint32_t i = threadIdx.x; i < PV_KB * (PV_M / 4); i += blockDim.x) {
        const uint32_t pp = i / (PV_M / 4), d = 4 * (i % (PV_M / 4)), p = p0 + pp;
        int4 v = make_int4(0, 0, 0, 0);
        if (p < n) v = *reinterpret_cast<const int4*>(Vh + size_t(p) * PV_M + d);
        const int32_t e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int32_t x = e4[e] >> 16;
            bad |= uint32_t(x + 128) > 255u;  // |V| < 2^23
            T[d + e][pp] = uint8_t(int8_t(x));
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < PV_M * (PV_KB / 16); i += blockDim.x) {
        const uint32_t d = i / (PV_KB / 16), c = 16 * (i % (PV_KB / 16));
        *reinterpret_cast<int4*>(vh + (size_t(h) * PV_M + d) * n_pad + p0 + c) =
            *reinterpret_cast<const int4*>(&T[d][c]);
    }
    if (bad) *wide = 1;
}

// grid (H, ceil(n / 32)); vmap: the vh planes [H * 128 rows][n_pad bytes];
// strips: the probabilities [H][n rounded to 32][ld] (pf_attn_kernel); fl:
// U = sum_p ((P V mod 2^32) >> 16) [H][n][128]; out: the attention vector's three
// signed digit planes (WO's B operand).
__global__ void __launch_bounds__(PV_THREADS, 1) pf_pv_kernel(const __grid_constant__ CUtensorMap vmap,
                                                              const int32_t* __restrict__ strips,
                                                              const int32_t* __restrict__ fl,
                                                              const int32_t* __restrict__ V32, size_t head_stride,
                                                              uint32_t n, uint8_t* planes, uint32_t rows_pad,
                                                              uint32_t ldp, uint32_t* wide) {
    extern __shared__ uint8_t pv_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pv_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                      // 2 x [128 dims][128 positions]
    uint8_t* B = smem + 2 * PV_A_BYTES;     // 2 x [64 rows = digit * 32 + query][128 positions]
    __shared__ __align__(8) uint64_t full[2], mma_done;
    __shared__ uint32_t tmem_slot;
    const uint32_t h = blockIdx.x, q0 = blockIdx.y * PV_Q;
    const uint32_t last_q = min(n, q0 + PV_Q) - 1;
    const uint32_t n_tiles = last_q / PV_KB + 1;
    const uint32_t ld = (n + 3) & ~3u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int big = 0;

    if (threadIdx.x == 0) {
        tg_mbar_init(&full[0], 1);
        tg_mbar_init(&full[1], 1);
        tg_mbar_init(&mma_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tg_smem_u32(&tmem_slot)), "n"(PV_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    pdl_launch_dependents();
    pdl_wait();  // the strips and fl (pf_attn_kernel), the vh planes (pf_vh_kernel)
    tg_fence_before();
    __syncthreads();
    tg_fence_after();
    const uint32_t tmem = tmem_slot;
    auto load_a = [&](uint32_t t) {
        tg_expect_tx_w(&full[t & 1], PV_A_BYTES);
        tg_tma_2d_w(A + (t & 1) * PV_A_BYTES, &vmap, int32_t(t * PV_KB), int32_t(h * PV_M), &full[t & 1]);
    };
    if (warp == 0) load_a(0);
    const int32_t* Sc = strips + (size_t(h) * gridDim.y + blockIdx.y) * PV_Q * ld;  // the CTA's rows
    for (uint32_t t = 0; t < n_tiles; ++t) {
        // B tile: thread = (query, 4 positions), both digits as 4-byte words
        uint8_t* Bt = B + (t & 1) * PV_B_BYTES;
        for (uint32_t i = threadIdx.x; i < PV_Q * (PV_KB / 4); i += PV_THREADS) {
            const uint32_t qi = i / (PV_KB / 4), c = 4 * (i % (PV_KB / 4)), tq = q0 + qi;
            uint32_t w0 = 0, w1 = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t p = t * PV_KB + c + e;
                // query 0: its single P = 2^16 (position 0) is left out here (epilogue)
                const uint32_t pv = (tq < n && p <= tq && tq > 0) ? uint32_t(Sc[size_t(qi) * ld + p]) : 0u;
                w0 |= (pv & 0xFFu) << (8 * e);
                w1 |= ((pv >> 8) & 0xFFu) << (8 * e);
            }
            *reinterpret_cast<uint32_t*>(Bt + pv_sw128(qi, c)) = w0;
            *reinterpret_cast<uint32_t*>(Bt + pv_sw128(PV_Q + qi, c)) = w1;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> MMA operand reads
        tg_fence_before();
        __syncthreads();
        tg_fence_after();
        if (t > 0) tg_mbar_wait(&mma_done, (t - 1) & 1);  // tile t - 1's MMAs done: its A buffer is free
        if (warp == 0 && t + 1 < n_tiles) load_a(t + 1);
        tg_mbar_wait(&full[t & 1], (t >> 1) & 1);
        tg_fence_after();
        if (warp == 0) {
            const uint32_t sa = tg_smem_u32(A + (t & 1) * PV_A_BYTES), sb = tg_smem_u32(Bt);
#pragma unroll
            for (int kk = 0; kk < PV_KB / 32; ++kk)
                tg_mma_w(tmem, tg_desc(sa + 32 * kk), tg_desc(sb + 32 * kk), pv_idesc(), (t | kk) != 0);
            tg_commit_w(&mma_done);
        }
    }
    tg_mbar_wait(&mma_done, (n_tiles - 1) & 1);
    tg_fence_after();
    // epilogue: thread = head dim (TMEM lane of quarter warp % 4), the warp's
    // half of the 32 queries; 16 queries per TMEM read
    {
        const uint32_t j = 32 * (warp & 3) + lane;
        const uint32_t tb = tmem + ((32 * (warp & 3)) << 16);
        const int half = warp >> 2;
        int32_t d0[16], d1[16];
        tg_ld16(tb + 16 * half, d0);
        tg_ld16(tb + PV_Q + 16 * half, d1);
        tg_ld_wait();
        const size_t plane = size_t(rows_pad) * ldp;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const uint32_t tq = q0 + 16 * half + e;
            if (tq >= n) break;
            int64_t v;
            if (tq == 0) v = V32[size_t(h) * head_stride + j];  // P(0, 0) = 2^16: the output is V(0)
            else {
                const int64_t T = int64_t(d0[e]) + 256 * int64_t(d1[e]);  // sum_p P vh
                const uint32_t U = uint32_t(fl[(size_t(h) * n + tq) * PV_M + j]);
                v = T + int64_t((U - uint32_t(T)) & 0xFFFFu);  // + sum_p floor(P vl / 2^16)
            }
            if (!put_sdigits(planes + size_t(tq) * ldp + h * PV_M + j, plane, v)) big = 1;
        }
    }
    if (big) *wide = 1;
    tg_fence_before();
    __syncthreads();
    if (warp == 0) {
        tg_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(PV_TMEM_COLS)
                     : "memory");
    }
}

}  // namespace dimg::dev
