// Exact int8 x int64 dense products for many tokens on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// dense_forward (proj/src/kernels.cpp:18-30) for T tokens at once:
//   y[t][n] = ((sum_j W[n][j] * x[t][j])_int64 * s[n]) >> 16
// with int8 W and int64 activations. Activations in [-0x808080, 0x7F7F7F]
// are split into three balanced signed byte digits x = l0 + 2^8 l1 + 2^16 l2
// (put_sdigits, q16.cuh), so each limb product is a plain s8 x s8 GEMM with
// int32 accumulation -- exact: K * 128 * 128 < 2^31 for K < 131072 -- and
// acc = D0 + 2^8 D1 + 2^16 D2 is recombined exactly in int64 in the epilogue.
// (Larger activations are detected by the producers; the engine then takes
// the exact CUDA-core path instead.)
//
// Tiles are 128 features x BN tokens (64, or 16 for decode batches): the
// weights are the MMA A operand (M = features, K-major); the three limb
// planes of the tokens land as three contiguous BN-row B tiles, which one
// MMA with N = 3 BN consumes together (every limb is s8, so one instruction
// descriptor fits all three: a third of the MMA instructions of a per-limb
// issue, whose fixed per-instruction cost dominated small-N tiles), and a
// tile's accumulators take 3 x BN TMEM columns. The kernel is persistent (one
// CTA per SM walks tiles round-robin) with two accumulator sets in TMEM, so
// the epilogue of one tile overlaps the MMAs of the next. TMA loads 128-byte
// K slices of every operand with the 128B swizzle that the UMMA smem
// descriptors describe; an mbarrier ring of ~200 KB feeds the MMA warp.
// When there are too few output tiles to occupy every SM (decode batches),
// several CTAs split a tile's K range (split-K, see TgArgs).
// Warp roles: 0 = TMA producer, 1 = TMEM owner + MMA issuer, 2..5 = epilogue
// (warp w reads TMEM lane quarter w % 4, i.e. features 32 (w % 4) .. +31,
// one feature per thread -> coalesced stores across the warp).
#pragma once

#include <cuda.h>

#include <cstdint>

#include "q16.cuh"

namespace dimg::dev {

constexpr int TG_BM = 128;      // features per tile (MMA M)
constexpr int TG_BN = 64;       // tokens per tile (MMA N), prefill / large batches
constexpr int TG_BN_SMALL = 16; // tokens per tile for decode batches of <= 16 sequences
constexpr int TG_BK = 128;      // K bytes per stage = one 128-byte swizzle row
constexpr int TG_L = 3;         // activation limbs
constexpr int TG_A_BYTES = TG_BM * TG_BK;
constexpr int TG_THREADS = 192;  // BN 16: producer + MMA warp + 4 epilogue warps
template <int BN>
struct TgShape {
    static constexpr int B_BYTES = BN * TG_BK;
    static constexpr int STAGE_BYTES = TG_A_BYTES + TG_L * B_BYTES;  // 40 KB (BN 64) / 22 KB (BN 16)
    // BN 64: one CTA per SM with a ~200 KB ring; BN 16 (decode batches, few
    // tiles): a ~100 KB ring so two CTAs share an SM and more tiles stream at once
#ifndef TG_RING_SMALL
#define TG_RING_SMALL (100 * 1024)
#endif
    static constexpr int RING = BN >= 64 ? 200 * 1024 : TG_RING_SMALL;
    // 16-token tiles: the register bound that lets one of these CTAs share an
    // SM with the previous kernel's CTAs (PDL) -- 3 -> <= 113 registers
#ifndef TG_SMALL_MINB
#define TG_SMALL_MINB 2
#endif
    static constexpr int STAGES = RING / STAGE_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;  // + alignment slack
    static constexpr int ACC = TG_L * BN;  // TMEM columns of one tile's accumulators
    static constexpr int NB = 2;  // accumulator sets (double-buffered: epilogue || next MMAs)
    // epilogue warps: 8 for 64-token tiles (two per TMEM lane quarter, each
    // taking half of the tile's 16-column chunks: the SiLU epilogue of a tile
    // is then not exposed behind a short tile list), 4 for 16-token tiles
    static constexpr int EPI_WARPS = BN >= 64 ? 8 : 4;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
    static constexpr int MIN_BLOCKS = BN >= 64 ? 1 : TG_SMALL_MINB;
    static constexpr uint32_t TMEM_COLS = NB * ACC <= 128 ? 128 : NB * ACC <= 256 ? 256 : 512;
};

enum { TG_STORE = 0, TG_RESID = 1, TG_SILU = 2 };

struct TgArgs {
    uint32_t n_out;      // output features (rows of W)
    uint32_t n_tok;      // tokens
    uint32_t n_kblk;     // K / 128, rounded up
    uint32_t limb_rows;  // rows of one limb plane in the B tensor map
    uint32_t a_rows;     // rows per K block of the K-block-major A operand (n_out padded to 128)
    uint32_t epi;
    const int64_t* scales;  // [n_out]
    int64_t* y;             // STORE: y[t][n]; SILU: h[t][n / 2]
    int32_t* x32;           // RESID: the residual stream x[t][n] updated (|x| <= 2^24 after the clamp)
    uint32_t ldy;           // row stride of y (elements)
    // SILU: also the three limb planes of h for the next GEMM, [3][limb_rows_out][ldp] bytes
    uint8_t* planes;
    uint32_t limb_rows_out, ldp;
    const int64_t* lut;     // exp LUT (SILU)
    uint32_t* wide;         // set to 1 if an output needs more than 3 limbs (SILU planes)
    // split-K (few output tiles, e.g. decode batches): ksplit CTAs share a
    // tile; each adds its int32 limb partials into the tile's accumulator
    // with red.global.add (integer sums: exact in any order, and the total
    // is the unsplit int32 accumulator, so no overflow), the last one to
    // finish reads it once, zeroes it and runs the epilogue.
    uint32_t ksplit;
    // stream-K instead (streamk != 0; ksplit ignored): CTA c of G takes the
    // contiguous run [c T / G, (c + 1) T / G) of the T = tiles x n_kblk K
    // blocks in tile order, so every CTA streams the same number of weight
    // bytes (+-1 block) whatever the tile count; a tile shared by several
    // CTAs is finished like a split-K tile by the last piece to arrive.
    uint32_t streamk;
    int32_t* partial;       // [tiles][3][BN / 2][128] int64 token-pair sums, zero between launches (the last CTA resets)
    uint32_t* tile_cnt;     // [tiles], zero between launches (the last CTA resets)
    // tile order: 0 = feature tiles fastest (concurrent CTAs share the token
    // tile; weights re-read per token tile), 1 = token tiles fastest
    // (concurrent CTAs share the weight tile, which streams from HBM once;
    // the activation planes are re-read and must fit L2)
    uint32_t token_fast;
#ifdef TG_TRACE
    uint64_t* trace;        // [grid][128] globaltimer stamps (tools/gemm_bench.cu)
#endif
};

__device__ __forceinline__ uint64_t tg_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- PTX wrappers --------------------------------------------------------------

__device__ __forceinline__ uint32_t tg_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tg_mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tg_smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void tg_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tg_smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tg_mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(tg_smem_u32(b)), "r"(parity)
            : "memory");
    }
}


__device__ __forceinline__ void tg_tma_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            tg_smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tg_smem_u32(bar))
        : "memory");
}

// Warp-wide forms of the single-thread instructions: the whole (converged)
// warp executes them and one elected lane issues. The operands are then
// provably warp-uniform and go straight to uniform registers; issued from a
// `lane == 0` branch instead, every tcgen05.mma / TMA went through a
// divergent R2UR.BROADCAST waterfall loop that cost ~120 cycles per MMA
// (tools/mma_rate.cu), three times the N <= 64 MMA time itself.
__device__ __forceinline__ void tg_expect_tx_w(uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(tg_smem_u32(b)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void tg_tma_2d_w(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(
            tg_smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tg_smem_u32(bar))
        : "memory");
}

// K-major operand in the 128B-swizzled canonical layout: 128-byte rows,
// 8-row core groups 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t tg_desc(uint32_t smem_addr) {
    return uint64_t((smem_addr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Instruction descriptor, kind::i8: D s32, A = W (s8), B = signed digits
// (s8), both K-major, M = 128, N = n (multiple of 16, <= 256).
__host__ __device__ constexpr uint32_t tg_idesc(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(TG_BM >> 4) << 24);
}

__device__ __forceinline__ void tg_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tg_mma_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tg_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     tg_smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tg_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(tg_smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tg_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tg_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tg_ld16(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tg_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- the kernel ---------------------------------------------------------------------

template <int BN>
__device__ __forceinline__ void tg_tile(uint32_t tile, uint32_t n_mt, uint32_t n_tt, uint32_t token_fast,
                                        uint32_t& n0, uint32_t& t0) {
    if (token_fast) {
        n0 = (tile / n_tt) * TG_BM;
        t0 = (tile % n_tt) * BN;
    } else {
        n0 = (tile % n_mt) * TG_BM;
        t0 = (tile / n_mt) * BN;
    }
}

// One CTA's work, in the same order for the producer, the MMA issuer and the
// epilogue: items (tile, K split) strided over the grid, or with stream-K one
// contiguous run of K blocks cut at tile boundaries into pieces. `pieces` =
// how many CTAs contribute to the tile (1: no partial sums).
struct TgIter {
    uint32_t item, g, g1, nk, ksplit, n_items, n_tiles, G;
    bool sk;
    __device__ __forceinline__ TgIter(const TgArgs& a, uint32_t tiles) {
        nk = a.n_kblk;
        n_tiles = tiles;
        G = gridDim.x;
        sk = a.streamk != 0;
        ksplit = a.ksplit ? a.ksplit : 1;
        n_items = tiles * ksplit;
        item = blockIdx.x;
        const uint64_t T = uint64_t(tiles) * nk;
        g = uint32_t(T * blockIdx.x / G);
        g1 = uint32_t(T * (blockIdx.x + 1) / G);
    }
    // the CTA whose run holds K block b: the largest c with c T / G <= b
    __device__ __forceinline__ uint32_t cta_of(uint64_t b) const {
        return uint32_t(((b + 1) * G - 1) / (uint64_t(n_tiles) * nk));
    }
    __device__ __forceinline__ bool next(uint32_t& tile, uint32_t& kb0, uint32_t& kb1, uint32_t& pieces);
};

// work item -> (tile, K-block range)
__device__ __forceinline__ void tg_item(uint32_t item, uint32_t ksplit, uint32_t n_kblk, uint32_t& tile,
                                        uint32_t& ks, uint32_t& kb0, uint32_t& kb1) {
    tile = item / ksplit;
    ks = item % ksplit;
    kb0 = uint32_t(uint64_t(n_kblk) * ks / ksplit);
    kb1 = uint32_t(uint64_t(n_kblk) * (ks + 1) / ksplit);
}

__device__ __forceinline__ bool TgIter::next(uint32_t& tile, uint32_t& kb0, uint32_t& kb1, uint32_t& pieces) {
    if (sk) {
        if (g >= g1) return false;
        tile = g / nk;
        kb0 = g - tile * nk;
        kb1 = min(nk, kb0 + (g1 - g));
        g += kb1 - kb0;
        pieces = cta_of(uint64_t(tile + 1) * nk - 1) - cta_of(uint64_t(tile) * nk) + 1;
        return true;
    }
    if (item >= n_items) return false;
    uint32_t ks;
    tg_item(item, ksplit, nk, tile, ks, kb0, kb1);
    pieces = ksplit;
    item += G;
    return true;
}

template <int BN>
__global__ void __launch_bounds__(TgShape<BN>::THREADS, TgShape<BN>::MIN_BLOCKS)
    limb_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const TgArgs a) {
    using S = TgShape<BN>;
    extern __shared__ uint8_t tg_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tg_smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[S::STAGES], empty[S::STAGES], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_slot, s_last;
    __shared__ int64_t s_lut[257];  // exp LUT for the SILU epilogue

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef TG_TRACE
    uint64_t* tr = a.trace + size_t(blockIdx.x) * 128;
    if (threadIdx.x == 0) tr[0] = tg_now();
#endif
    const uint32_t n_mt = (a.n_out + TG_BM - 1) / TG_BM, n_tt = (a.n_tok + BN - 1) / BN;
    const uint32_t n_tiles = n_mt * n_tt;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S::STAGES; ++s) {
            tg_mbar_init(&full[s], 1);
            tg_mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tg_mbar_init(&acc_full[b], 1);
            tg_mbar_init(&acc_empty[b], S::EPI_WARPS);  // every epilogue warp releases the set
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: two accumulator sets of 3 x BN columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tg_smem_u32(&tmem_slot)), "n"(S::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tg_fence_before();
    __syncthreads();
    tg_fence_after();
    const uint32_t tmem = tmem_slot;
    pdl_launch_dependents();
#ifdef TG_TRACE
    if (threadIdx.x == 0) tr[1] = tg_now();
#endif

    if (warp == 0) {
        // TMA producer (the whole warp walks the loop, one lane issues): the K
        // slices of every work item of this CTA, in order. The weights are
        // constant: the first ring of A tiles streams in while the previous
        // kernel (which writes the B planes) finishes.
        uint32_t it = 0;
        TgIter w0(a, n_tiles);
        uint32_t tile, kb0, kb1, pieces, n0, t0;
        while (it < S::STAGES && w0.next(tile, kb0, kb1, pieces)) {
            tg_tile<BN>(tile, n_mt, n_tt, a.token_fast, n0, t0);
            for (uint32_t kb = kb0; kb < kb1 && it < S::STAGES; ++kb, ++it) {
                tg_expect_tx_w(&full[it], S::STAGE_BYTES);
                tg_tma_2d_w(smem + size_t(it) * S::STAGE_BYTES, &tmA, 0, int32_t(kb * a.a_rows + n0), &full[it]);
            }
        }
        const uint32_t pre = it;
        pdl_wait();
#ifdef TG_TRACE
        if (lane == 0) tr[2] = tg_now();
#endif
        it = 0;
        TgIter w1(a, n_tiles);
        while (w1.next(tile, kb0, kb1, pieces)) {
            tg_tile<BN>(tile, n_mt, n_tt, a.token_fast, n0, t0);
            for (uint32_t kb = kb0; kb < kb1; ++kb, ++it) {
                const uint32_t s = it % S::STAGES;
                uint8_t* st = smem + size_t(s) * S::STAGE_BYTES;
                if (it >= pre) {
                    if (it >= S::STAGES) tg_mbar_wait(&empty[s], ((it / S::STAGES) & 1) ^ 1);
#ifdef TG_TRACE
                    if (lane == 0 && it < 40) tr[8 + it] = tg_now();
#endif
                    tg_expect_tx_w(&full[s], S::STAGE_BYTES);
                    tg_tma_2d_w(st, &tmA, 0, int32_t(kb * a.a_rows + n0), &full[s]);  // K-block-major A
                }
#pragma unroll
                for (int l = 0; l < TG_L; ++l)
                    tg_tma_2d_w(st + TG_A_BYTES + l * S::B_BYTES, &tmB, int32_t(kb * TG_BK), int32_t(l * a.limb_rows + t0),
                                &full[s]);
            }
        }
    } else if (warp == 1) {
        // MMA issuer (whole warp, one elected lane issues)
        uint32_t it = 0, j = 0;
        TgIter w(a, n_tiles);
        uint32_t tile, kb0, kb1, pieces;
        for (; w.next(tile, kb0, kb1, pieces); ++j) {
            const uint32_t b = j % S::NB;
            if (j >= S::NB) tg_mbar_wait(&acc_empty[b], ((j / S::NB) & 1) ^ 1);  // epilogue drained set b
            tg_fence_after();
            const uint32_t dacc = tmem + b * S::ACC;
            for (uint32_t kb = kb0; kb < kb1; ++kb, ++it) {
                const uint32_t s = it % S::STAGES;
                tg_mbar_wait(&full[s], (it / S::STAGES) & 1);
#ifdef TG_TRACE
                if (lane == 0 && it < 40) tr[48 + it] = tg_now();
#endif
                tg_fence_after();
                const uint32_t sa = tg_smem_u32(smem + size_t(s) * S::STAGE_BYTES);
                // the three limb tiles are contiguous 128B-swizzled rows: one
                // MMA with N = 3 BN reads them all (column l BN + t = limb l of token t)
#pragma unroll
                for (int kk = 0; kk < TG_BK / 32; ++kk)  // K = 32 bytes per MMA
                    tg_mma_w(dacc, tg_desc(sa + 32 * kk), tg_desc(sa + TG_A_BYTES + 32 * kk), tg_idesc(TG_L * BN),
                             (kb != kb0) || (kk != 0));
                tg_commit_w(&empty[s]);  // frees the stage once these MMAs have read it
            }
            tg_commit_w(&acc_full[b]);
        }
    } else {
        // epilogue: thread = feature n, columns = tokens
        if (a.epi == TG_SILU) {  // constant: before the dependency wait
            for (int i = threadIdx.x - 64; i < 257; i += 32 * S::EPI_WARPS) s_lut[i] = a.lut[i];
            asm volatile("bar.sync 1, %0;" ::"n"(32 * S::EPI_WARPS) : "memory");
        }
        pdl_wait();  // reads / writes data the previous kernels own
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        constexpr uint32_t NH = S::EPI_WARPS / 4;      // warps per lane quarter
        const uint32_t c_first = 16 * ((warp - 2) / 4);  // this warp's first 16-column chunk
        const uint32_t fl = 32 * q + lane;  // feature within the tile
        uint32_t j = 0;
        TgIter w(a, n_tiles);
        uint32_t tile, kb0, kb1, pieces, n0, t0;
        for (; w.next(tile, kb0, kb1, pieces); ++j) {
            tg_tile<BN>(tile, n_mt, n_tt, a.token_fast, n0, t0);
            const uint32_t b = j % S::NB;
            const uint32_t n = n0 + fl;
            const bool nv = n < a.n_out;
            tg_mbar_wait(&acc_full[b], (j / S::NB) & 1);
            tg_fence_after();
            const uint32_t tbase = tmem + ((32 * q) << 16) + b * S::ACC;
            // split-K accumulator of the tile: int32 sums of token pairs (2c, 2c + 1)
            // packed into one int64 word lo + 2^32 hi -- a 64-bit add sums both
            // exactly (each total fits int32), halving the atomics
            unsigned long long* part =
                pieces > 1 ? reinterpret_cast<unsigned long long*>(a.partial) + size_t(tile) * (TG_L * (BN / 2) * TG_BM)
                           : nullptr;
            bool last = true;
            if (pieces > 1) {
                // this split's partials added into the tile accumulator (fire and
                // forget); token columns past the batch are skipped (never read)
                const uint32_t nvalid = a.n_tok - t0;
                for (uint32_t c0 = c_first; c0 < BN; c0 += 16 * NH) {
                    int32_t d[TG_L][16];
#pragma unroll
                    for (int l = 0; l < TG_L; ++l) tg_ld16(tbase + l * BN + c0, d[l]);
                    tg_ld_wait();
#pragma unroll
                    for (int l = 0; l < TG_L; ++l)
#pragma unroll
                        for (int jj = 0; jj < 16; jj += 2)
                            if (c0 + jj < nvalid)
                                asm volatile("red.global.add.u64 [%0], %1;" ::"l"(part + (size_t(l) * (BN / 2) + (c0 + jj) / 2) * TG_BM + fl),
                                             "l"(uint64_t(int64_t(d[l][jj])) + (uint64_t(uint32_t(d[l][jj + 1])) << 32))
                                             : "memory");
                }
                tg_fence_before();
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tg_smem_u32(&acc_empty[b])) : "memory");
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(32 * S::EPI_WARPS) : "memory");
                if (threadIdx.x == 64) s_last = atomicAdd(a.tile_cnt + tile, 1u) == pieces - 1;
                asm volatile("bar.sync 1, %0;" ::"n"(32 * S::EPI_WARPS) : "memory");
                last = s_last != 0;
                if (last) {
                    __threadfence();
                    if (threadIdx.x == 64) a.tile_cnt[tile] = 0;  // ready for the next launch
                }
            }
            if (!last) continue;
            const int64_t sc = nv ? a.scales[n] : 0;
            for (uint32_t c0 = c_first; c0 < BN; c0 += 16 * NH) {
                int32_t d[TG_L][16];
                if (pieces > 1) {
                    // the summed accumulator: 24 independent loads, then zero it for the next launch
                    unsigned long long sp[TG_L][8];
#pragma unroll
                    for (int l = 0; l < TG_L; ++l)
#pragma unroll
                        for (int jp = 0; jp < 8; ++jp) sp[l][jp] = __ldcg(part + (size_t(l) * (BN / 2) + c0 / 2 + jp) * TG_BM + fl);
#pragma unroll
                    for (int l = 0; l < TG_L; ++l)
#pragma unroll
                        for (int jp = 0; jp < 8; ++jp) {
                            __stcg(part + (size_t(l) * (BN / 2) + c0 / 2 + jp) * TG_BM + fl, 0ull);
                            const int32_t lo = int32_t(uint32_t(sp[l][jp]));  // exact: the total fits int32
                            d[l][2 * jp] = lo;
                            d[l][2 * jp + 1] = int32_t(uint32_t((sp[l][jp] - uint64_t(int64_t(lo))) >> 32));
                        }
                } else {
#pragma unroll
                    for (int l = 0; l < TG_L; ++l) tg_ld16(tbase + l * BN + c0, d[l]);
                    tg_ld_wait();
                    if (c0 + 16 * NH >= BN) {  // this warp's columns of set b are in registers: hand it back
                        tg_fence_before();
                        __syncwarp();
                        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tg_smem_u32(&acc_empty[b])) : "memory");
                    }
                }
                int64_t val[16];  // the limb accumulators recombined and scaled (d dies here)
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    val[jj] = scale_row(int64_t(d[0][jj]) + (int64_t(d[1][jj]) << 8) + (int64_t(d[2][jj]) << 16), sc);
                if (a.epi == TG_SILU) {
                    // rows (2i, 2i+1) = (gate_i, up_i) sit on adjacent lanes; the
                    // pair splits the tokens (even lane: even tokens, odd lane: odd
                    // ones), so every lane runs half the SiLUs, branch-free
                    const uint32_t odd = n & 1, i = n >> 1;
                    const size_t plane = size_t(a.limb_rows_out) * a.ldp;
                    bool bad = false;
#pragma unroll
                    for (int jp = 0; jp < 8; ++jp) {
                        const int64_t ve = val[2 * jp], vo = val[2 * jp + 1];
                        const int64_t recv = __shfl_xor_sync(0xffffffffu, odd ? ve : vo, 1);
                        const int64_t g = odd ? recv : ve, u = odd ? vo : recv;
                        const uint32_t t = t0 + c0 + 2 * jp + odd;
                        const int64_t hv = mul16(silu_q16(g, s_lut), u);
                        if (nv && t < a.n_tok) {
                            if (a.y) a.y[size_t(t) * a.ldy + i] = hv;
                            bad |= !put_sdigits(a.planes + size_t(t) * a.ldp + i, plane, hv);
                        }
                    }
                    if (bad) *a.wide = 1;
                } else {
                    // RESID: all 16 residual loads in flight before the first store
                    // (the compiler may not hoist a load above a possibly aliasing store)
                    if (a.epi == TG_RESID) {
                        int32_t xold[16];
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const uint32_t t = t0 + c0 + jj;
                            xold[jj] = nv && t < a.n_tok ? a.x32[size_t(t) * a.ldy + n] : 0;
                        }
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const uint32_t t = t0 + c0 + jj;
                            if (nv && t < a.n_tok) a.x32[size_t(t) * a.ldy + n] = int32_t(add_clamp(xold[jj], val[jj]));
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const uint32_t t = t0 + c0 + jj;
                            if (nv && t < a.n_tok) a.y[size_t(t) * a.ldy + n] = val[jj];
                        }
                    }
                }
            }
        }
    }
    tg_fence_before();
    __syncthreads();
#ifdef TG_TRACE
    if (threadIdx.x == 0) tr[3] = tg_now();
#endif
    if (warp == 1) {
        tg_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(S::TMEM_COLS) : "memory");
    }
}

}  // namespace dimg::dev
