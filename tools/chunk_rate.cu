// Per-warp consumption rate of one 6 KB weight chunk held in shared memory
// (no HBM): the decode kernel's DP4A row-group dot product (4 rows x 1536 B,
// 3 byte limbs) against warp-level int8 tensor-core MMAs (mma.sync
// m16n8k32 s8: A = the 3 signed-digit limb rows, B = 8 weight rows x 32 B per
// instruction, operands pre-arranged in fragment order so every fragment is
// one 16-byte shared load). 8 warps per CTA, one CTA per SM, 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_libs/chunk_rate tools/chunk_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int CH = 6144;  // chunk bytes
constexpr int REP = 2000;

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
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
    return r;
}
__device__ __forceinline__ void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_su(int (&c)[4], uint4 a, uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}
__device__ __forceinline__ void mma_ss2(int (&c)[4], uint4 a, uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}
constexpr int PSTR = 4096 + 64;  // plane stride (bytes): 16 words mod 32 -> conflict-free LDS.64

// mode 0: DP4A (the decode kernel's loop); mode 1: mma.sync
template <int MODE>
__global__ void __launch_bounds__(256, 1) rate(unsigned long long* out, int* sink) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* chunk = sm + warp * CH;           // this warp's weight chunk
    uint8_t* planes = sm + 8 * CH;             // 3 x 4096 B limb planes (shared by all warps)
    for (int i = threadIdx.x; i < 8 * CH + 3 * PSTR; i += 256) sm[i] = uint8_t(i * 131 + 7);
    __syncthreads();
    const uint32_t cs = static_cast<uint32_t>(__cvta_generic_to_shared(chunk));
    const uint32_t ps = static_cast<uint32_t>(__cvta_generic_to_shared(planes));
    int sum = 0;
    const long long t0 = clock64();
    if constexpr (MODE == 0) {
        for (int r = 0; r < REP; ++r) {
            int32_t acc[4][3] = {};
            for (uint32_t c = lane * 16; c < 1536; c += 512) {
                uint4 xl[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) xl[k] = lds128(ps + k * 4096 + (c + (r & 1) * 1536));
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const uint4 wv = lds128(cs + rr * 1536 + c);
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        acc[rr][k] = dp4a_su(wv.x, xl[k].x, acc[rr][k]);
                        acc[rr][k] = dp4a_su(wv.y, xl[k].y, acc[rr][k]);
                        acc[rr][k] = dp4a_su(wv.z, xl[k].z, acc[rr][k]);
                        acc[rr][k] = dp4a_su(wv.w, xl[k].w, acc[rr][k]);
                    }
                    acc[rr][2] = dp4a_ss(wv.x, xl[2].x, acc[rr][2]);
                    acc[rr][2] = dp4a_ss(wv.y, xl[2].y, acc[rr][2]);
                    acc[rr][2] = dp4a_ss(wv.z, xl[2].z, acc[rr][2]);
                    acc[rr][2] = dp4a_ss(wv.w, xl[2].w, acc[rr][2]);
                }
            }
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) sum += acc[rr][0] ^ acc[rr][1] ^ acc[rr][2];
        }
    } else if constexpr (MODE == 1) {
        // B = weights (8 rows x 32 B per mma), A = limbs (3 real rows): 24 mma
        // per chunk, 4 independent accumulators
        for (int r = 0; r < REP; ++r) {
            int c[4][4] = {};
            const bool arow = lane < 12;
#pragma unroll
            for (int j = 0; j < 24; j += 4) {
                const uint4 b0 = lds128(cs + j * 256 + lane * 16);
                const uint4 b1 = lds128(cs + (j + 2) * 256 + lane * 16);
                const uint4 a0 = arow ? lds128(ps + (r & 1) * 1536 + j * 128 + lane * 16) : make_uint4(0, 0, 0, 0);
                const uint4 a1 = arow ? lds128(ps + (r & 1) * 1536 + (j + 2) * 128 + lane * 16) : make_uint4(0, 0, 0, 0);
                mma_s8(c[0], a0.x, 0u, a0.y, 0u, b0.x, b0.y);
                mma_s8(c[1], a0.z, 0u, a0.w, 0u, b0.z, b0.w);
                mma_s8(c[2], a1.x, 0u, a1.y, 0u, b1.x, b1.y);
                mma_s8(c[3], a1.z, 0u, a1.w, 0u, b1.z, b1.w);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) sum += c[q][0] ^ c[q][1] ^ c[q][2] ^ c[q][3];
        }
    } else if constexpr (MODE >= 3) {
        // the 4-row group kept: A = 4 rows x 4 K-quarters of a 128-byte block
        // (one LDS.128 fragment), B = (quarter, limb) columns; pair MMA for
        // limbs 0/1 (u8), single MMA for limb 2 (s8); the diagonal is used.
        constexpr int NS = MODE - 1;  // independent accumulator sets (2, 3, 4)
        const int g = lane >> 2, t = lane & 3;
        const uint32_t bp_off = (g & 1) * PSTR + (g >> 1) * 32 + 8 * t;
        const uint32_t bs_off = 2 * PSTR + (g & 3) * 32 + 8 * t;
        for (int r = 0; r < REP; ++r) {
            int cp[NS][4] = {}, cq[NS][4] = {};
            const uint32_t pb = ps + (r & 1) * 1536;
#pragma unroll
            for (int kb = 0; kb < 12; ++kb) {
                const uint4 a = lds128(cs + kb * 512 + lane * 16);
                const uint2 bp = lds64(pb + kb * 128 + bp_off);
                const uint2 bq = lds64(pb + kb * 128 + bs_off);
                mma_su(cp[kb % NS], a, bp);
                mma_ss2(cq[kb % NS], a, bq);
            }
#pragma unroll
            for (int q = 0; q < NS; ++q) sum += cp[q][0] ^ cp[q][1] ^ cp[q][2] ^ cp[q][3] ^ cq[q][0] ^ cq[q][3];
        }
    } else {
        // A = weights (16 rows x 32 B per mma, one LDS.128 fragment), B = limbs
        // (N = 8, 3 real columns: lanes 0-11): 12 mma per chunk, 4 accumulators
        for (int r = 0; r < REP; ++r) {
            int c[4][4] = {};
            const bool bcol = lane < 12;
#pragma unroll
            for (int j = 0; j < 12; j += 4) {
                uint4 a[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) a[q] = lds128(cs + (j + q) * 512 + lane * 16);
                const uint4 b = bcol ? lds128(ps + (r & 1) * 1536 + j * 64 + lane * 16) : make_uint4(0, 0, 0, 0);
                mma_s8(c[0], a[0].x, a[0].y, a[0].z, a[0].w, b.x, b.y);
                mma_s8(c[1], a[1].x, a[1].y, a[1].z, a[1].w, b.z, b.w);
                mma_s8(c[2], a[2].x, a[2].y, a[2].z, a[2].w, b.x, b.w);
                mma_s8(c[3], a[3].x, a[3].y, a[3].z, a[3].w, b.z, b.y);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) sum += c[q][0] ^ c[q][1] ^ c[q][2] ^ c[q][3];
        }
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    if (sum == 0x12345) sink[0] = sum;
}

int main() {
    unsigned long long* d;
    int* sink;
    cudaMalloc(&d, 148 * 8 * 8);
    cudaMalloc(&sink, 4);
    const int smem = 8 * CH + 3 * PSTR;
    unsigned long long h[148 * 8];
    for (int mode = 0; mode < 6; ++mode) {
        auto k = mode == 0 ? rate<0> : mode == 1 ? rate<1> : mode == 2 ? rate<2> : mode == 3 ? rate<3> : mode == 4 ? rate<4> : rate<5>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int it = 0; it < 2; ++it) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<148, 256, smem>>>(d, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148 * 8; ++i) avg += h[i];
            avg /= 148 * 8;
            const double clk_per_chunk = avg / REP;
            const double bytes = 148.0 * 8 * REP * CH;
            printf("%s: %.0f clk per 6 KB chunk per warp (8 warps/SM), %.2f TB/s of weights GPU-wide (%.3f ms) %s\n",
                   mode == 0 ? "dp4a         " : mode == 1 ? "mma B=weights" : mode == 2 ? "mma A=weights" : mode == 3 ? "diag4 acc2   " : mode == 4 ? "diag4 acc3   " : "diag4 acc4   ", clk_per_chunk, bytes / (ms * 1e-3) / 1e12, ms,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
