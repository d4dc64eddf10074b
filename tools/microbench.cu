// Microbenchmarks that size the persistent decode kernel's weight pipeline on
// B200 (sm_100a):
//   ring   : per-warp cp.async.bulk rings (chunk S bytes, depth D) streaming a
//            buffer larger than L2, optionally with the 3-limb DP4A work per
//            chunk -> GB/s
//   ldg    : plain LDG.128 streaming (no smem) for comparison
//   idp    : IDP4A issue rate per SM
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ int32_t dp4a_su(int32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Each warp streams chunks w, w+W, ... of its CTA's contiguous range.
template <bool COMPUTE>
__global__ void ring_kernel(const int8_t* buf, size_t bytes, uint32_t S, uint32_t D, int* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warps = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(warps) * D * S);
    uint32_t* limbs = reinterpret_cast<uint32_t*>(bars + warps * D);  // 3 x 2048 B
    if (threadIdx.x < warps * D) mbar_init(&bars[threadIdx.x], 1);
    for (int i = threadIdx.x; i < 3 * 512; i += blockDim.x) limbs[i] = i * 2654435761u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    size_t per_cta = bytes / gridDim.x / S * S;
    const int8_t* base = buf + per_cta * blockIdx.x;
    size_t nchunks = per_cta / S;
    uint8_t* my = smem + size_t(warp) * D * S;
    uint64_t* mb = bars + warp * D;
    size_t q_issue = 0;
    for (uint32_t d = 0; d < D; ++d) {
        size_t c = warp + q_issue * warps;
        if (c < nchunks && lane == 0) {
            mbar_expect_tx(&mb[d], S);
            bulk_g2s(my + d * S, base + c * S, S, &mb[d]);
        }
        ++q_issue;
    }
    int32_t acc[4][3] = {};
    for (size_t q = 0;; ++q) {
        size_t c = warp + q * warps;
        if (c >= nchunks) break;
        uint32_t sl = q % D;
        while (!mbar_try_wait(&mb[sl], (q / D) & 1)) {
        }
        const uint8_t* slot = my + sl * S;
        if (COMPUTE) {
            const uint32_t w = S / 4;  // 4 rows of S/4 bytes
            for (uint32_t cc = lane * 16; cc < w; cc += 512) {
                uint4 xl[3];
                for (int k = 0; k < 3; ++k) xl[k] = *reinterpret_cast<const uint4*>(limbs + k * 512 + (cc % 2048) / 4);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    int4 wv = *reinterpret_cast<const int4*>(slot + r * w + cc);
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        acc[r][k] = dp4a_su(wv.x, xl[k].x, acc[r][k]);
                        acc[r][k] = dp4a_su(wv.y, xl[k].y, acc[r][k]);
                        acc[r][k] = dp4a_su(wv.z, xl[k].z, acc[r][k]);
                        acc[r][k] = dp4a_su(wv.w, xl[k].w, acc[r][k]);
                    }
                }
            }
        } else {
            acc[0][0] += slot[lane * 4];
        }
        __syncwarp();
        size_t cn = warp + q_issue * warps;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (cn < nchunks) {
                mbar_expect_tx(&mb[sl], S);
                bulk_g2s(my + sl * S, base + cn * S, S, &mb[sl]);
            }
        }
        ++q_issue;
    }
    int s = 0;
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 3; ++k) s += acc[r][k];
    if (s == 0x12345678) sink[0] = s;
}

__global__ void ldg_kernel(const int4* buf, size_t n16, int* sink) {
    int acc = 0;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int4* p = buf + i + u * stride;
            asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void idp_kernel(int iters, int* sink) {
    int a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = 1, a5 = 2, a6 = 3, a7 = 4;
    uint32_t b = 0x01020304u * (threadIdx.x | 1);
    for (int i = 0; i < iters; ++i) {
        a0 = dp4a_su(a0, b, a0); a1 = dp4a_su(a1, b, a1); a2 = dp4a_su(a2, b, a2); a3 = dp4a_su(a3, b, a3);
        a4 = dp4a_su(a4, b, a4); a5 = dp4a_su(a5, b, a5); a6 = dp4a_su(a6, b, a6); a7 = dp4a_su(a7, b, a7);
    }
    int s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 0x12345678) sink[0] = s;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const int sms = p.multiProcessorCount;
    const size_t bytes = size_t(4) << 30;
    int8_t* buf;
    int* sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto time_it = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms / 3;
    };
    {
        float ms = time_it([&] { ldg_kernel<<<sms * 4, 512>>>((const int4*)buf, bytes / 16, sink); });
        printf("ldg  LDG.128 x8 unroll                : %7.1f GB/s\n", bytes / ms / 1e6);
    }
    struct Cfg { uint32_t S, D, W; };
    {  // L2-resident source: the same ring over a 48 MB buffer streamed repeatedly
        const size_t small = size_t(48) << 20;
        for (Cfg c : std::vector<Cfg>{{6144, 3, 8}, {8192, 2, 8}, {6144, 4, 8}, {4096, 4, 8}}) {
            size_t smem = size_t(c.W) * c.D * c.S + c.W * c.D * 8 + 6144;
            CK(cudaFuncSetAttribute(ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            CK(cudaFuncSetAttribute(ring_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            float m0 = time_it([&] { ring_kernel<false><<<sms, c.W * 32, smem>>>(buf, small, c.S, c.D, sink); });
            float m1 = time_it([&] { ring_kernel<true><<<sms, c.W * 32, smem>>>(buf, small, c.S, c.D, sink); });
            printf("L2 ring S=%5u D=%u warps=%2u (%3zu KB/SM) : copy %7.1f GB/s   +dp4a %7.1f GB/s\n", c.S, c.D, c.W,
                   size_t(c.W) * c.D * c.S / 1024, small / m0 / 1e6, small / m1 / 1e6);
        }
    }
    std::vector<Cfg> cfgs = {{6144, 3, 8}, {8192, 2, 8}, {8192, 3, 8}, {16384, 2, 4}, {16384, 1, 8}, {4096, 4, 8},
                             {8192, 2, 12}, {16384, 2, 6}, {32768, 1, 6}, {4096, 2, 16}, {8192, 1, 16}};
    for (auto c : cfgs) {
        size_t smem = size_t(c.W) * c.D * c.S + c.W * c.D * 8 + 6144;
        if (smem > 227 * 1024) continue;
        CK(cudaFuncSetAttribute(ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(ring_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        float m0 = time_it([&] { ring_kernel<false><<<sms, c.W * 32, smem>>>(buf, bytes, c.S, c.D, sink); });
        float m1 = time_it([&] { ring_kernel<true><<<sms, c.W * 32, smem>>>(buf, bytes, c.S, c.D, sink); });
        printf("ring S=%5u D=%u warps=%2u (%3zu KB/SM) : copy %7.1f GB/s   +dp4a %7.1f GB/s\n", c.S, c.D, c.W,
               size_t(c.W) * c.D * c.S / 1024, bytes / m0 / 1e6, bytes / m1 / 1e6);
    }
    // per-SM fill rate when only some SMs stream (8 warps x 2 x 8 KB ring)
    for (int g : {16, 32, 64, 96, 148}) {
        const uint32_t S = 8192, D = 2, W = 8;
        size_t smem = size_t(W) * D * S + W * D * 8 + 6144;
        CK(cudaFuncSetAttribute(ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const size_t part = bytes / 148 * g;  // same bytes per CTA as the full-grid run
        float ms = time_it([&] { ring_kernel<false><<<g, W * 32, smem>>>(buf, part, S, D, sink); });
        printf("ring %3d CTAs: %7.1f GB/s total, %6.1f GB/s per SM\n", g, part / ms / 1e6, part / ms / 1e6 / g);
    }
    {
        int iters = 1 << 16;
        float ms = time_it([&] { idp_kernel<<<sms * 4, 256>>>(iters, sink); });
        double ops = double(sms) * 4 * 256 * iters * 8;
        printf("idp  IDP4A: %.2f T/s = %.1f per SM per clk @1.965GHz\n", ops / ms / 1e9,
               ops / ms / 1e-3 / sms / 1.965e9);
    }
    return 0;
}
