// Issue rate of tcgen05.mma (cta_group::1, M = 128, both operands in shared
// memory, 128B-swizzled K-major descriptors as in kernels/tc_gemm.cuh):
// cycles per instruction for kind::i8 (K = 32 bytes) and kind::f16 (K = 16
// halves) at several N, operands resident (no TMA), R back-to-back MMAs into
// one accumulator, then one commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//        -Ipaper_2603_24904_b200/csrc -o tools/_libs/mma_rate tools/mma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/tc_gemm.cuh"

using namespace dimg::dev;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

// kind::f16 idesc: D f32 (c_format 1), A/B bf16 (format 1), K-major, M 128
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

// variant bits: 1 = rotate over 4 stage buffers (A 16 KB + B 24 KB each);
// 2 = tcgen05.fence::after_thread_sync per K block; 4 = tcgen05.commit per
// K block; 8 = wait for the commit two K blocks back (ring hand-off)
constexpr int STG = 40960;
template <int N, bool F16>
__global__ void __launch_bounds__(128, 1) rate_kernel(int R, unsigned long long* out, int variant) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar, kbar[4];
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 4 * STG; i += blockDim.x) smem[i] = uint8_t(i * 37);
    if (threadIdx.x == 0) {
        tg_mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) tg_mbar_init(&kbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tg_smem_u32(&slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tg_fence_before();
    __syncthreads();
    tg_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t base = tg_smem_u32(smem);
        const long long t0 = clock64();
        for (int r = 0, kb = 0; r < R; r += 4, ++kb) {
            const uint32_t sa = base + ((variant & 1) ? (kb & 3) * STG : 0), sb = sa + 16384;
            if ((variant & 8) && kb >= 2) tg_mbar_wait(&kbar[(kb - 2) & 3], ((kb - 2) >> 2) & 1);
            if (variant & 2) tg_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (F16) mma_f16(tmem, tg_desc(sa + 32 * kk), tg_desc(sb + 32 * kk), idesc_bf16(N), 1);
                else tg_mma(tmem, tg_desc(sa + 32 * kk), tg_desc(sb + 32 * kk), tg_idesc(N), 1);
            }
            if (variant & 4) tg_commit(&kbar[kb & 3]);
        }
        tg_commit(&bar);
        tg_mbar_wait(&bar, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) *out = (unsigned long long)(t1 - t0);
    }
    tg_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tg_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    }
}

template <int N, bool F16>
void run(int grid, int variant = 0) {
    const int smem = 4 * STG + 1024;
    cudaFuncSetAttribute(rate_kernel<N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int R = 4096;
    rate_kernel<N, F16><<<grid, 128, smem>>>(R, d, variant);
    rate_kernel<N, F16><<<grid, 128, smem>>>(R, d, variant);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const double per = double(cyc) / R;
    const double macs = 128.0 * N * (F16 ? 16 : 32);
    printf("%s N=%3d grid=%3d variant %d: %.1f cyc/MMA  (%.0f MAC/cyc/SM)  %s\n", F16 ? "f16" : "i8 ", N, grid, variant,
           per, macs / per,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

// Whole-GPU dense kind::i8 rate: one CTA per SM issuing N = 192 MMAs back to
// back (operands resident), CUDA-event timed: the roofline denominator of the
// tensor-core prefill (bench.py reads profiles/r02_mma_rate.json).
void peak() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int smem = 4 * STG + 1024;
    cudaFuncSetAttribute(rate_kernel<192, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int R = 1 << 16;
    rate_kernel<192, false><<<sms, 128, smem>>>(R, d, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate_kernel<192, false><<<sms, 128, smem>>>(R, d, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * sms * double(R) * 128 * 192 * 32;
    printf("{\"i8_tops\": %.1f, \"sms\": %d, \"ms\": %.3f, \"N\": 192, \"mmas_per_sm\": %d, "
           "\"max_clock_mhz\": %d, \"err\": \"%s\"}\n",
           ops / (ms * 1e-3) / 1e12, sms, ms, R, clk / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'p') {
        peak();
        return 0;
    }
    for (int v : {0, 1, 3, 5, 7, 13, 15}) {
        run<16, false>(1, v);
        run<48, false>(1, v);
        run<192, false>(1, v);
    }
    return 0;
}
