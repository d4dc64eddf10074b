// Sizing for the split-K (column) GEMV hand-off of the persistent decode kernel:
//   red  : G CTAs each red.global.add.u64 one partial per row into the same
//          R-row int64 accumulator (the WO / w_down split-K reduction)
//   bar  : bare grid-barrier round trip (counter barrier, 148 CTAs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_red tools/microbench_red.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__global__ void red_kernel(unsigned long long* acc, uint32_t R, int reps) {
    for (int r = 0; r < reps; ++r)
        for (uint32_t i = threadIdx.x; i < R; i += blockDim.x)
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(acc + i), "l"((unsigned long long)(i + blockIdx.x)) : "memory");
}

__global__ void red_distinct_kernel(unsigned long long* acc, uint32_t R, int reps) {
    for (int r = 0; r < reps; ++r)
        for (uint32_t i = threadIdx.x; i < R; i += blockDim.x)
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(acc + size_t(blockIdx.x) * R + i), "l"((unsigned long long)i)
                         : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const unsigned int* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void bar_kernel(unsigned int* bar, int n) {
    for (int k = 0; k < n; ++k) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(bar, 1u);
            const uint32_t target = (k + 1) * gridDim.x;
            while (ld_acquire(bar) < target) {
            }
        }
        __syncthreads();
    }
}

__global__ void bar_red_kernel(unsigned int* bar, int n) {  // arrive with red.release, poll relaxed
    for (int k = 0; k < n; ++k) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            const uint32_t target = (k + 1) * gridDim.x;
            uint32_t v;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            } while (v < target);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    unsigned long long* acc;
    CK(cudaMalloc(&acc, size_t(sms) * 16384 * 8));
    for (uint32_t R : {4096u, 8192u}) {
        for (int G : {128, sms}) {
            const int reps = 20;
            red_kernel<<<G, 256>>>(acc, R, 1);
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            red_kernel<<<G, 256>>>(acc, R, reps);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double n = double(G) * R * reps;
            printf("red same-addr R=%u G=%d: %.3f us per round (%.1f G red/s)\n", R, G, ms * 1e3 / reps,
                   n / (ms * 1e-3) / 1e9);
            CK(cudaEventRecord(e0));
            red_distinct_kernel<<<G, 256>>>(acc, R, reps);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("red distinct  R=%u G=%d: %.3f us per round (%.1f G red/s)\n", R, G, ms * 1e3 / reps,
                   n / (ms * 1e-3) / 1e9);
        }
    }
    unsigned int* bar;
    CK(cudaMalloc(&bar, 256));
    for (int variant = 0; variant < 2; ++variant) {
        const int n = 2000;
        for (int it = 0; it < 2; ++it) {
            CK(cudaMemset(bar, 0, 256));
            int nn = n;
            void* args[] = {&bar, &nn};
            CK(cudaEventRecord(e0));
            CK(cudaLaunchCooperativeKernel(variant ? (void*)bar_red_kernel : (void*)bar_kernel, sms, 256, args, 0, 0));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (it) printf("grid barrier (%s): %.3f us each\n", variant ? "red.release" : "fence+atomic", ms * 1e3 / n);
        }
    }
    return 0;
}
