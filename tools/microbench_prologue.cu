// Cycle costs of the persistent kernel's serial pieces, run in isolation
// (one CTA of 256 threads, nothing else on the GPU): u128 block sum, the
// 128-bit Newton inv-sqrt, the normalise+pack pass, a __syncthreads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
//        -I paper_2603_24904_b200/csrc -o tools/microbench_prologue tools/microbench_prologue.cu
#include <cstdio>

#include "kernels/q16.cuh"

using namespace dimg::dev;

__global__ void bench(const int64_t* x, const int64_t* seeds_g, long long* out, int iters) {
    __shared__ int64_t xb[4096];
    __shared__ uint32_t planes[3 * 1024];
    __shared__ u128 red[32];
    __shared__ int64_t seeds[64];
    if (threadIdx.x < 64) seeds[threadIdx.x] = seeds_g[threadIdx.x];
    for (int j = threadIdx.x; j < 4096; j += blockDim.x) xb[j] = x[j];
    __syncthreads();
    long long t_sync = 0, t_sum = 0, t_r = 0, t_norm = 0;
    int64_t sink = 0;
    for (int it = 0; it < iters; ++it) {
        long long c0 = clock64();
        __syncthreads();
        long long c1 = clock64();
        u128 ss = 0;
#pragma unroll 4
        for (uint32_t j = threadIdx.x; j < 4096; j += blockDim.x) {
            const int64_t v = xb[j];
            ss += uint64_t(int64_t(int32_t(v)) * int32_t(v));
        }
        ss = block_sum_u128(ss, red);
        long long c2 = clock64();
        __shared__ int64_t s_r;
        if (threadIdx.x == 0) {
            int64_t ms = int64_t((uint64_t(ss) / 4096u) >> 16);
            s_r = inv_sqrt_q16(ms + 1, seeds);
        }
        __syncthreads();
        const int64_t r = s_r;
        long long c3 = clock64();
        int fits = 1;
#pragma unroll 2
        for (uint32_t w = threadIdx.x; w < 1024; w += blockDim.x) {
            uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t v = mul16_small(xb[4 * w + e], r);
                fits &= (v >= -(int64_t(1) << 23)) & (v < (int64_t(1) << 23));
                w0 |= uint32_t(v & 0xFF) << (8 * e);
                w1 |= uint32_t((v >> 8) & 0xFF) << (8 * e);
                w2 |= uint32_t((v >> 16) & 0xFF) << (8 * e);
            }
            planes[w] = w0;
            planes[1024 + w] = w1;
            planes[2048 + w] = w2;
        }
        fits = __syncthreads_and(fits);
        long long c4 = clock64();
        t_sync += c1 - c0;
        t_sum += c2 - c1;
        t_r += c3 - c2;
        t_norm += c4 - c3;
        sink += fits + planes[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        out[0] = t_sync / iters;
        out[1] = t_sum / iters;
        out[2] = t_r / iters;
        out[3] = t_norm / iters;
        out[4] = sink;
    }
}

int main() {
    int64_t hx[4096], hs[64];
    for (int i = 0; i < 4096; ++i) hx[i] = ((i * 2654435761u) % 300000) - 150000;
    for (int b = 0; b < 64; ++b) hs[b] = (int64_t(1) << 48) >> (b / 2);
    int64_t *dx, *ds;
    long long* dout;
    cudaMalloc(&dx, sizeof hx);
    cudaMalloc(&ds, sizeof hs);
    cudaMalloc(&dout, 5 * sizeof(long long));
    cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs, sizeof hs, cudaMemcpyHostToDevice);
    bench<<<1, 256>>>(dx, ds, dout, 200);
    long long h[5];
    cudaMemcpy(h, dout, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles: syncthreads %lld  sum+block_sum_u128 %lld  r(div+inv_sqrt) %lld  normalise+pack %lld\n", h[0],
           h[1], h[2], h[3]);
    return 0;
}
