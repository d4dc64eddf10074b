// prologue_norm (persistent.cuh) in isolation: one CTA, fake NORM stage,
// clock64 stamps from the function's own trace hooks.
#include <cstdio>
#include "kernels/persistent.cuh"
using namespace dimg::dev;

__global__ void bench(PkArgs a, PkStage st, unsigned long long* tr, int iters) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ u128 red[32];
    __shared__ int64_t s_seeds[64];
    if (threadIdx.x < 64) s_seeds[threadIdx.x] = a.seeds[threadIdx.x];
    __syncthreads();
    a.seeds = s_seeds;
    int64_t* xb = reinterpret_cast<int64_t*>(smem);
    uint32_t* planes = reinterpret_cast<uint32_t*>(xb + st.Kp);
    unsigned long long acc[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        unsigned long long t[12];
        t[8] = clock64();
        prologue_norm(a, st, 0, xb, planes, red, threadIdx.x == 0 ? t : nullptr);
        unsigned long long end = clock64();
        if (threadIdx.x == 0) {
            acc[0] += t[4] - t[8];
            acc[1] += t[5] - t[4];
            acc[2] += t[6] - t[5];
            acc[3] += t[7] - t[6];
        }
        (void)end;
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) tr[k] = acc[k] / iters;
}

int main() {
    const int K = 4096;
    int64_t* hx = new int64_t[K];
    for (int i = 0; i < K; ++i) hx[i] = int64_t((i * 2654435761u) % 300000) - 150000;
    int64_t hs[64];
    for (int b = 0; b < 64; ++b) hs[b] = (int64_t(1) << 48) >> (b / 2);
    int64_t *dx, *ds;
    unsigned long long* dt;
    Ctl* ctl;
    cudaMalloc(&dx, K * 8);
    cudaMalloc(&ds, 512);
    cudaMalloc(&dt, 64);
    cudaMalloc(&ctl, sizeof(Ctl));
    cudaMemset(ctl, 0, sizeof(Ctl));
    cudaMemcpy(dx, hx, K * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs, 512, cudaMemcpyHostToDevice);
    PkArgs a{};
    a.seeds = ds;
    a.ctl = ctl;
    PkStage st{};
    st.kind = SK_GEMV; st.mode = MODE_NORM; st.K = K; st.Kp = K; st.gamma_unit = 1; st.x = dx;
    size_t smem = size_t(K) * 16;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bench<<<1, PK_THREADS, smem>>>(a, st, dt, 100);
    unsigned long long h[4];
    cudaError_t e = cudaMemcpy(h, dt, 32, cudaMemcpyDeviceToHost);
    printf("%s cycles: stage-x %llu  reduce %llu  r %llu  normalise+pack %llu\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
}
