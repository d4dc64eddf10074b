// Timing harness for the tensor-core limb GEMM (kernels/tc_gemm.cuh) alone:
// CUDA events around R launches that cycle through enough weight copies to
// exceed L2, so every launch streams its weights from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//        -Ipaper_2603_24904_b200/csrc -Iinclude -o tools/_libs/gemm_bench tools/gemm_bench.cu
//   tools/_libs/gemm_bench N K T bn ksplit epi [per_sm]     (epi 0 store, 1 resid)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels/tc_gemm.cuh"

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

using namespace dimg::dev;

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}

static CUtensorMap tmap(const void* base, uint64_t inner, uint64_t outer, uint64_t stride, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {stride};
    const cuuint32_t box[2] = {TG_BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    if (enc()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("tmap failed\n");
        exit(1);
    }
    return m;
}

__global__ void fill_kernel(uint8_t* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = uint8_t((i * 2654435761u + seed) >> 13);
}

static bool g_pdl = false;
static cudaStream_t g_st = nullptr;

template <int BN>
static void launch(const CUtensorMap& ta, const CUtensorMap& tb, const TgArgs& a, uint32_t grid) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = TgShape<BN>::THREADS;
    cfg.dynamicSmemBytes = TgShape<BN>::SMEM;
    cfg.stream = g_st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, limb_gemm_kernel<BN>, ta, tb, a));
}

__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 1000) *p = 1;
}

int main(int argc, char** argv) {
    if (argc == 2) {  // gemm_bench G: back-to-back empty launches of G CTAs
        const int G = atoi(argv[1]), R = 1000;
        for (int i = 0; i < 10; ++i) empty_kernel<<<G, 192>>>(nullptr);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        for (int i = 0; i < R; ++i) empty_kernel<<<G, 192>>>(nullptr);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("empty kernel, %d CTAs: %.2f us per launch\n", G, 1e3 * ms / R);
        return 0;
    }
    if (argc < 7) {
        printf("usage: gemm_bench N K T bn ksplit epi [per_sm]\n");
        return 1;
    }
    const uint32_t N = atoi(argv[1]), K = atoi(argv[2]), T = atoi(argv[3]), bn = atoi(argv[4]),
                   ks = atoi(argv[5]), epi = atoi(argv[6]);
    const uint32_t per_sm = argc > 7 ? atoi(argv[7]) : (bn == 16 ? 2 : 1);
    CK(cudaFuncSetAttribute(limb_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TgShape<64>::SMEM));
    CK(cudaFuncSetAttribute(limb_gemm_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, TgShape<16>::SMEM));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t kblk = (K + 127) / 128, rows128 = (N + 127) / 128 * 128, Kp = kblk * 128;
    const uint32_t Tp = (T + 63) / 64 * 64;
    const size_t wbytes = size_t(kblk) * rows128 * 128;
    const int nbuf = int(std::max<size_t>(2, (400u << 20) / wbytes + 1));
    std::vector<uint8_t*> W(nbuf);
    for (int i = 0; i < nbuf; ++i) {
        CK(cudaMalloc(&W[i], wbytes));
        fill_kernel<<<1024, 256>>>(W[i], wbytes, i);
    }
    uint8_t* planes;
    CK(cudaMalloc(&planes, size_t(3) * Tp * Kp));
    fill_kernel<<<1024, 256>>>(planes, size_t(3) * Tp * Kp, 99);
    int64_t *sc, *y;
    CK(cudaMalloc(&sc, size_t(N) * 8));
    CK(cudaMemset(sc, 0, size_t(N) * 8));
    CK(cudaMalloc(&y, size_t(T) * N * 8));
    CK(cudaMemset(y, 0, size_t(T) * N * 8));
    const uint32_t tiles = (rows128 / 128) * ((T + bn - 1) / bn);
    int32_t* partial;
    uint32_t* cnt;
    CK(cudaMalloc(&partial, size_t(tiles) * 3 * bn * 128 * 4));
    CK(cudaMemset(partial, 0, size_t(tiles) * 3 * bn * 128 * 4));
    CK(cudaMalloc(&cnt, size_t(tiles) * 4));
    CK(cudaMemset(cnt, 0, size_t(tiles) * 4));
    std::vector<CUtensorMap> ta(nbuf);
    for (int i = 0; i < nbuf; ++i) ta[i] = tmap(W[i], 128, size_t(kblk) * rows128, 128, 128);
    const CUtensorMap tb = tmap(planes, K, size_t(3) * Tp, Kp, bn);
    TgArgs a{};
    a.n_out = N;
    a.a_rows = rows128;
    a.n_tok = T;
    a.n_kblk = kblk;
    a.limb_rows = Tp;
    a.epi = epi;
    a.scales = sc;
    a.y = y;
    a.ldy = N;
    if (epi == TG_SILU) {  // exp LUT (any values in range), output planes for the next GEMM
        std::vector<int64_t> lut(257);
        for (int i = 0; i < 257; ++i) lut[i] = (int64_t(i) << 8);
        int64_t* dl;
        CK(cudaMalloc(&dl, 257 * 8));
        CK(cudaMemcpy(dl, lut.data(), 257 * 8, cudaMemcpyHostToDevice));
        a.lut = dl;
        a.y = nullptr;
        a.ldp = N / 2;
        a.limb_rows_out = Tp;
        CK(cudaMalloc(&a.planes, size_t(3) * Tp * a.ldp));
        CK(cudaMalloc(&a.wide, 4));
    }
    a.ksplit = std::max(1u, ks);
    a.partial = partial;
    a.tile_cnt = cnt;
    const uint32_t items = tiles * a.ksplit;
    const uint32_t grid = std::min<uint32_t>(items, per_sm * sms);
#ifdef TG_TRACE
    CK(cudaMalloc(&a.trace, size_t(grid) * 128 * 8));
    CK(cudaMemset(a.trace, 0, size_t(grid) * 128 * 8));
#endif
    auto go = [&](int i) {
        if (bn == 16) launch<16>(ta[i % nbuf], tb, a, grid);
        else launch<64>(ta[i % nbuf], tb, a, grid);
    };
    // GB_PDL=1: programmatic dependent launches; GB_GRAPH=1: the R launches
    // replayed from one CUDA graph (no host launch cost)
    g_pdl = getenv("GB_PDL") && atoi(getenv("GB_PDL"));
    const bool graph = getenv("GB_GRAPH") && atoi(getenv("GB_GRAPH"));
    CK(cudaStreamCreateWithFlags(&g_st, cudaStreamNonBlocking));
    for (int i = 0; i < 10; ++i) go(i);
    CK(cudaDeviceSynchronize());
    const int R = 200;
    cudaGraphExec_t ge = nullptr;
    if (graph) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(g_st, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < R; ++i) go(i);
        CK(cudaStreamEndCapture(g_st, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, g_st));
        CK(cudaStreamSynchronize(g_st));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, g_st));
    if (graph) CK(cudaGraphLaunch(ge, g_st));
    else
        for (int i = 0; i < R; ++i) go(i);
    CK(cudaEventRecord(e1, g_st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = 1e3 * ms / R;
#ifdef TG_TRACE
    {  // the last launch's timeline, CTA 0 and the slowest CTA (ns from CTA 0's start)
        std::vector<uint64_t> h(size_t(grid) * 128);
        CK(cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost));
        uint64_t t0 = ~0ull, tend = 0;
        uint32_t slow = 0;
        for (uint32_t c = 0; c < grid; ++c) {
            t0 = std::min(t0, h[size_t(c) * 128]);
            if (h[size_t(c) * 128 + 3] > tend) { tend = h[size_t(c) * 128 + 3]; slow = c; }
        }
        for (uint32_t c : {0u, slow}) {
            const uint64_t* r = &h[size_t(c) * 128];
            printf("CTA %u: start %lld setup %lld wait %lld end %lld\n  issue:", c, (long long)(r[0] - t0),
                   (long long)(r[1] - t0), (long long)(r[2] - t0), (long long)(r[3] - t0));
            for (int k = 0; k < 40; ++k) if (r[8 + k]) printf(" %lld", (long long)(r[8 + k] - t0));
            printf("\n  full: ");
            for (int k = 0; k < 40; ++k) if (r[48 + k]) printf(" %lld", (long long)(r[48 + k] - t0));
            printf("\n");
        }
    }
#endif
    const double ops = 2.0 * 3 * double(N) * K * T;
    printf("%s%sN=%u K=%u T=%u bn=%u ksplit=%u epi=%u grid=%u: %.2f us  %.0f GB/s (weights)  %.1f TOP/s (limb ops)\n", g_pdl ? "pdl " : "",
           graph ? "graph " : "", N, K, T, bn, a.ksplit, epi, grid, us, wbytes / us * 1e-3, ops / us * 1e-6);
    return 0;
}
