// Device half of include/dimg.h: model upload (HBM layout), sessions (KV
// cache + control block) and the reference-shaped entry points
// generate_greedy / forward.
//
// Every forward step runs inside ONE cooperative launch of
// decode_persistent_kernel (kernels/persistent.cuh): per layer the stages
//   QKV GEMV (rmsnorm prologue; layer 0 also embeds the token)
//   -> attention step -> WO GEMV (+residual clamp)
//   -> GATE/UP GEMV (rmsnorm prologue, silu*up epilogue)
//   -> DOWN GEMV (+residual clamp)
// then the LM_HEAD GEMV with the greedy argmax, separated by grid barriers,
// while every warp keeps streaming its next weight chunks. A whole
// generate_greedy call (P-1 prompt steps + N decode steps) is one launch; the
// position and the token ring live in device memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host/blake3.hpp"
#include "host/common.hpp"
#include "host/model.hpp"
#include "kernels/attention.cuh"
#include "kernels/gemv.cuh"
#include "kernels/persistent.cuh"
#include "kernels/tc_gemm.cuh"
#include "kernels/prefill.cuh"
#include "kernels/pf_scores.cuh"
#include "kernels/pf_pv.cuh"
#include "kernels/batch.cuh"
#include "kernels/blake3.cuh"
#include "kernels/sample.cuh"
#include "kernels/chacha.cuh"
#include "host/blake3.hpp"
#include "host/chacha20.hpp"

using namespace dimg;
using namespace dimg::dev;

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            fail(DIMG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));        \
    } while (0)

namespace {

constexpr int R_ROWS = 4;   // rows per warp group
constexpr int U_3 = 4;      // 512-byte column chunks in flight per row (3-limb path)

uint32_t pad16(uint32_t k) { return (k + 15u) & ~15u; }

// ---- per-device context: tables shared by every model/op on that device ----
struct DevCtx {
    int device = -1;
    int sm_count = 0;
    int64_t* exp_lut = nullptr;
    int64_t* seeds = nullptr;
    int smem_optin = 0;
    Ctl* op_ctl = nullptr;  // control block for the operator-level exports
    cudaStream_t op_stream = nullptr;
    // the operator exports share op_ctl / op_stream: one op at a time per
    // device (recursive: dense_tokens falls back to dense inside its scope)
    std::recursive_mutex op_mu;
};

std::mutex g_ctx_mu;
DevCtx g_ctx[64];

template <int EPI, int MODE>
void set_gemv_attrs() {
    CK(cudaFuncSetAttribute(gemv_kernel<EPI, MODE, R_ROWS, U_3>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
}

DevCtx& dev_ctx(int device) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (device < 0 || device >= 64) fail(DIMG_EINVAL, "bad device index");
    DevCtx& c = g_ctx[device];
    if (c.device >= 0) return c;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(DIMG_ECUDA, std::string("need an sm_100 GPU, found ") + prop.name);
    c.sm_count = prop.multiProcessorCount;
    int64_t lut[257], seeds[64];
    for (int i = 0; i <= 256; ++i) lut[i] = exp_lut_entry(i);
    for (int b = 0; b < 64; ++b) seeds[b] = invsqrt_seed(b);
    CK(cudaMalloc(&c.exp_lut, sizeof lut));
    CK(cudaMalloc(&c.seeds, sizeof seeds));
    CK(cudaMemcpy(c.exp_lut, lut, sizeof lut, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.seeds, seeds, sizeof seeds, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.op_ctl, sizeof(Ctl)));
    CK(cudaMemset(c.op_ctl, 0, sizeof(Ctl)));
    CK(cudaStreamCreateWithFlags(&c.op_stream, cudaStreamNonBlocking));
    set_gemv_attrs<EPI_STORE, MODE_PLAIN>();
    set_gemv_attrs<EPI_STORE, MODE_NORM>();
    CK(cudaFuncSetAttribute(limb_gemm_kernel<TG_BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            TgShape<TG_BN>::SMEM));
    CK(cudaFuncSetAttribute(limb_gemm_kernel<TG_BN_SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            TgShape<TG_BN_SMALL>::SMEM));
    {
        auto set = [&](auto kern) {
            cudaFuncAttributes fa;
            CK(cudaFuncGetAttributes(&fa, kern));
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(prop.sharedMemPerBlockOptin - fa.sharedSizeBytes)));
        };
        set(pf_attn_kernel<1, false>);
        set(pf_attn_kernel<2, false>);
        set(pf_attn_kernel<4, false>);
        set(pf_attn_kernel<8, false>);
        set(pf_attn_kernel<4, true>);
        CK(cudaFuncSetAttribute(pf_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pf_scores_smem())));
        CK(cudaFuncSetAttribute(pf_pv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pf_pv_smem())));
        set(bd_attn_kernel<false>);
        set(bd_attn_kernel<true>);
    }
    set_gemv_attrs<EPI_STORE, MODE_EMBED>();
    set_gemv_attrs<EPI_RESID, MODE_PLAIN>();
    set_gemv_attrs<EPI_SILU, MODE_NORM>();
    set_gemv_attrs<EPI_SILU, MODE_PLAIN>();
    set_gemv_attrs<EPI_ARGMAX, MODE_NORM>();
    set_gemv_attrs<EPI_RAW, MODE_PLAIN>();
    CK(cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(attn_op_scratch_bytes(8192))));
    // dynamic shared memory of the persistent kernels: what the larger
    // static footprint of the two leaves (the tensor-parallel group kernel
    // also holds its rank's arguments)
    cudaFuncAttributes fa, fg;
    CK(cudaFuncGetAttributes(&fa, decode_persistent_kernel));
    CK(cudaFuncGetAttributes(&fg, decode_persistent_group_kernel));
    c.smem_optin = int(prop.sharedMemPerBlockOptin) - int(std::max(fa.sharedSizeBytes, fg.sharedSizeBytes));
    CK(cudaFuncSetAttribute(decode_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            c.smem_optin));
    CK(cudaFuncSetAttribute(decode_persistent_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            c.smem_optin));
    CK(cudaDeviceSynchronize());  // the tables above landed before any non-blocking stream reads them
    c.device = device;
    return c;
}

struct DevBuf {
    std::vector<void*> ptrs;
    uint64_t bytes = 0;
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        size_t b = std::max<size_t>(n * sizeof(T), 16);
        CK(cudaMalloc(&p, b));
        ptrs.push_back(p);
        bytes += b;
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
};

// ---- tensor-core GEMM plumbing ------------------------------------------------

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) fail(DIMG_ECUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// 2-D byte matrix [outer][inner] with row stride `stride` bytes, read in
// 128-byte x box_rows boxes with the 128-byte swizzle the UMMA descriptors expect;
// out-of-range elements read as zero.
CUtensorMap tmap_bytes(const void* base, uint64_t inner, uint64_t outer, uint64_t stride, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {stride};
    const cuuint32_t box[2] = {TG_BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = tmap_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(DIMG_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

// Three signed byte digits of int64 rows x[t][0..K) into planes
// [3][rows_pad][ldp] (put_sdigits: exact for -0x808080 <= x <= 0x7F7F7F);
// *wide = 1 if some element is outside that range.
__global__ void limbs_kernel(const int64_t* __restrict__ x, uint32_t T, uint32_t K, uint32_t ldx,
                             uint8_t* __restrict__ planes, uint32_t rows_pad, uint32_t ldp, uint32_t* wide) {
    const size_t plane = size_t(rows_pad) * ldp;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < size_t(T) * K;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(i / K), j = uint32_t(i % K);
        const int64_t v = x[size_t(t) * ldx + j];
        if (!put_sdigits(planes + size_t(t) * ldp + j, plane, v)) *wide = 1;
    }
}

uint32_t gemm_tiles(const TgArgs& a, uint32_t bn) {
    return ((a.n_out + TG_BM - 1) / TG_BM) * ((a.n_tok + bn - 1) / bn);
}

// Split-K factor for a GEMM with few output tiles (decode batches).
uint32_t pick_ksplit(uint32_t tiles, uint32_t n_kblk, uint32_t slots) {
    // the largest k with every split owning its own CTA slot (one item per
    // CTA: the split epilogue's fence/atomic latency is paid once), >= 4 K
    // blocks per split
    uint32_t best = 1;
    for (uint32_t k = 2; k <= 8 && n_kblk / k >= 4 && tiles * k <= slots; ++k) best = k;
    return best;
}

// Programmatic dependent launch for the batch step's kernel chain (see
// pdl_wait in q16.cuh): each kernel may start, and the GEMMs stream their
// first weight tiles, while the previous one drains. DIMG_PDL=0 turns it off.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DIMG_PDL");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

template <typename... P, typename... A>
void launch_k(bool pdl, void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...));
}

// bn = token tile (TG_BN or TG_BN_SMALL; tb must be built with that box).
void launch_limb_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const TgArgs& a, cudaStream_t st,
                      uint32_t bn = TG_BN, bool pdl = false) {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint32_t items = gemm_tiles(a, bn) * (a.streamk ? a.n_kblk : std::max(1u, a.ksplit));
    const uint32_t per_sm = bn == TG_BN_SMALL ? 2u : 1u;
    const uint32_t grid = std::min<uint32_t>(items, per_sm * uint32_t(sms));
    if (bn == TG_BN_SMALL)
        launch_k(pdl, limb_gemm_kernel<TG_BN_SMALL>, grid, TgShape<TG_BN_SMALL>::THREADS, TgShape<TG_BN_SMALL>::SMEM,
                 st, ta, tb, a);
    else launch_k(pdl, limb_gemm_kernel<TG_BN>, grid, TgShape<TG_BN>::THREADS, TgShape<TG_BN>::SMEM, st, ta, tb, a);
}

}  // namespace

// ---------------------------------------------------------------------------
// Model in HBM
// ---------------------------------------------------------------------------
// Every dense matrix is stored "row-group blocked" for the persistent
// kernel: rows padded to a multiple of 4, K padded to 16, then chunk
// (group g, K-segment s) = rows 4g..4g+3 x columns [PK_SEG s, PK_SEG s + w) laid
// out contiguously, so one cp.async.bulk moves one chunk. q/k/v are one
// matrix (3D rows); gate/up are interleaved (gate_i row 2i, up_i row 2i+1) so
// a row group holds whole (gate, up) pairs for the silu*up epilogue.
struct DevMat {
    int8_t* w = nullptr;       // blocked (decode kernel)
    int64_t* s = nullptr;      // scales [rows]
    uint32_t rows = 0, K = 0, Kp = 0, n_groups = 0, n_segs = 0;
    int8_t* plain = nullptr;   // K-block-major [kblk][rows128][128] (tensor-core A operand)
    int8_t* rm = nullptr;      // row-major [rows][Kp] (tensor-parallel shards' GEMVs)
    uint32_t kblk = 0, rows128 = 0;
    CUtensorMap tmap;          // its TMA map (128 x 128-byte boxes, 128B swizzle)
};

struct BatchCache;  // batched-generation buffers + captured step graph (see below)

struct dimg_model {
    std::shared_ptr<BatchCache> batch;  // declared first: released after the weights' users
    std::mutex batch_mu;                // one batched generation at a time uses `batch`
    int device;
    DevCtx* ctx;
    dimg_config cfg;
    uint32_t D, F, V, H, dh, L, Kd, Kf;
    int tp_rank, tp_size;
    bool rowmajor = false;  // weights in the row-major GEMV layout only (tensor-parallel groups)
    // this rank's shard: heads [h0, h0 + Hl) (q/k/v rows and wo
    // columns [h0 dh, (h0 + Hl) dh)), FFN rows/columns [f0, f0 + Fl), vocab
    // rows [v0, v0 + Vl); the whole model when tp_size == 1
    uint32_t Hl, Dl, Fl, Vl, h0, f0, v0;
    struct Layer {
        DevMat qkv, wo, gu, down;
        int64_t* attn_norm;
        int64_t* ffn_norm;
        bool attn_unit, ffn_unit;  // gains all == ONE (mul16(v, ONE) == v: skipped)
    };
    std::vector<Layer> layers;
    DevMat head;
    bool final_unit;
    int8_t* embd;      // [V][D] row-major (one row gathered per token)
    int64_t* embd_s;
    int64_t* final_norm;
    int64_t* rope_cos;
    int64_t* rope_sin;
    int64_t inv_scale;
    DevBuf mem;
};

namespace {

// Copies rows x cols int8 (row-major, pitch cols) into a device buffer with
// row pitch dpitch, starting at row offset `row0` with row stride `rstride`.
// The copy is ordered on `st` (the stream whose kernels read dst): a plain
// cudaMemcpy2D from pageable memory may return before its DMA lands and is not
// ordered against a non-blocking stream. src_pitch = row stride of the source
// (cols for a whole matrix; the full width for a column slice).
void put_rows(int8_t* dst, size_t dpitch, size_t row0, size_t rstride, const int8_t* src,
              uint32_t rows, uint32_t cols, cudaStream_t st, size_t src_pitch = 0) {
    if (rows == 0) return;
    CK(cudaMemcpy2DAsync(dst + row0 * dpitch, dpitch * rstride, src, src_pitch ? src_pitch : cols, cols, rows,
                         cudaMemcpyHostToDevice, st));
}

template <class T>
T* upload(DevBuf& mem, const T* src, size_t n) {
    T* d = mem.alloc<T>(n);
    CK(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

bool all_one(const int64_t* g, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (g[i] != kOne) return false;
    return true;
}

// row-major [rows4][Kp] -> blocked [groups]{[segs][4][seg], 4 int64 scales}
// (16-byte units; persistent.cuh pk_group_bytes)
__global__ void blockify_kernel(const int4* __restrict__ src, const int64_t* __restrict__ scales,
                                uint32_t rows, int4* __restrict__ dst, uint32_t Kp, uint32_t n_groups,
                                uint32_t n_segs) {
    const size_t gbytes = pk_group_bytes(Kp);
    const size_t total = size_t(n_groups) * gbytes / 16;
    const uint32_t last = Kp - (n_segs - 1) * PK_SEG;
    for (size_t o = blockIdx.x * size_t(blockDim.x) + threadIdx.x; o < total;
         o += size_t(gridDim.x) * blockDim.x) {
        const size_t byte = o * 16;
        const size_t g = byte / gbytes;
        const size_t in_g = byte % gbytes;
        if (in_g >= size_t(PK_ROWS) * Kp) {  // the group's scales
            const uint32_t r = uint32_t((in_g - size_t(PK_ROWS) * Kp) / 8);
            const uint32_t row0 = uint32_t(g) * PK_ROWS + r;
            longlong2 v;
            v.x = row0 < rows ? scales[row0] : 0;
            v.y = row0 + 1 < rows ? scales[row0 + 1] : 0;
            reinterpret_cast<longlong2*>(dst)[o] = v;
            continue;
        }
        const uint32_t s = uint32_t(in_g / (PK_ROWS * PK_SEG));
        const uint32_t w = s + 1 < n_segs ? PK_SEG : last;
        const size_t in_s = in_g - size_t(s) * PK_ROWS * PK_SEG;
        const uint32_t r = uint32_t(in_s / w), c = uint32_t(in_s % w);
        const size_t sb = (g * PK_ROWS + r) * Kp + size_t(s) * PK_SEG + c;
        dst[o] = src[sb / 16];
    }
}

__global__ void kmajor_kernel(const int8_t* __restrict__ src, uint32_t Kp, uint32_t rows, uint32_t K,
                              int8_t* __restrict__ dst, uint32_t rows128, uint32_t kblk) {
    const size_t total = size_t(kblk) * rows128 * (TG_BK / 16);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t c16 = uint32_t(i % (TG_BK / 16));
        const size_t rb = i / (TG_BK / 16);
        const uint32_t r = uint32_t(rb % rows128), kb = uint32_t(rb / rows128);
        const uint32_t k = kb * TG_BK + c16 * 16;
        int4 v = make_int4(0, 0, 0, 0);
        if (r < rows && k < K) {
            v = *reinterpret_cast<const int4*>(src + size_t(r) * Kp + k);  // Kp % 16 == 0; bytes past K are zero
        }
        reinterpret_cast<int4*>(dst)[i] = v;
    }
}

// Uploads one dense matrix given as `parts` row blocks (each row-major,
// placed at row offset row0 with row stride rstride), then blockifies it.
struct RowPart {
    const int8_t* src;
    uint32_t rows, row0, rstride;
    size_t src_pitch = 0;  // source row stride (0: K, a whole matrix)
};

DevMat upload_mat(dimg_model& m, uint32_t rows, uint32_t K, const std::vector<RowPart>& parts,
                  const std::vector<int64_t>& scales, int8_t* staging) {
    DevMat d;
    d.rows = rows;
    d.K = K;
    d.Kp = pad16(K);
    d.n_groups = (rows + PK_ROWS - 1) / PK_ROWS;
    d.n_segs = (d.Kp + PK_SEG - 1) / PK_SEG;
    const size_t bytes = size_t(d.n_groups) * PK_ROWS * d.Kp;
    if (m.rowmajor) {
        // a tensor-parallel shard: the row-major [rows][Kp] layout the
        // per-stage GEMVs stream (no persistent-kernel or tensor-core copy)
        d.rm = m.mem.alloc<int8_t>(bytes);
        CK(cudaMemset(d.rm, 0, bytes));
        for (const auto& p : parts) put_rows(d.rm, d.Kp, p.row0, p.rstride, p.src, p.rows, K, nullptr, p.src_pitch);
        d.s = upload(m.mem, scales.data(), scales.size());
        CK(cudaDeviceSynchronize());
        return d;
    }
    CK(cudaMemset(staging, 0, bytes));
    for (const auto& p : parts) put_rows(staging, d.Kp, p.row0, p.rstride, p.src, p.rows, K, nullptr, p.src_pitch);
    d.s = upload(m.mem, scales.data(), scales.size());
    // tensor-core copy, K-block-major: [K/128][rows padded to 128][128 bytes],
    // so every 128-row x 128-byte TMA box is one contiguous 16 KB block
    d.kblk = (K + TG_BK - 1) / TG_BK;
    d.rows128 = (rows + TG_BM - 1) / TG_BM * TG_BM;
    d.plain = m.mem.alloc<int8_t>(size_t(d.kblk) * d.rows128 * TG_BK);
    kmajor_kernel<<<1024, 256>>>(staging, d.Kp, rows, K, d.plain, d.rows128, d.kblk);
    CK(cudaGetLastError());
    d.tmap = tmap_bytes(d.plain, TG_BK, size_t(d.kblk) * d.rows128, TG_BK, TG_BM);
    d.w = m.mem.alloc<int8_t>(size_t(d.n_groups) * pk_group_bytes(d.Kp));
    blockify_kernel<<<1024, 256>>>(reinterpret_cast<const int4*>(staging), d.s, rows,
                                   reinterpret_cast<int4*>(d.w), d.Kp, d.n_groups, d.n_segs);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return d;
}

}  // namespace

// ---------------------------------------------------------------------------
// Session: one sequence (KV cache, control block, token ring)
// ---------------------------------------------------------------------------
// Prefill workspace: all prompt tokens through a layer at once.
struct PrefillWs {
    uint32_t cap = 0, cap_pad = 0;   // tokens
    int32_t* x = nullptr;            // [cap][D] residual stream (int32: clamped to +-2^24)
    int64_t* qkv = nullptr;          // [cap][3D] projections (q rotated in place)
    uint8_t* pa = nullptr;           // [3][cap_pad][Kd] limb planes of D-wide inputs
    uint8_t* ph = nullptr;           // [3][cap_pad][Kf] limb planes of the FFN hidden vector
    uint32_t* wide = nullptr;        // some value needed the exact path
    int32_t* strips = nullptr;       // attention score / probability strips (pf_attn_strip_elems)
    CUtensorMap tm_pa, tm_ph;
    CUtensorMap tm_pa_s, tm_ph_s;    // box rows TG_BN_SMALL (prompts of <= 16 tokens)
    int32_t* partial = nullptr;      // split-K accumulators of the 16-token tiles (zero between launches)
    uint32_t* tile_cnt = nullptr;
    size_t partial_elems = 0;
    uint32_t tiles = 0;
    // set while a prefill is in flight: a call that fails part-way leaves the
    // split-K scratch possibly nonzero, so the next prefill re-zeroes it
    bool dirty = false;
    int8_t* kdig = nullptr;          // key digit planes [H][4][kdig_pad][128] (tensor-core scores, dh 128)
    int8_t* vh = nullptr;            // V >> 16 planes [H][128 dims][kdig_pad positions] (tensor-core PV)
    int32_t* fl = nullptr;           // sum_p floor(P vl / 2^16) [H][cap][128] (tensor-core PV)
    CUtensorMap tm_vh;
    uint32_t* kd4 = nullptr;         // [layers]: some key of the layer needs the 4th digit
    uint32_t kdig_pad = 0;
    CUtensorMap tm_kdig;
};

struct dimg_session {
    dimg_model* m;
    PrefillWs pf;
    uint64_t tc_prefills = 0, tc_fallbacks = 0;
    cudaStream_t stream = nullptr;
    DevBuf mem;
    int64_t *x, *qkv, *att, *h, *kc, *vc, *scores, *logits;
    int32_t* x32;  // [Kd] the residual stream as int32 (written by the residual epilogues)
    ArgPart* parts;
    uint32_t* tokens;  // [max_ctx + 1]
    Ctl* ctl;
    unsigned int* bar;
    unsigned long long* xg;  // [H][max_ctx][2] tagged score exchange words
    unsigned long long* qkv_x;  // [3D][2] tagged q/k/v words
    uint32_t* xwords;           // [2][Kd] tagged residual-stream words (after WO / after down)
    unsigned long long* parts_w;  // [2][grid][4] tagged lm_head partials
    uint32_t attn_tag = 0;   // attention stages tagged so far (xg tags)
    int32_t *kc32, *vc32;  // int32 mirror of the KV cache
    uint32_t* kvwide;      // [L][H] mirror unusable (sticky per sequence)
    uint32_t* words_att;   // [Kd] tagged limb words of the attention output
    uint32_t* words_h;     // [Kf] tagged limb words of the FFN hidden vector
    unsigned long long* ssq;  // [2L] sums of squares of x after wo / after down (per layer)
    PkStage* stages;   // [5L + 1] device
    std::vector<PkStage> host_stages;
    PkStage* probe_stages = nullptr;  // [L] scratch program for time_kernel
    uint32_t keep_cap = 0;
    uint32_t* draws = nullptr;        // generate_sampled: the steps' ChaCha20 draws
    uint32_t draws_cap = 0;
    int64_t* sample_scratch = nullptr;  // [vocab] scaled logits / probabilities
    uint32_t len = 0;  // host mirror of the cache length
    uint32_t n_prompt = 0, max_new = 0;
    uint32_t grid = 0, planes_bytes = 0, ring_depth = 2, wide_stride = 0;
    uint32_t* wide_planes = nullptr;
    size_t smem = 0;
    bool own_stream = true;  // false: a tensor-parallel group's shared stream
    ~dimg_session() {
        if (stream && own_stream) cudaStreamDestroy(stream);
    }
};

namespace {

uint32_t gemv_grid(const DevCtx& c, uint32_t rows, uint32_t unit) {
    uint32_t units = (rows + unit - 1) / unit;
    uint32_t g = uint32_t(c.sm_count) * 2;
    return std::max(1u, std::min(g, units));
}

template <int EPI, int MODE>
void launch_gemv(const GemvArgs& a, const DevCtx& c, cudaStream_t st, uint32_t grid = 0) {
    if (!grid) grid = gemv_grid(c, a.rows, EPI == EPI_SILU ? 2 : 1);
    size_t smem = size_t(8) * a.Kp;
    gemv_kernel<EPI, MODE, R_ROWS, U_3><<<grid, GEMV_THREADS, smem, st>>>(a);
}

PkStage gemv_stage(const DevMat& d, uint32_t mode, uint32_t epi, const int64_t* x, const int64_t* gamma,
                   int64_t* y, bool gamma_unit = false) {
    PkStage st{};
    st.kind = SK_GEMV;
    st.mode = mode;
    st.epi = epi;
    st.rows = d.rows; st.K = d.K; st.Kp = d.Kp; st.n_groups = d.n_groups; st.n_segs = d.n_segs;
    st.W = d.w; st.scales = d.s; st.x = x; st.gamma = gamma; st.y = y;
    st.gamma_unit = gamma_unit ? 1 : 0;
    return st;
}

// Which word hand-offs run without a grid barrier (1 qkv->attention,
// 2 attention->wo, 4 gate/up->down); DIMG_BARRIER_SKIP overrides for
// experiments. With the barrier kept, the consumer still polls the words.
uint32_t barrier_skip_mask() {
    const char* v = std::getenv("DIMG_BARRIER_SKIP");
    return v ? uint32_t(std::strtoul(v, nullptr, 0)) : 15u;
}

// The stage program of one forward step (proj/src/engine.cpp:85-101).
std::vector<PkStage> step_program(const dimg_session& s) {
    // Hand-offs between stages are tagged words, so a decode step has no grid
    // barrier at all: q/k/v -> attention, attention -> WO and gate/up -> down
    // as limb words; the residual stream after WO (buffer A) and after down
    // (buffer B) as x words that the next rmsnorm polls (it sums x^2 itself)
    // and the next residual reads; the lm_head partials as tagged entries.
    // DIMG_BARRIER_SKIP (bit 0 qkv, 1 attention, 2 gate/up, 3 residuals+head)
    // puts grid barriers back for experiments; the words are used either way.
    const dimg_model& m = *s.m;
    const uint32_t skip = barrier_skip_mask();
    std::vector<PkStage> p;
    uint32_t* xa = s.xwords;
    uint32_t* xb = s.xwords + m.Kd;
    for (uint32_t l = 0; l < m.L; ++l) {
        const auto& lw = m.layers[l];
        PkStage qkv = gemv_stage(lw.qkv, l == 0 ? MODE_EMBED : MODE_NORM, EPI_STORE, s.x, lw.attn_norm,
                                 s.qkv, lw.attn_unit);
        if (l > 0) qkv.xw_in = xb;  // down(l-1), same layer tag (attention has not advanced it yet)
        qkv.ytag = s.qkv_x;
        qkv.no_barrier = (skip & 1) ? 1 : 0;
        p.push_back(qkv);
        PkStage at{};
        at.kind = SK_ATTN;
        at.layer = l;
        at.out_words = s.words_att;
        at.no_barrier = (skip & 2) ? 1 : 0;
        p.push_back(at);
        PkStage wo = gemv_stage(lw.wo, MODE_PLAIN, EPI_RESID, s.att, nullptr, s.x);
        wo.in_words = s.words_att;
        wo.xw_out = xa;
        if (l > 0) {
            wo.xw_in = xb;  // residual input: down(l-1)'s words, one layer tag back
            wo.xw_lag = 1;
        } else {
            wo.resid_embed = 1;  // layer 0: the residual input is the token's embedding
        }
        wo.no_barrier = (skip & 8) ? 1 : 0;
        wo.tp_sum = 1;  // row-parallel under tensor parallelism: inbox buffer 0
        p.push_back(wo);
        PkStage gu = gemv_stage(lw.gu, MODE_NORM, EPI_SILU, s.x, lw.ffn_norm, s.h, lw.ffn_unit);
        gu.xw_in = xa;
        gu.out_words = s.words_h;
        gu.no_barrier = (skip & 4) ? 1 : 0;
        p.push_back(gu);
        PkStage dn = gemv_stage(lw.down, MODE_PLAIN, EPI_RESID, s.h, nullptr, s.x);
        dn.in_words = s.words_h;
        dn.xw_in = xa;
        dn.xw_out = xb;
        dn.no_barrier = (skip & 8) ? 1 : 0;
        dn.tp_sum = 2;  // inbox buffer 1
        p.push_back(dn);
    }
    PkStage head = gemv_stage(m.head, MODE_NORM, EPI_ARGMAX, s.x, m.final_norm, s.logits, m.final_unit);
    head.xw_in = xb;
    head.no_barrier = (skip & 8) ? 1 : 0;  // the partials go out as tagged words
    p.push_back(head);
    return p;
}

PkArgs pk_args(dimg_session& s, const PkStage* stages, uint32_t n_layer_stages, uint32_t n_steps,
               uint32_t n_prefill) {
    const dimg_model& m = *s.m;
    PkArgs a{};
    a.stages = stages;
    a.n_layer_stages = n_layer_stages;
    a.n_steps = n_steps;
    a.n_prefill = n_prefill;
    a.planes_bytes = s.planes_bytes;
    a.ring_depth = s.ring_depth;
    a.wide_planes = s.wide_planes;
    a.wide_stride = s.wide_stride;
    a.ctl = s.ctl;
    a.bar = s.bar;
    a.embd = m.embd;
    a.embd_scales = m.embd_s;
    a.d_model = m.D;
    a.vocab = m.V;
    a.tokens = s.tokens;
    a.logits = s.logits;
    a.parts = s.parts;
    a.x_resid = s.x;
    AttnArgs& t = a.attn;
    t.qkv = s.qkv;
    t.kc = s.kc;
    t.vc = s.vc;
    t.rope_cos = m.rope_cos;
    t.rope_sin = m.rope_sin;
    t.scores = s.scores;
    t.out = s.att;
    t.ctl = s.ctl;
    t.H = m.Hl;  // this rank's heads (all of them on one GPU)
    t.dh = m.dh;
    t.max_ctx = m.cfg.max_ctx;
    t.inv_scale = m.inv_scale;
    t.exp_lut = m.ctx->exp_lut;
    a.kv_layer_stride = size_t(m.Hl) * m.cfg.max_ctx * m.dh;
    // CTAs per head: split the head's dims over the SMs the heads leave idle,
    // at most 4 (measured best at 7B for the whole model and for its
    // tensor-parallel shards: 16 parts per head cost a TP-8 rank 911 vs 852
    // us/token, tools/tp_fused_probe.py --solo with DIMG_ATTN_PARTS)
    a.attn_parts = std::max(1u, std::min({s.grid / m.Hl, std::max(1u, m.dh / 8), 4u}));
    if (const char* e = std::getenv("DIMG_ATTN_PARTS"))  // experiments: CTAs per head
        a.attn_parts = std::max(1u, std::min(a.attn_parts, uint32_t(std::strtoul(e, nullptr, 0))));
    {
        auto log2_or = [](uint32_t x) { return x && !(x & (x - 1)) ? int32_t(__builtin_ctz(x)) : -1; };
        uint32_t dpp = (m.dh + a.attn_parts - 1) / a.attn_parts;
        dpp = (dpp + 3) & ~3u;  // whole 4-dim quads
        a.attn_dpp = dpp;
        a.attn_np_shift = log2_or(a.attn_parts);
        a.attn_nq_shift = log2_or(dpp / 4);
    }
    a.xg = s.xg;
    a.parts_w = s.parts_w;
    a.qkv_x = s.qkv_x;
    a.kc32 = s.kc32;
    a.vc32 = s.vc32;
    a.kvwide = s.kvwide;
    a.exp_lut = m.ctx->exp_lut;
    a.seeds = m.ctx->seeds;
    return a;
}

void launch_pk(dimg_session& s, const PkStage* stages, uint32_t n_layer_stages, uint32_t n_steps,
               uint32_t n_prefill, unsigned long long* trace = nullptr, uint32_t trace_cap = 0,
               unsigned long long* trace_all = nullptr) {
    if (n_steps == 0) return;
    PkArgs a = pk_args(s, stages, n_layer_stages, n_steps, n_prefill);
    a.trace = trace;
    a.trace_cap = trace_cap;
    a.trace_all = trace_all;

    // tags of the attention score exchange: unique per attention stage, never 0
    const uint64_t n_attn = uint64_t(n_steps) * s.m->L;
    if (uint64_t(s.attn_tag) + n_attn + 2 > 0xFFFFFFFFull) {
        CK(cudaMemsetAsync(s.xg, 0, size_t(s.m->Hl) * s.m->cfg.max_ctx * 16, s.stream));
        CK(cudaMemsetAsync(s.parts_w, 0, size_t(64) * s.grid, s.stream));
        s.attn_tag = 0;
    }
    a.tag_base = s.attn_tag;
    s.attn_tag += uint32_t(n_attn);
    CK(cudaMemsetAsync(s.bar, 0, 64 * sizeof(unsigned int), s.stream));
    CK(cudaMemsetAsync(s.ssq, 0, size_t(2) * s.m->L * sizeof(unsigned long long), s.stream));
    void* params[] = {&a};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(decode_persistent_kernel), dim3(s.grid),
                                   dim3(PK_THREADS), params, s.smem, s.stream));
}

// Writes the control header (pos, logit_base, keep_cap, argmax_count, err).
void write_ctl(dimg_session& s, uint32_t pos, uint32_t logit_base, uint32_t keep) {
    uint32_t hdr[5] = {pos, logit_base, keep, 0, 0};
    CK(cudaMemcpyAsync(s.ctl, hdr, sizeof hdr, cudaMemcpyHostToDevice, s.stream));
}

void check_ctl_err(dimg_session& s) {
    uint32_t err = 0;
    CK(cudaMemcpyAsync(&err, &s.ctl->err, 4, cudaMemcpyDeviceToHost, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    if (err & 4u) fail(DIMG_ECUDA, "persistent kernel: grid barrier timed out");
    if (err & 1u) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
}

// The sampler's sticky error word (write_ctl does not clear it).
void check_sample_err(dimg_session& s) {
    uint32_t err = 0;
    CK(cudaMemcpyAsync(&err, &s.ctl->serr, 4, cudaMemcpyDeviceToHost, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    if (err & 2u) fail(DIMG_EDOMAIN, "exp_neg_lut: argument outside [0, 8]");
}

void ensure_keep(dimg_session& s, uint32_t need) {
    if (need <= s.keep_cap) return;
    CK(cudaStreamSynchronize(s.stream));
    void* p = nullptr;
    CK(cudaMalloc(&p, size_t(need + 1) * s.m->Vl * sizeof(int64_t)));
    s.mem.ptrs.push_back(p);
    s.logits = static_cast<int64_t*>(p);
    s.keep_cap = need;
    // the head stage's output pointer lives in the stage table
    s.host_stages.back().y = s.logits;
    CK(cudaMemcpyAsync(s.stages + s.host_stages.size() - 1, &s.host_stages.back(), sizeof(PkStage),
                       cudaMemcpyHostToDevice, s.stream));
}

void check_prompt(const dimg_model& m, const uint32_t* prompt, uint32_t p, uint32_t n) {
    // check_generate_pre (proj/src/engine.cpp:21-29)
    if (p == 0) fail(DIMG_EINVAL, "generate: empty prompt");
    if (uint64_t(p) + n > m.cfg.max_ctx)
        fail(DIMG_ECTX, "generate: prompt plus continuation exceeds max_ctx");
    for (uint32_t i = 0; i < p; ++i)
        if (prompt[i] >= m.cfg.vocab) fail(DIMG_ERANGE, "generate: prompt token out of range");
}

void begin(dimg_session& s, const uint32_t* prompt, uint32_t p, uint32_t n, bool keep_logits) {
    check_prompt(*s.m, prompt, p, n);
    CK(cudaSetDevice(s.m->device));
    if (keep_logits) ensure_keep(s, n);
    CK(cudaMemcpyAsync(s.tokens, prompt, size_t(p) * 4, cudaMemcpyHostToDevice, s.stream));
    write_ctl(s, 0, p - 1, keep_logits ? n : 0);
    s.n_prompt = p;
    s.max_new = n;
    s.len = 0;
}

uint32_t n_layer_stages(const dimg_session& s) { return 5 * s.m->L; }

// Largest prompt the tensor-core prefill takes (its attention keeps every
// head's score strips in a global scratch of H * n^2 int32, 2 GB at 4096
// tokens and 32 heads); longer prompts and shapes it does not cover go
// through the decode kernel, one token per step.
constexpr uint32_t kTcPrefillMaxTokens = 4096;

uint32_t prefill_mode() {  // DIMG_PREFILL: 0 auto, 1 always tensor cores, 2 always decode steps
    const char* v = std::getenv("DIMG_PREFILL");
    return v ? uint32_t(std::strtoul(v, nullptr, 0)) : 0u;
}

bool tc_prefill_ok(const dimg_session& s, uint32_t n) {
    const dimg_model& m = *s.m;
    const uint32_t mode = prefill_mode();
    if (mode == 2 || n == 0) return false;
    if (m.dh % 4 || m.dh > 256 || n > kTcPrefillMaxTokens) return false;
    if (pf_attn_smem(m.dh) > size_t(m.ctx->smem_optin)) return false;
    return mode == 1 || n >= 3;  // tools/prefill_small.py: 3.3 ms flat vs 1.7 ms per decode step
}

void ensure_prefill_ws(dimg_session& s, uint32_t n) {
    PrefillWs& w = s.pf;
    if (w.cap >= n) return;
    const dimg_model& m = *s.m;
    w.cap = std::max(n, 128u);
    w.cap_pad = (w.cap + TG_BN - 1) / TG_BN * TG_BN;
    w.x = s.mem.alloc<int32_t>(size_t(w.cap) * m.D);
    w.qkv = s.mem.alloc<int64_t>(size_t(w.cap) * 3 * m.D);
    w.pa = s.mem.alloc<uint8_t>(size_t(3) * w.cap_pad * m.Kd);
    w.ph = s.mem.alloc<uint8_t>(size_t(3) * w.cap_pad * m.Kf);
    // zeroed on the session stream (a legacy-stream cudaMemset of device
    // memory is not ordered before the non-blocking session stream's kernels)
    CK(cudaMemsetAsync(w.pa, 0, size_t(3) * w.cap_pad * m.Kd, s.stream));
    CK(cudaMemsetAsync(w.ph, 0, size_t(3) * w.cap_pad * m.Kf, s.stream));
    if (!w.wide) w.wide = s.mem.alloc<uint32_t>(1);
    w.strips = s.mem.alloc<int32_t>(pf_attn_strip_elems(m.H, w.cap));
    w.tm_pa = tmap_bytes(w.pa, m.D, size_t(3) * w.cap_pad, m.Kd, TG_BN);
    w.tm_ph = tmap_bytes(w.ph, m.F, size_t(3) * w.cap_pad, m.Kf, TG_BN);
    w.tm_pa_s = tmap_bytes(w.pa, m.D, size_t(3) * w.cap_pad, m.Kd, TG_BN_SMALL);
    if (m.dh == PS_DH) {
        w.kdig_pad = (w.cap + PS_M - 1) / PS_M * PS_M;
        w.kdig = s.mem.alloc<int8_t>(size_t(m.H) * PS_KD * w.kdig_pad * PS_DH);
        w.tm_kdig = tmap_bytes(w.kdig, PS_DH, size_t(m.H) * PS_KD * w.kdig_pad, PS_DH, PS_M);
        w.vh = s.mem.alloc<int8_t>(size_t(m.H) * PV_M * w.kdig_pad);
        w.tm_vh = tmap_bytes(w.vh, w.kdig_pad, size_t(m.H) * PV_M, w.kdig_pad, PV_M);
        w.fl = s.mem.alloc<int32_t>(size_t(m.H) * w.cap * PV_M);
        if (!w.kd4) w.kd4 = s.mem.alloc<uint32_t>(m.L);
    }
    w.tm_ph_s = tmap_bytes(w.ph, m.F, size_t(3) * w.cap_pad, m.Kf, TG_BN_SMALL);
    if (!w.partial) {  // one 16-token tile column: the largest matrix's row tiles
        const uint32_t tiles = (std::max({3 * m.D, 2 * m.F, m.V}) + TG_BM - 1) / TG_BM;
        w.partial_elems = size_t(tiles) * TG_L * TG_BN_SMALL * TG_BM;
        w.partial = s.mem.alloc<int32_t>(w.partial_elems);
        w.tile_cnt = s.mem.alloc<uint32_t>(tiles);
        w.tiles = tiles;
        CK(cudaMemsetAsync(w.partial, 0, w.partial_elems * 4, s.stream));
        CK(cudaMemsetAsync(w.tile_cnt, 0, size_t(tiles) * 4, s.stream));
    }
}

template <class... A>
void launch_pf_attn(uint32_t dh, dim3 grid, size_t smem, cudaStream_t st, A... args) {
    const uint32_t dpl = (dh + 31) / 32;
    if (dpl <= 1) launch_k(true, pf_attn_kernel<1, false>, grid, PA_THREADS, smem, st, args..., (int32_t*)nullptr);
    else if (dpl <= 2) launch_k(true, pf_attn_kernel<2, false>, grid, PA_THREADS, smem, st, args..., (int32_t*)nullptr);
    else if (dpl <= 4) launch_k(true, pf_attn_kernel<4, false>, grid, PA_THREADS, smem, st, args..., (int32_t*)nullptr);
    else launch_k(true, pf_attn_kernel<8, false>, grid, PA_THREADS, smem, st, args..., (int32_t*)nullptr);  // dh <= 256
}

// Positions 0..n-1 of the prompt through every layer on the tensor cores;
// returns false (nothing usable written) if some value needed the exact path.
bool run_prefill_tc(dimg_session& s, uint32_t n) {
    const dimg_model& m = *s.m;
    ensure_prefill_ws(s, n);
    PrefillWs& w = s.pf;
    cudaStream_t st = s.stream;
    const uint32_t D = m.D, dh = m.dh, H = m.H;
    const size_t kv_layer = size_t(H) * m.cfg.max_ctx * dh;
    if (w.dirty) {  // the previous prefill failed part-way: its split-K scratch may be dirty
        CK(cudaMemsetAsync(w.partial, 0, w.partial_elems * 4, st));
        CK(cudaMemsetAsync(w.tile_cnt, 0, size_t(w.tiles) * 4, st));
    }
    w.dirty = true;
    CK(cudaMemsetAsync(w.wide, 0, 4, st));
    CK(cudaMemsetAsync(s.kvwide, 0, size_t(m.L) * H * 4, st));
    // every kernel of the chain by programmatic dependent launch (pdl_wait in each)
    launch_k(true, pf_embed_kernel, 1024, 256, 0, st, (const uint32_t*)s.tokens, n, (const int8_t*)m.embd,
             (const int64_t*)m.embd_s, D, w.x, w.wide);
    // short prompts: 16-token tiles split over K (one split per CTA slot), as the decode batches
    const bool small = n <= uint32_t(TG_BN_SMALL);
    const uint32_t bn = small ? TG_BN_SMALL : TG_BN;
    const uint32_t sms = uint32_t(m.ctx->sm_count);
    auto gemm = [&](const DevMat& W, const CUtensorMap& tb_big, uint32_t epi, void* y, uint32_t ldy) {
        const CUtensorMap& tb = !small ? tb_big : (&tb_big == &w.tm_ph ? w.tm_ph_s : w.tm_pa_s);
        TgArgs a{};
        a.n_out = W.rows;
        a.a_rows = W.rows128;
        a.n_tok = n;
        a.n_kblk = (W.K + TG_BK - 1) / TG_BK;
        a.limb_rows = w.cap_pad;
        a.epi = epi;
        a.scales = W.s;
        if (epi == TG_RESID) a.x32 = static_cast<int32_t*>(y);  // the int32 residual stream
        else a.y = static_cast<int64_t*>(y);
        a.ldy = ldy;
        a.planes = w.ph;
        a.limb_rows_out = w.cap_pad;
        a.ldp = m.Kf;
        a.lut = m.ctx->exp_lut;
        a.wide = w.wide;
        if (small) {
            a.ksplit = pick_ksplit(gemm_tiles(a, bn), a.n_kblk, 2 * sms);
            a.partial = w.partial;
            a.tile_cnt = w.tile_cnt;
        }
        // token tiles fastest when the activation planes stay L2-resident
        // (K = d_model: 25 MB at 2048 tokens); w_down's 68 MB do not
        a.token_fast = size_t(3) * n * W.K <= (size_t(32) << 20) ? 1 : 0;
        launch_limb_gemm(W.tmap, tb, a, st, bn, true);
    };
    const size_t asmem = pf_attn_smem(dh);
    // attention scores on the tensor cores when dh = 128 (pf_scores.cuh);
    // DIMG_PF_SCORES=0 keeps them on the CUDA cores
    const char* ps_env = std::getenv("DIMG_PF_SCORES");
    const bool tc_scores = w.kdig && (!ps_env || std::atoi(ps_env) != 0);
    // DIMG_PF_KD4=1 forces the 4th key digit plane (tests of that path)
    const char* kd4_env = std::getenv("DIMG_PF_KD4");
    if (tc_scores) CK(cudaMemsetAsync(w.kd4, kd4_env && std::atoi(kd4_env) ? 1 : 0, size_t(m.L) * 4, st));
    // PV's linear half on the tensor cores when dh = 128 (pf_pv.cuh);
    // DIMG_PF_PV=0 keeps all of PV on the CUDA cores
    const char* pv_env = std::getenv("DIMG_PF_PV");
    const bool tc_pv = w.vh && dh == PV_M && (!pv_env || std::atoi(pv_env) != 0);
    for (uint32_t l = 0; l < m.L; ++l) {
        const auto& lw = m.layers[l];
        launch_k(true, pf_norm_limbs_kernel, n, 256, 0, st, (const int32_t*)w.x, D, (const int64_t*)lw.attn_norm,
                 int(lw.attn_unit), (const int64_t*)m.ctx->seeds, w.pa, w.cap_pad, m.Kd, w.wide);
        gemm(lw.qkv, w.tm_pa, TG_STORE, w.qkv, 3 * D);
        const bool last = l + 1 == m.L;  // the last layer's output feeds only the lm_head
        launch_k(true, pf_rope_kv_kernel, dim3(n, H), dh / 2, 0, st, w.qkv, D, dh, (const int64_t*)m.rope_cos,
                 (const int64_t*)m.rope_sin, s.kc + l * kv_layer, s.vc + l * kv_layer, s.kc32 + l * kv_layer,
                 s.vc32 + l * kv_layer, size_t(m.cfg.max_ctx) * dh, w.wide, tc_scores && !last ? w.kdig : nullptr,
                 w.kdig_pad, tc_scores ? w.kd4 + l : (uint32_t*)nullptr);
        if (last) break;
        if (tc_scores)
            launch_k(true, pf_scores_kernel, dim3(H, (n + PS_Q - 1) / PS_Q), PS_THREADS, pf_scores_smem(), st,
                     w.tm_kdig, (const int64_t*)w.qkv, n, w.kdig_pad, D, m.inv_scale, w.strips, w.wide,
                     (const uint32_t*)(w.kd4 + l));
        if (tc_pv) {
            // PV's linear half on the tensor cores (pf_pv.cuh): vh planes, then
            // softmax + the per-product half, then the MMAs + output planes
            launch_k(true, pf_vh_kernel, dim3(H, (n + PV_KB - 1) / PV_KB), 256, 0, st,
                     (const int32_t*)(s.vc32 + l * kv_layer), size_t(m.cfg.max_ctx) * dh, n, w.kdig_pad, w.vh, w.wide);
            launch_k(true, pf_attn_kernel<4, true>, dim3(H, (n + PA_Q - 1) / PA_Q), PA_THREADS, asmem, st,
                     (const int64_t*)w.qkv, n, D, dh, (const int32_t*)(s.kc32 + l * kv_layer),
                     (const int32_t*)(s.vc32 + l * kv_layer), size_t(m.cfg.max_ctx) * dh, m.inv_scale,
                     (const int64_t*)m.ctx->exp_lut, w.strips, w.pa, w.cap_pad, m.Kd, w.wide, tc_scores, w.fl);
            launch_k(true, pf_pv_kernel, dim3(H, (n + PV_Q - 1) / PV_Q), PV_THREADS, pf_pv_smem(), st, w.tm_vh,
                     (const int32_t*)w.strips, (const int32_t*)w.fl, (const int32_t*)(s.vc32 + l * kv_layer),
                     size_t(m.cfg.max_ctx) * dh, n, w.pa, w.cap_pad, m.Kd, w.wide);
        } else {
            launch_pf_attn(dh, dim3(H, (n + PA_Q - 1) / PA_Q), asmem, st, (const int64_t*)w.qkv, n, D, dh,
                           (const int32_t*)(s.kc32 + l * kv_layer), (const int32_t*)(s.vc32 + l * kv_layer),
                           size_t(m.cfg.max_ctx) * dh, m.inv_scale, (const int64_t*)m.ctx->exp_lut, w.strips, w.pa,
                           w.cap_pad, m.Kd, w.wide, tc_scores);
        }
        gemm(lw.wo, w.tm_pa, TG_RESID, w.x, D);
        launch_k(true, pf_norm_limbs_kernel, n, 256, 0, st, (const int32_t*)w.x, D, (const int64_t*)lw.ffn_norm,
                 int(lw.ffn_unit), (const int64_t*)m.ctx->seeds, w.pa, w.cap_pad, m.Kd, w.wide);
        gemm(lw.gu, w.tm_pa, TG_SILU, nullptr, 0);
        gemm(lw.down, w.tm_ph, TG_RESID, w.x, D);
    }
    CK(cudaGetLastError());
    uint32_t wide = 0;
    CK(cudaMemcpyAsync(&wide, w.wide, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    w.dirty = false;  // every split-K launch completed: the scratch is zero again
    return wide == 0;
}

// The prompt's first n_prompt - 1 positions on the tensor cores when the
// shapes allow; true if done (cache length and the kernel's position set).
bool try_prefill_tc(dimg_session& s) {
    const uint32_t n = s.n_prompt - 1;
    if (!tc_prefill_ok(s, n)) return false;
    if (!run_prefill_tc(s, n)) {
        ++s.tc_fallbacks;
        return false;
    }
    ++s.tc_prefills;
    CK(cudaMemcpyAsync(&s.ctl->pos, &n, 4, cudaMemcpyHostToDevice, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    s.len = n;
    return true;
}

void run_prefill(dimg_session& s) {
    if (try_prefill_tc(s)) return;
    uint32_t n = s.n_prompt - 1;
    launch_pk(s, s.stages, n_layer_stages(s), n, n);
    s.len = n;
}

void run_decode(dimg_session& s, uint32_t steps) {
    launch_pk(s, s.stages, n_layer_stages(s), steps, 0);
    s.len += steps;
}

}  // namespace

// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// Batched generation (C5): independent sequences stepped together
// ---------------------------------------------------------------------------
namespace {

struct BatchRun {
    dimg_model* m;
    cudaStream_t st = nullptr;
    DevBuf mem;
    uint32_t B = 0, ctx = 0, nmax = 0, nmax_pad = 0, max_new = 0;
    uint32_t *tok = nullptr, *seq = nullptr, *pos = nullptr, *out = nullptr, *step = nullptr, *wide = nullptr;
    int32_t* x = nullptr;  // residual stream, int32 (clamped to +-2^24)
    int64_t *qkv = nullptr, *logits = nullptr;
    uint8_t *pa = nullptr, *ph = nullptr;
    int32_t *K32 = nullptr, *V32 = nullptr;
    size_t seq_stride = 0, layer_stride = 0;
    CUtensorMap tm_pa, tm_ph;           // box rows TG_BN (prompt phase)
    CUtensorMap tm_pa_s, tm_ph_s;       // box rows TG_BN_SMALL (decode steps of <= 16 sequences)
    int32_t* partial = nullptr;         // split-K partials
    uint32_t* tile_cnt = nullptr;
    size_t partial_elems = 0;
    uint32_t tiles_max = 0;
    bool dirty = false;  // a batch call failed part-way: re-zero the split-K scratch first
    ~BatchRun() {
        if (st) cudaStreamDestroy(st);
    }
};

bool batch_shape_ok(const dimg_model& m) { return m.dh % 4 == 0 && m.dh / 2 <= 1024; }

}  // namespace

struct BatchCache {
    BatchRun r;                    // buffers for up to r.B sequences (capacity)
    cudaGraphExec_t ge = nullptr;  // the captured decode step of ge_B sequences (r's buffers)
    uint32_t ge_B = 0;
    ~BatchCache() {
        if (ge) cudaGraphExecDestroy(ge);
    }
};

namespace {

void batch_alloc(BatchRun& r, dimg_model* m, uint32_t B, uint32_t ctx, uint32_t nmax, uint32_t max_new) {
    r.m = m;
    r.B = B;
    r.ctx = ctx;
    r.nmax = nmax;
    r.nmax_pad = (nmax + TG_BN - 1) / TG_BN * TG_BN;
    r.max_new = max_new;
    CK(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
    r.tok = r.mem.alloc<uint32_t>(nmax);
    r.seq = r.mem.alloc<uint32_t>(nmax);
    r.pos = r.mem.alloc<uint32_t>(nmax);
    r.out = r.mem.alloc<uint32_t>(size_t(B) * std::max(1u, max_new));
    r.step = r.mem.alloc<uint32_t>(1);
    r.wide = r.mem.alloc<uint32_t>(1);
    r.x = r.mem.alloc<int32_t>(size_t(nmax) * m->D);
    r.qkv = r.mem.alloc<int64_t>(size_t(nmax) * 3 * m->D);
    r.logits = r.mem.alloc<int64_t>(size_t(B) * m->V);
    r.pa = r.mem.alloc<uint8_t>(size_t(3) * r.nmax_pad * m->Kd);
    r.ph = r.mem.alloc<uint8_t>(size_t(3) * r.nmax_pad * m->Kf);
    CK(cudaMemsetAsync(r.pa, 0, size_t(3) * r.nmax_pad * m->Kd, r.st));
    CK(cudaMemsetAsync(r.ph, 0, size_t(3) * r.nmax_pad * m->Kf, r.st));
    r.layer_stride = size_t(m->H) * ctx * m->dh;
    r.seq_stride = r.layer_stride * m->L;
    r.K32 = r.mem.alloc<int32_t>(r.seq_stride * B);
    r.V32 = r.mem.alloc<int32_t>(r.seq_stride * B);
    CK(cudaMemsetAsync(r.step, 0, 4, r.st));
    CK(cudaMemsetAsync(r.wide, 0, 4, r.st));
    r.tm_pa = tmap_bytes(r.pa, m->D, size_t(3) * r.nmax_pad, m->Kd, TG_BN);
    r.tm_ph = tmap_bytes(r.ph, m->F, size_t(3) * r.nmax_pad, m->Kf, TG_BN);
    r.tm_pa_s = tmap_bytes(r.pa, m->D, size_t(3) * r.nmax_pad, m->Kd, TG_BN_SMALL);
    r.tm_ph_s = tmap_bytes(r.ph, m->F, size_t(3) * r.nmax_pad, m->Kf, TG_BN_SMALL);
    // split-K scratch for the decode steps: tiles x k x 3 limbs x BN x 128 int32
    const uint32_t bn = B <= TG_BN_SMALL ? TG_BN_SMALL : TG_BN;
    const uint32_t tok_tiles = (B + bn - 1) / bn;
    const uint32_t rows[5] = {3 * m->D, m->D, 2 * m->F, m->D, m->V};
    for (uint32_t rw : rows) {
        const uint32_t tiles = (rw + TG_BM - 1) / TG_BM * tok_tiles;
        r.tiles_max = std::max(r.tiles_max, tiles);
        r.partial_elems = std::max(r.partial_elems, size_t(tiles) * TG_L * bn * TG_BM);
    }
    r.partial = r.mem.alloc<int32_t>(r.partial_elems);
    CK(cudaMemsetAsync(r.partial, 0, r.partial_elems * 4, r.st));
    r.tile_cnt = r.mem.alloc<uint32_t>(r.tiles_max);
    CK(cudaMemsetAsync(r.tile_cnt, 0, size_t(r.tiles_max) * 4, r.st));
}

// One forward pass of n tokens (each its own sequence/position); with
// logits: the lm_head, greedy selection and the token/position feedback.
void batch_step(BatchRun& r, uint32_t n, bool logits) {
    const dimg_model& m = *r.m;
    cudaStream_t st = r.st;
    const uint32_t D = m.D, dh = m.dh, H = m.H;
    const BatchTok bt{r.tok, r.seq, r.pos};
    launch_k(true, bd_embed_kernel, 1024, 256, 0, st, bt, n, (const int8_t*)m.embd, (const int64_t*)m.embd_s, D, r.x,
             r.wide);
    const bool small = n <= uint32_t(TG_BN_SMALL);
    const uint32_t bn = small ? TG_BN_SMALL : TG_BN;
    // split-K (DIMG_SPLITK=0 turns it off): 16-token tiles split whenever the
    // tiles leave CTA slots free (two CTAs per SM); 64-token tiles only for
    // long K (w_down), where the saved K blocks outweigh the accumulation
    // traffic (tools/gemm_bench.cu: 30 -> 22 us at 64 tokens)
    const char* sk = std::getenv("DIMG_SPLITK");
    const bool split_k = sk ? std::atoi(sk) != 0 : true;
    const char* skv = std::getenv("DIMG_STREAMK");
    const bool streamk = skv ? std::atoi(skv) != 0 : false;
    int sms = m.ctx->sm_count;
    // DIMG_BD_SKIP (timing experiments only; results are wrong): bit 0 skips
    // the norms, 1 RoPE/KV, 2 attention -- what each launch chain costs
    static const uint32_t skip = [] {
        const char* e = std::getenv("DIMG_BD_SKIP");
        return e ? uint32_t(std::strtoul(e, nullptr, 0)) : 0u;
    }();
    auto gemm = [&](const DevMat& W, const CUtensorMap& tb_big, uint32_t epi, void* y, uint32_t ldy) {
        const bool in_h = &tb_big == &r.tm_ph;
        const CUtensorMap& tb = small ? (in_h ? r.tm_ph_s : r.tm_pa_s) : tb_big;
        TgArgs a{};
        a.n_out = W.rows;
        a.a_rows = W.rows128;
        a.n_tok = n;
        a.n_kblk = (W.K + TG_BK - 1) / TG_BK;
        a.limb_rows = r.nmax_pad;
        a.epi = epi;
        a.scales = W.s;
        if (epi == TG_RESID) a.x32 = static_cast<int32_t*>(y);  // the int32 residual stream
        else a.y = static_cast<int64_t*>(y);
        a.ldy = ldy;
        a.planes = r.ph;
        a.limb_rows_out = r.nmax_pad;
        a.ldp = m.Kf;
        a.lut = m.ctx->exp_lut;
        a.wide = r.wide;
        a.ksplit = !split_k ? 1
                   : small  ? pick_ksplit(gemm_tiles(a, bn), a.n_kblk, 2 * uint32_t(sms))
                   : a.n_kblk >= 64 ? std::min(4u, pick_ksplit(gemm_tiles(a, bn), a.n_kblk, uint32_t(sms)))
                                    : 1;
        if (size_t(gemm_tiles(a, bn)) * TG_L * bn * TG_BM > r.partial_elems) a.ksplit = 1;
        // DIMG_STREAMK=1 (experiment, off): stream-K for the decode steps --
        // every CTA the same number of weight K blocks (gate/up's 172 tiles
        // on 296 CTA slots), but nearly every tile then goes through the
        // red.add partial sums: C5 B=8 0.381 s vs 0.334 s, B=64 equal
        a.streamk = small && streamk && split_k &&
                    size_t(gemm_tiles(a, bn)) * TG_L * bn * TG_BM <= r.partial_elems ? 1u : 0u;
        a.partial = r.partial;
        a.tile_cnt = r.tile_cnt;
        launch_limb_gemm(W.tmap, tb, a, st, bn, true);
    };
    auto norm_ = [&](const int64_t* g, int unit) {  // decode steps: one 1024-thread CTA per token
        if (n <= 64u)
            launch_k(true, bd_norm1k_kernel, n, 1024, 0, st, (const int32_t*)r.x, D, g, unit,
                     (const int64_t*)m.ctx->seeds, r.pa, r.nmax_pad, m.Kd, r.wide);
        else
            launch_k(true, pf_norm_limbs_kernel, n, 256, 0, st, (const int32_t*)r.x, D, g, unit,
                     (const int64_t*)m.ctx->seeds, r.pa, r.nmax_pad, m.Kd, r.wide);
    };
    const size_t asmem = bd_attn_smem(dh, r.ctx) + 8;
    auto norm = [&](const int64_t* g, int unit) {
        if (!(skip & 1)) norm_(g, unit);
    };
    for (uint32_t l = 0; l < m.L; ++l) {
        const auto& lw = m.layers[l];
        norm(lw.attn_norm, lw.attn_unit);
        gemm(lw.qkv, r.tm_pa, TG_STORE, r.qkv, 3 * D);
        // decode steps: RoPE + the KV append run inside the attention kernel
        if (!(skip & 2) && !logits) launch_k(true, bd_rope_kv_kernel, dim3(n, H), dh / 2, 0, st, r.qkv, bt, D, dh, (const int64_t*)m.rope_cos,
                 (const int64_t*)m.rope_sin, r.K32 + l * r.layer_stride, r.V32 + l * r.layer_stride, r.seq_stride,
                 r.ctx, r.wide);
        if (l + 1 == m.L && !logits) break;  // prompt positions only feed the KV caches
        if (!(skip & 4)) launch_k(true, small ? bd_attn_kernel<true> : bd_attn_kernel<false>, dim3(H, n), BD_THREADS, asmem, st, (const int64_t*)r.qkv, bt, D, dh,
                 r.K32 + l * r.layer_stride, r.V32 + l * r.layer_stride, r.seq_stride, r.ctx, m.inv_scale,
                 (const int64_t*)m.ctx->exp_lut, r.pa, r.nmax_pad, m.Kd, r.wide,
                 logits ? (const int64_t*)m.rope_cos : nullptr, logits ? (const int64_t*)m.rope_sin : nullptr);
        gemm(lw.wo, r.tm_pa, TG_RESID, r.x, D);
        norm(lw.ffn_norm, lw.ffn_unit);
        gemm(lw.gu, r.tm_pa, TG_SILU, nullptr, 0);
        gemm(lw.down, r.tm_ph, TG_RESID, r.x, D);
    }
    if (logits) {
        norm(m.final_norm, m.final_unit);
        gemm(m.head, r.tm_pa, TG_STORE, r.logits, m.V);
        launch_k(true, bd_argmax_kernel, n, 1024, 0, st, (const int64_t*)r.logits, m.V, r.tok, r.pos,
                 (const uint32_t*)r.seq, r.out, r.max_new, r.step);
        launch_k(true, bd_step_kernel, 1, 1, 0, st, r.step);
    }
    CK(cudaGetLastError());
}

// The batch path: true if every sequence's tokens were produced exactly.
bool generate_batch_tc(dimg_model* m, uint32_t B, const std::vector<std::vector<uint32_t>>& prompts,
                       uint32_t max_new, uint32_t* tokens_out) {
    uint32_t ctx = 0, n_prompt_pos = 0;
    for (const auto& p : prompts) {
        ctx = std::max<uint32_t>(ctx, uint32_t(p.size()) + max_new);
        n_prompt_pos += uint32_t(p.size()) - 1;
    }
    if (bd_attn_smem(m->dh, ctx) + 8 > size_t(m->ctx->smem_optin)) return false;
    // buffers (and the captured step graph) are kept on the model and reused
    // while the batch fits them
    const uint32_t nmax = std::max(n_prompt_pos, B);
    if (!m->batch || m->batch->r.B < B || m->batch->r.ctx < ctx || m->batch->r.nmax < nmax ||
        m->batch->r.max_new < std::max(1u, max_new)) {
        m->batch.reset();
        auto c = std::make_shared<BatchCache>();
        batch_alloc(c->r, m, B, std::max(ctx, 64u), nmax, std::max(max_new, 128u));
        m->batch = c;
    }
    BatchCache& c = *m->batch;
    BatchRun& r = c.r;
    if (r.dirty) {
        CK(cudaMemsetAsync(r.partial, 0, r.partial_elems * 4, r.st));
        CK(cudaMemsetAsync(r.tile_cnt, 0, size_t(r.tiles_max) * 4, r.st));
    }
    r.dirty = true;
    CK(cudaMemsetAsync(r.step, 0, 4, r.st));
    CK(cudaMemsetAsync(r.wide, 0, 4, r.st));
    // prompt phase: all positions but each prompt's last, one forward pass
    if (n_prompt_pos) {
        std::vector<uint32_t> tok, seq, pos;
        for (uint32_t b = 0; b < B; ++b)
            for (uint32_t i = 0; i + 1 < prompts[b].size(); ++i) {
                tok.push_back(prompts[b][i]);
                seq.push_back(b);
                pos.push_back(i);
            }
        CK(cudaMemcpyAsync(r.tok, tok.data(), tok.size() * 4, cudaMemcpyHostToDevice, r.st));
        CK(cudaMemcpyAsync(r.seq, seq.data(), seq.size() * 4, cudaMemcpyHostToDevice, r.st));
        CK(cudaMemcpyAsync(r.pos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, r.st));
        batch_step(r, n_prompt_pos, false);
    }
    // decode: one token per sequence per step, the step captured once as a CUDA graph
    {
        std::vector<uint32_t> tok(B), seq(B), pos(B);
        for (uint32_t b = 0; b < B; ++b) {
            tok[b] = prompts[b].back();
            seq[b] = b;
            pos[b] = uint32_t(prompts[b].size()) - 1;
        }
        CK(cudaMemcpyAsync(r.tok, tok.data(), B * 4, cudaMemcpyHostToDevice, r.st));
        CK(cudaMemcpyAsync(r.seq, seq.data(), B * 4, cudaMemcpyHostToDevice, r.st));
        CK(cudaMemcpyAsync(r.pos, pos.data(), B * 4, cudaMemcpyHostToDevice, r.st));
        CK(cudaStreamSynchronize(r.st));
    }
    if (max_new > 0) {
        if (c.ge && c.ge_B != B) {
            CK(cudaGraphExecDestroy(c.ge));
            c.ge = nullptr;
        }
        if (!c.ge) {
            cudaGraph_t g = nullptr;
            CK(cudaStreamBeginCapture(r.st, cudaStreamCaptureModeThreadLocal));
            batch_step(r, B, true);
            CK(cudaStreamEndCapture(r.st, &g));
            CK(cudaGraphInstantiate(&c.ge, g, 0));
            cudaGraphDestroy(g);
            c.ge_B = B;
        }
        for (uint32_t s = 0; s < max_new; ++s) CK(cudaGraphLaunch(c.ge, r.st));
    }
    uint32_t wide = 0;
    CK(cudaMemcpyAsync(&wide, r.wide, 4, cudaMemcpyDeviceToHost, r.st));
    if (max_new > 0)
        CK(cudaMemcpy2DAsync(tokens_out, size_t(max_new) * 4, r.out, size_t(r.max_new) * 4, size_t(max_new) * 4, B,
                             cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    r.dirty = false;
    return wide == 0;
}

}  // namespace

namespace dimg::chacha {

// The toy-model weight stream on the GPU (kernels/chacha.cuh), copied into
// the host spans in order: the same bytes as weight_stream.
void gpu_weight_stream(int device, uint64_t seed, const Span* spans, size_t n_spans) {
    uint64_t n = 0;
    for (size_t i = 0; i < n_spans; ++i) n += spans[i].len;
    if (n == 0) return;
    CK(cudaSetDevice(device));
    const Key hk = key_from_seed(seed);
    dev::CcKey key;
    for (int i = 0; i < 8; ++i) key.k[i] = hk[i];
    DevBuf mem;
    int8_t* out = mem.alloc<int8_t>(n);
    uint64_t* grand = mem.alloc<uint64_t>(1);
    // 64 bytes per block accept 63.75 on average: n / 63 blocks (+ slack)
    // almost always suffice; otherwise grow and count again
    for (uint64_t nb = n / 63 + 4096;; nb += nb / 16) {
        if (nb >= (uint64_t(1) << 32)) fail(DIMG_EINVAL, "gen_toy_model: weight stream exceeds the block counter");
        const uint64_t g = (nb + dev::CC_THREADS - 1) / dev::CC_THREADS;
        DevBuf scratch;
        uint8_t* cnt = scratch.alloc<uint8_t>(nb);
        uint64_t* tot = scratch.alloc<uint64_t>(g);
        dev::cc_count_kernel<<<uint32_t(g), dev::CC_THREADS>>>(key, nb, cnt, tot);
        dev::cc_scan_kernel<<<1, dev::CC_THREADS>>>(tot, g, grand);
        uint64_t have = 0;
        CK(cudaMemcpy(&have, grand, 8, cudaMemcpyDeviceToHost));
        if (have < n) continue;
        dev::cc_compact_kernel<<<uint32_t(g), dev::CC_THREADS>>>(key, nb, cnt, tot, n, out);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        break;
    }
    uint64_t o = 0;
    for (size_t i = 0; i < n_spans; ++i) {
        CK(cudaMemcpy(spans[i].dst, out + o, spans[i].len, cudaMemcpyDeviceToHost));
        o += spans[i].len;
    }
}

}  // namespace dimg::chacha

// generation_counter (proj/src/engine.cpp:165-168): one per run_generation
static std::atomic<uint64_t> g_generations{0};

extern "C" {

dimg_status dimg_device_count(int* n) { DIMG_API_GUARD(CK(cudaGetDeviceCount(n))) }

}  // extern "C"

namespace {
dimg_model* model_upload(int device, const dimg_model_desc* d, int tp_rank, int tp_size, bool rowmajor);
}

extern "C" dimg_status dimg_model_upload(int device, const dimg_model_desc* d, int tp_rank, int tp_size,
                              dimg_model** out) {
    DIMG_API_GUARD(*out = model_upload(device, d, tp_rank, tp_size, tp_size > 1))
}

namespace {
// rowmajor: the per-stage GEMV layout of tensor-parallel groups (dimg_tp),
// instead of the persistent kernel's and tensor cores' copies
dimg_model* model_upload(int device, const dimg_model_desc* d, int tp_rank, int tp_size, bool rowmajor) {
    {
        validate_config(d->cfg);
        if (pad16(d->cfg.d_model) > 8192)
            fail(DIMG_EINVAL, "model_upload: d_model above 8192");  // persistent.cuh MAXW
        if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
            fail(DIMG_EINVAL, "model_upload: bad tensor-parallel rank/size");
        if (d->cfg.n_heads % uint32_t(tp_size))
            fail(DIMG_EINVAL, "model_upload: n_heads must be a multiple of the tensor-parallel size");
        DevCtx& c = dev_ctx(device);
        CK(cudaSetDevice(device));
        auto m = std::make_unique<dimg_model>();
        m->device = device;
        m->ctx = &c;
        m->cfg = d->cfg;
        m->D = d->cfg.d_model; m->F = d->cfg.d_ffn; m->V = d->cfg.vocab; m->H = d->cfg.n_heads;
        m->dh = m->D / m->H; m->L = d->cfg.n_layers; m->Kd = pad16(m->D); m->Kf = pad16(m->F);
        m->tp_rank = tp_rank; m->tp_size = tp_size; m->rowmajor = rowmajor;
        const uint32_t D = m->D, F = m->F, V = m->V;
        const uint32_t g = uint32_t(tp_size), r = uint32_t(tp_rank);
        m->Hl = m->H / g; m->h0 = r * m->Hl; m->Dl = m->Hl * m->dh;
        m->f0 = uint32_t(uint64_t(F) * r / g); m->Fl = uint32_t(uint64_t(F) * (r + 1) / g) - m->f0;
        m->v0 = uint32_t(uint64_t(V) * r / g); m->Vl = uint32_t(uint64_t(V) * (r + 1) / g) - m->v0;
        const uint32_t Dl = m->Dl, Fl = m->Fl, q0 = m->h0 * m->dh, f0 = m->f0;
        auto check_qt = [&](const dimg_qtensor& t, uint32_t rr, uint32_t k, const char* what) {
            if (t.rows != rr || t.cols != k) fail(DIMG_EINVAL, std::string("model_upload: bad shape of ") + what);
        };
        // staging for the largest matrix (row-major, rows padded to 4)
        size_t stage_bytes = 0;
        auto grow = [&](uint32_t rows, uint32_t K) {
            stage_bytes = std::max(stage_bytes, size_t((rows + 3) / 4) * 4 * pad16(K));
        };
        grow(3 * D, D); grow(2 * F, D); grow(D, F); grow(V, D);
        int8_t* staging = nullptr;
        if (!rowmajor) CK(cudaMalloc(&staging, stage_bytes));
        struct Free { int8_t* p; ~Free() { if (p) cudaFree(p); } } free_staging{staging};
        m->layers.resize(m->L);
        for (uint32_t l = 0; l < m->L; ++l) {
            const dimg_qtensor* t = d->layers + 7 * size_t(l);
            const char* names[7] = {"wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"};
            for (int i = 0; i < 7; ++i)
                check_qt(t[i], i < 4 ? D : (i < 6 ? F : D), i < 6 ? D : F, names[i]);
            auto& lw = m->layers[l];
            // column-parallel q/k/v: this rank's heads (rows q0 .. q0 + Dl of each)
            std::vector<int64_t> s(3 * size_t(Dl));
            for (int i = 0; i < 3; ++i)
                std::copy(t[i].scales + q0, t[i].scales + q0 + Dl, s.begin() + size_t(i) * Dl);
            const size_t qo = size_t(q0) * D;
            lw.qkv = upload_mat(*m, 3 * Dl, D,
                                {{t[0].data + qo, Dl, 0, 1}, {t[1].data + qo, Dl, Dl, 1}, {t[2].data + qo, Dl, 2 * Dl, 1}},
                                s, staging);
            // row-parallel wo: the same heads' input columns, every output row
            lw.wo = upload_mat(*m, D, Dl, {{t[3].data + q0, D, 0, 1, D}},
                               std::vector<int64_t>(t[3].scales, t[3].scales + D), staging);
            // column-parallel gate/up rows f0 .. f0 + Fl, interleaved
            std::vector<int64_t> gs(2 * size_t(Fl));
            for (uint32_t i = 0; i < Fl; ++i) {
                gs[2 * i] = t[4].scales[f0 + i];
                gs[2 * i + 1] = t[5].scales[f0 + i];
            }
            lw.gu = upload_mat(*m, 2 * Fl, D, {{t[4].data + size_t(f0) * D, Fl, 0, 2}, {t[5].data + size_t(f0) * D, Fl, 1, 2}},
                               gs, staging);
            // row-parallel w_down: input columns f0 .. f0 + Fl
            lw.down = upload_mat(*m, D, Fl, {{t[6].data + f0, D, 0, 1, F}},
                                 std::vector<int64_t>(t[6].scales, t[6].scales + D), staging);
            lw.attn_norm = upload(m->mem, d->norms + size_t(2 * l) * D, D);
            lw.ffn_norm = upload(m->mem, d->norms + size_t(2 * l + 1) * D, D);
            lw.attn_unit = all_one(d->norms + size_t(2 * l) * D, D);
            lw.ffn_unit = all_one(d->norms + size_t(2 * l + 1) * D, D);
        }
        check_qt(d->tok_embd, V, D, "tok_embd");
        check_qt(d->output, V, D, "output");
        m->embd = upload(m->mem, d->tok_embd.data, size_t(V) * D);
        m->embd_s = upload(m->mem, d->tok_embd.scales, V);
        // column-parallel lm_head: vocab rows v0 .. v0 + Vl
        m->head = upload_mat(*m, m->Vl, D, {{d->output.data + size_t(m->v0) * D, m->Vl, 0, 1}},
                             std::vector<int64_t>(d->output.scales + m->v0, d->output.scales + m->v0 + m->Vl),
                             staging);
        m->final_norm = upload(m->mem, d->norms + size_t(2 * m->L) * D, D);
        m->final_unit = all_one(d->norms + size_t(2 * m->L) * D, D);
        // RoPE tables: imported (RTAB) or built on the host (rope.cpp:17-39)
        const uint32_t half = m->dh / 2, ctx = d->cfg.max_ctx;
        if (d->rope_cos && d->rope_sin) {
            if (d->rope_max_ctx < ctx)
                fail(DIMG_EINVAL, "session: imported tables do not fit the model");
            m->rope_cos = upload(m->mem, d->rope_cos, size_t(ctx) * half);
            m->rope_sin = upload(m->mem, d->rope_sin, size_t(ctx) * half);
        } else {
            std::vector<int64_t> rc(size_t(ctx) * half), rs(size_t(ctx) * half);
            build_rope(d->cfg.rope_theta, m->dh, ctx, rc.data(), rs.data());
            m->rope_cos = upload(m->mem, rc.data(), rc.size());
            m->rope_sin = upload(m->mem, rs.data(), rs.size());
        }
        // inv_sqrt(dh * ONE) on the host with the same integer recurrence
        {
            int64_t x = int64_t(m->dh) * kOne;
            int b = 63 - __builtin_clzll(uint64_t(x));
            __int128 y = invsqrt_seed(b);
            for (int it = 0; it < 3; ++it) {
                __int128 t = (y * y) >> 48;
                __int128 u = (__int128(x) * t) >> 16;
                y = (y * ((__int128(3) << 48) - u)) >> 49;
            }
            m->inv_scale = int64_t((y + (__int128(1) << 31)) >> 32);
        }
        CK(cudaDeviceSynchronize());
        return m.release();
    }
}
// A session on model m (or on one tensor-parallel shard of it: the local
// heads, FFN rows and vocab rows; the sizes below are the shard's), with
// `grid` CTAs for the persistent kernel (0: one per SM).
dimg_session* session_new(dimg_model* m, uint32_t keep_logits_cap, uint32_t grid) {
    {
        CK(cudaSetDevice(m->device));
        auto s = std::make_unique<dimg_session>();
        s->m = m;
        CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        const size_t ctx = m->cfg.max_ctx;
        s->x = s->mem.alloc<int64_t>(m->D);
        s->x32 = s->mem.alloc<int32_t>(m->Kd);
        CK(cudaMemsetAsync(s->x32, 0, size_t(m->Kd) * 4, s->stream));
        s->qkv = s->mem.alloc<int64_t>(3 * size_t(m->Dl));
        s->att = s->mem.alloc<int64_t>(m->Dl);
        s->h = s->mem.alloc<int64_t>(m->Fl);
        size_t kv = size_t(m->L) * m->Hl * ctx * m->dh;
        s->kc = s->mem.alloc<int64_t>(kv);
        s->vc = s->mem.alloc<int64_t>(kv);
        s->scores = s->mem.alloc<int64_t>(size_t(m->Hl) * ctx);
        s->keep_cap = keep_logits_cap;
        s->logits = s->mem.alloc<int64_t>(size_t(keep_logits_cap + 1) * m->Vl);
        s->tokens = s->mem.alloc<uint32_t>(ctx + 1);
        s->ctl = s->mem.alloc<Ctl>(1);
        s->bar = s->mem.alloc<unsigned int>(64);
        s->xg = s->mem.alloc<unsigned long long>(size_t(m->Hl) * ctx * 2);
        s->qkv_x = s->mem.alloc<unsigned long long>(size_t(3) * m->Dl * 2);
        s->xwords = s->mem.alloc<uint32_t>(size_t(2) * m->Kd);
        CK(cudaMemsetAsync(s->xwords, 0, size_t(8) * m->Kd, s->stream));
        CK(cudaMemsetAsync(s->qkv_x, 0, size_t(3) * m->Dl * 16, s->stream));
        CK(cudaMemsetAsync(s->xg, 0, size_t(m->Hl) * ctx * 16, s->stream));
        s->kc32 = s->mem.alloc<int32_t>(kv);
        s->vc32 = s->mem.alloc<int32_t>(kv);
        s->kvwide = s->mem.alloc<uint32_t>(size_t(m->L) * m->Hl);
        CK(cudaMemsetAsync(s->kvwide, 0, size_t(m->L) * m->Hl * 4, s->stream));
        // one CTA per SM; shared memory = weight ring + limb planes + row accumulators
        s->grid = grid ? grid : uint32_t(m->ctx->sm_count);
        s->parts = s->mem.alloc<ArgPart>(s->grid);
        s->parts_w = s->mem.alloc<unsigned long long>(size_t(8) * s->grid);
        CK(cudaMemsetAsync(s->parts_w, 0, size_t(64) * s->grid, s->stream));
        s->words_att = s->mem.alloc<uint32_t>(pad16(m->Dl));
        s->words_h = s->mem.alloc<uint32_t>(pad16(m->Fl));
        CK(cudaMemsetAsync(s->words_att, 0, size_t(4) * pad16(m->Dl), s->stream));
        CK(cudaMemsetAsync(s->words_h, 0, size_t(4) * pad16(m->Fl), s->stream));
        s->ssq = s->mem.alloc<unsigned long long>(2 * size_t(m->L));
        s->host_stages = step_program(*s);
        // shared staging: rmsnorm = the int64 vector + 3 planes (11 Kp bytes);
        // plain = 3 planes; attention = head scratch + score strip. 8-limb
        // planes (out-of-range inputs) live in a global per-CTA scratch. The
        // rest of shared memory is the weight ring: as many 4 KB slots per
        // warp as fit (up to PK_MAX_DEPTH).
        size_t need = attn_scratch_bytes(m->dh, m->cfg.max_ctx);
        uint32_t kp_max = 0;
        for (const auto& st : s->host_stages) {
            if (st.kind != SK_GEMV) continue;
            size_t b = size_t(st.mode == MODE_PLAIN ? 3 : 11) * st.Kp;
            need = std::max(need, b);
            kp_max = std::max(kp_max, st.Kp);
        }
        s->planes_bytes = uint32_t((need + 127) & ~size_t(127));
        const size_t bars = size_t(PK_WARPS) * PK_MAX_DEPTH * 8;
        // per-stage stream info (FetchInfo) for the step program or a probe program
        const size_t fi_bytes = std::max<size_t>(s->host_stages.size(), 129) * sizeof(FetchInfo);
        const size_t avail = size_t(m->ctx->smem_optin) > s->planes_bytes + bars + fi_bytes
                                 ? size_t(m->ctx->smem_optin) - s->planes_bytes - bars - fi_bytes
                                 : 0;
        s->ring_depth = uint32_t(std::min<size_t>(PK_MAX_DEPTH, avail / (size_t(PK_WARPS) * PK_SLOT)));
        if (s->ring_depth < 2)
            fail(DIMG_EINVAL, "session: shapes need " + std::to_string(s->planes_bytes) +
                                  " B of shared staging per CTA (d_ffn or max_ctx too large for this build)");
        s->smem = size_t(PK_WARPS) * s->ring_depth * PK_SLOT + s->planes_bytes + bars + fi_bytes;
        s->wide_stride = 2 * kp_max;  // 8 planes x Kp/4 words
        s->wide_planes = s->mem.alloc<uint32_t>(size_t(s->grid) * s->wide_stride);
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_persistent_kernel, PK_THREADS,
                                                         s->smem));
        if (per_sm < 1) fail(DIMG_ECUDA, "session: persistent kernel does not fit one SM");
        s->stages = s->mem.alloc<PkStage>(s->host_stages.size());
        CK(cudaMemcpyAsync(s->stages, s->host_stages.data(), s->host_stages.size() * sizeof(PkStage),
                           cudaMemcpyHostToDevice, s->stream));
        CK(cudaMemsetAsync(s->ctl, 0, sizeof(Ctl), s->stream));
        CK(cudaMemsetAsync(s->tokens, 0, (ctx + 1) * 4, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        return s.release();
    }
}

}  // namespace

extern "C" {

dimg_status dimg_model_free(dimg_model* m) {
    DIMG_API_GUARD({
        if (m) {
            cudaSetDevice(m->device);
            delete m;
        }
    })
}

dimg_status dimg_inv_sqrt_q16(int64_t x, int64_t* out) {
    // the device kernels' inv_sqrt_q16 (kernels/q16.cuh: the 64-bit Newton
    // path, else int128), run on the host -- for its parity test
    DIMG_API_GUARD({
        if (x <= 0) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
        const int b = 63 - __builtin_clzll(uint64_t(x));
        int64_t r = inv_sqrt_q16_u64(x, b, invsqrt_seed(b));
        if (r < 0) {
            __int128 y = invsqrt_seed(b);
            for (int it = 0; it < 3; ++it) {
                __int128 t = (y * y) >> 48;
                __int128 u = (__int128(x) * t) >> 16;
                y = (y * ((__int128(3) << 48) - u)) >> 49;
            }
            r = int64_t((y + (__int128(1) << 31)) >> 32);
        }
        *out = r;
    })
}

dimg_status dimg_model_bytes_on_device(const dimg_model* m, uint64_t* bytes) {
    DIMG_API_GUARD(*bytes = m->mem.bytes)
}

dimg_status dimg_session_create(dimg_model* m, uint32_t keep_logits_cap, dimg_session** out) {
    DIMG_API_GUARD({
        if (m->tp_size > 1 || m->rowmajor)
            fail(DIMG_EINVAL, "session: a tensor-parallel shard generates through dimg_tp");
        *out = session_new(m, keep_logits_cap, 0);
    })
}

dimg_status dimg_session_free(dimg_session* s) {
    DIMG_API_GUARD({
        if (s) {
            cudaSetDevice(s->m->device);
            cudaStreamSynchronize(s->stream);
            delete s;
        }
    })
}

dimg_status dimg_session_reset(dimg_session* s) {
    DIMG_API_GUARD({
        CK(cudaSetDevice(s->m->device));
        write_ctl(*s, 0, 0, 0);
        s->len = 0;
        CK(cudaStreamSynchronize(s->stream));
    })
}

dimg_status dimg_session_len(const dimg_session* s, uint32_t* len) { DIMG_API_GUARD(*len = s->len) }

dimg_status dimg_session_forward(dimg_session* s, uint32_t token, uint32_t pos, int64_t* logits) {
    // InferenceSession::forward checks (proj/src/engine.cpp:81-83)
    DIMG_API_GUARD({
        const dimg_model& m = *s->m;
        if (token >= m.cfg.vocab) fail(DIMG_ERANGE, "forward: token out of range");
        if (pos >= m.cfg.max_ctx) fail(DIMG_ECTX, "forward: context overflow");
        if (pos != s->len) fail(DIMG_ELOGIC, "forward: pos must equal cache length");
        CK(cudaSetDevice(m.device));
        CK(cudaMemcpyAsync(s->tokens + pos, &token, 4, cudaMemcpyHostToDevice, s->stream));
        // logits land in slot 0 (kept) or the scratch row 0 when keep_cap == 0;
        // the head appends the argmax at tokens[pos + 1], which the next
        // forward overwrites
        write_ctl(*s, pos, pos, s->keep_cap >= 1 ? 1 : 0);
        launch_pk(*s, s->stages, n_layer_stages(*s), 1, 0);
        s->len = pos + 1;
        if (logits)
            CK(cudaMemcpyAsync(logits, s->logits, size_t(m.V) * 8, cudaMemcpyDeviceToHost, s->stream));
        check_ctl_err(*s);
    })
}

dimg_status dimg_generate_greedy(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt,
                                 uint32_t max_new, uint32_t* tokens_out, uint8_t hash_out[32],
                                 int64_t* logits_out) {
    // run_generation (proj/src/engine.cpp:31-54): P + N - 1 forwards, the
    // lm_head only where a selection follows -- one persistent launch.
    DIMG_API_GUARD({
        begin(*s, prompt, n_prompt, max_new, logits_out != nullptr);
        g_generations.fetch_add(1, std::memory_order_relaxed);
        if (max_new > 0) {
            const uint32_t np = n_prompt - 1;
            if (try_prefill_tc(*s)) launch_pk(*s, s->stages, n_layer_stages(*s), max_new, 0);
            else launch_pk(*s, s->stages, n_layer_stages(*s), np + max_new, np);
            s->len = np + max_new;
            CK(cudaMemcpyAsync(tokens_out, s->tokens + n_prompt, size_t(max_new) * 4,
                               cudaMemcpyDeviceToHost, s->stream));
            if (logits_out)
                CK(cudaMemcpyAsync(logits_out, s->logits, size_t(max_new) * s->m->V * 8,
                                   cudaMemcpyDeviceToHost, s->stream));
        }
        check_ctl_err(*s);
        if (hash_out) {
            auto d = b3::hash(tokens_out, size_t(max_new) * 4, 1);
            std::memcpy(hash_out, d.data(), 32);
        }
    })
}

dimg_status dimg_generate_greedy_batch(dimg_model* m, uint32_t n_seqs, const uint32_t* prompts,
                                       const uint32_t* p_lens, uint32_t max_new, uint32_t* tokens_out,
                                       uint8_t* hashes_out, uint32_t* path) {
    // run_generation (proj/src/engine.cpp:31-54) for every sequence, stepped
    // together on the tensor cores; an exact per-sequence rerun when some
    // value falls outside the batch path's fast representations.
    DIMG_API_GUARD({
        if (m->rowmajor) fail(DIMG_EINVAL, "batch: a tensor-parallel shard generates through dimg_tp");
        CK(cudaSetDevice(m->device));
        std::vector<std::vector<uint32_t>> ps(n_seqs);
        size_t off = 0;
        for (uint32_t b = 0; b < n_seqs; ++b) {
            ps[b].assign(prompts + off, prompts + off + p_lens[b]);
            off += p_lens[b];
            check_prompt(*m, ps[b].data(), p_lens[b], max_new);
        }
        uint32_t used = 0;
        std::unique_lock<std::mutex> lk(m->batch_mu);
        if (n_seqs && batch_shape_ok(*m) && generate_batch_tc(m, n_seqs, ps, max_new, tokens_out)) {
            used = 1;
            g_generations.fetch_add(n_seqs, std::memory_order_relaxed);
        } else if (n_seqs) {
            dimg_session* s = nullptr;
            const dimg_status st = dimg_session_create(m, 0, &s);
            if (st != DIMG_OK) return st;
            std::unique_ptr<dimg_session, dimg_status (*)(dimg_session*)> keep(s, dimg_session_free);
            for (uint32_t b = 0; b < n_seqs; ++b) {
                const dimg_status g = dimg_generate_greedy(s, ps[b].data(), p_lens[b], max_new,
                                                           tokens_out + size_t(b) * max_new, nullptr, nullptr);
                if (g != DIMG_OK) return g;
            }
        }
        if (path) *path = used;
        for (uint32_t b = 0; b < n_seqs && hashes_out; ++b) {
            auto d = b3::hash(tokens_out + size_t(b) * max_new, size_t(max_new) * 4, 1);
            std::memcpy(hashes_out + 32 * size_t(b), d.data(), 32);
        }
    })
}

dimg_status dimg_session_begin(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt,
                               uint32_t max_new) {
    DIMG_API_GUARD(begin(*s, prompt, n_prompt, max_new, false))
}

dimg_status dimg_session_prefill(dimg_session* s) { DIMG_API_GUARD(run_prefill(*s)) }

dimg_status dimg_session_decode(dimg_session* s, uint32_t n_steps) {
    DIMG_API_GUARD({
        if (uint64_t(s->len) + n_steps > s->m->cfg.max_ctx)
            fail(DIMG_ECTX, "decode: context overflow");
        run_decode(*s, n_steps);
    })
}

dimg_status dimg_session_sync(dimg_session* s) { DIMG_API_GUARD(check_ctl_err(*s)) }

dimg_status dimg_session_tokens(dimg_session* s, uint32_t* out, uint32_t n_generated) {
    DIMG_API_GUARD({
        CK(cudaMemcpyAsync(out, s->tokens + s->n_prompt, size_t(n_generated) * 4,
                           cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    })
}

dimg_status dimg_session_stream(dimg_session* s, void** stream) { DIMG_API_GUARD(*stream = s->stream) }

dimg_status dimg_session_time_decode(dimg_session* s, uint32_t n_steps, float* ms) {
    DIMG_API_GUARD({
        if (uint64_t(s->len) + n_steps > s->m->cfg.max_ctx)
            fail(DIMG_ECTX, "decode: context overflow");
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(s->stream));
        CK(cudaEventRecord(e0, s->stream));
        run_decode(*s, n_steps);
        CK(cudaEventRecord(e1, s->stream));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        check_ctl_err(*s);
    })
}

dimg_status dimg_session_time_prefill(dimg_session* s, float* ms, uint32_t* tensor_cores) {
    // The prefill of the prompt given to dimg_session_begin, between CUDA
    // events on the session stream (tensor-core path when it applies).
    DIMG_API_GUARD({
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(s->stream));
        const uint64_t before = s->tc_prefills;
        CK(cudaEventRecord(e0, s->stream));
        run_prefill(*s);
        CK(cudaEventRecord(e1, s->stream));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tensor_cores = s->tc_prefills > before ? 1 : 0;
        check_ctl_err(*s);
    })
}

dimg_status dimg_session_time_kernel(dimg_session* s, int which, uint32_t n, float* ms_per_launch,
                                    uint64_t* bytes_per_launch) {
    // Runs a probe program of n stages of one kind (layers cycled, so the
    // weights stream from HBM) in one persistent launch between CUDA events;
    // the per-stage time includes its grid barrier, i.e. the real cost of the
    // stage inside a decode step. Algorithmic bytes = int8 weights + int64
    // scales + int64 gains + activation I/O.
    DIMG_API_GUARD({
        const dimg_model& m = *s->m;
        CK(cudaSetDevice(m.device));
        if (which < 0 || which > 4) fail(DIMG_EINVAL, "time_kernel: which in 0..4");
        if (n == 0 || n > 128) fail(DIMG_EINVAL, "time_kernel: n in 1..128");
        const uint64_t D = m.D, F = m.F, V = m.V;
        const uint64_t bytes[5] = {3 * D * D + 3 * D * 8 + D * 8 + D * 8 + 3 * D * 8,
                                   D * D + D * 8 + D * 8 + 2 * D * 8,
                                   2 * F * D + 2 * F * 8 + D * 8 + D * 8 + F * 8,
                                   D * F + D * 8 + F * 8 + 2 * D * 8,
                                   V * D + V * 8 + D * 8 + D * 8};
        const uint32_t idx[4] = {0, 2, 3, 4};
        std::vector<PkStage> prog;
        for (uint32_t i = 0; i < n; ++i) {
            PkStage st = which == 4 ? s->host_stages.back()
                                    : s->host_stages[5 * (i % m.L) + idx[which]];
            if (st.mode == MODE_EMBED) st.mode = MODE_NORM;
            if (st.epi == EPI_ARGMAX) st.epi = EPI_STORE;  // the probe never appends tokens
            st.ssq_in = nullptr;  // the probe has no producer stages: sums computed in place
            st.ssq_out = nullptr;
            st.ssq_clear = nullptr;
            st.ytag = nullptr;  // no attention stage follows
            st.no_barrier = 0;
            st.in_words = nullptr;  // plain inputs: planes straight from the int64 vector
            st.x32_in = nullptr;
            st.x32_out = nullptr;
            st.xw_in = nullptr;
            st.xw_out = nullptr;
            st.resid_embed = 0;
            st.out_words = nullptr;
            prog.push_back(st);
        }
        if (!s->probe_stages || n > 0) {
            s->probe_stages = s->mem.alloc<PkStage>(prog.size());
            CK(cudaMemcpyAsync(s->probe_stages, prog.data(), prog.size() * sizeof(PkStage),
                               cudaMemcpyHostToDevice, s->stream));
        }
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(s->stream));
        CK(cudaEventRecord(e0, s->stream));
        launch_pk(*s, s->probe_stages, n, 1, 1);
        CK(cudaEventRecord(e1, s->stream));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        check_ctl_err(*s);
        *ms_per_launch = ms / float(n);
        *bytes_per_launch = bytes[which];
    })
}

dimg_status dimg_session_trace(dimg_session* s, uint32_t n_steps, uint64_t* out, uint32_t cap) {
    // n decode steps with CTA 0 stamping %globaltimer at each stage's start,
    // after its prologue, after its chunk loop and before its grid barrier.
    DIMG_API_GUARD({
        if (uint64_t(s->len) + n_steps > s->m->cfg.max_ctx)
            fail(DIMG_ECTX, "decode: context overflow");
        unsigned long long* d = s->mem.alloc<unsigned long long>(size_t(cap) * DIMG_TRACE_WORDS);
        CK(cudaMemsetAsync(d, 0, size_t(cap) * DIMG_TRACE_WORDS * 8, s->stream));
        launch_pk(*s, s->stages, n_layer_stages(*s), n_steps, 0, d, cap);
        s->len += n_steps;
        CK(cudaMemcpyAsync(out, d, size_t(cap) * DIMG_TRACE_WORDS * 8, cudaMemcpyDeviceToHost, s->stream));
        check_ctl_err(*s);
    })
}

#ifdef DIMG_CHUNK_TRACE
// Experiment build only: copies the per-chunk ring-wait log (g_ct) out.
extern "C" int dimg_debug_chunk_trace(uint64_t* out) {
    return cudaMemcpyFromSymbol(out, dimg::dev::g_ct, sizeof(dimg::dev::g_ct)) == cudaSuccess ? 0 : 1;
}
#endif

dimg_status dimg_session_trace_all(dimg_session* s, uint32_t n_steps, uint64_t* out, uint32_t cap) {
    // n decode steps with EVERY CTA stamping %globaltimer at the end of each
    // GEMV stage's prologue and chunk loop: out[(i * grid + cta) * 2 + 0/1]
    // for the first cap stages (the hand-off skew between CTAs)
    DIMG_API_GUARD({
        if (uint64_t(s->len) + n_steps > s->m->cfg.max_ctx)
            fail(DIMG_ECTX, "decode: context overflow");
        const size_t n = size_t(cap) * s->grid * 2;
        unsigned long long* d = s->mem.alloc<unsigned long long>(n);
        unsigned long long* d0 = s->mem.alloc<unsigned long long>(size_t(cap) * DIMG_TRACE_WORDS);
        CK(cudaMemsetAsync(d, 0, n * 8, s->stream));
        CK(cudaMemsetAsync(d0, 0, size_t(cap) * DIMG_TRACE_WORDS * 8, s->stream));
        launch_pk(*s, s->stages, n_layer_stages(*s), n_steps, 0, d0, cap, d);
        s->len += n_steps;
        CK(cudaMemcpyAsync(out, d, n * 8, cudaMemcpyDeviceToHost, s->stream));
        check_ctl_err(*s);
    })
}

dimg_status dimg_session_launches(const dimg_session* s, uint32_t* per_decode, uint32_t* per_prefill) {
    // one persistent launch per call; it runs every stage of every step
    DIMG_API_GUARD({
        *per_decode = 1;
        *per_prefill = 1;
    })
}

dimg_status dimg_session_stats(dimg_session* s, uint64_t out[4]) {
    DIMG_API_GUARD({
        Ctl c;
        CK(cudaMemcpyAsync(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        out[0] = c.stats[0];
        out[1] = c.err;
        out[2] = c.stats[1];
        out[3] = (s->tc_prefills & 0xFFFFFFFFull) | (s->tc_fallbacks << 32);
    })
}

}  // extern "C"

// ---- operator-level exports ------------------------------------------------
// Each runs the engine's own device code on host buffers (upload, one launch,
// download) so proj/src/kernels.cpp's operators can be checked one by one.

namespace {

struct OpScope {
    DevCtx& c;
    std::unique_lock<std::recursive_mutex> lk;
    DevBuf mem;
    explicit OpScope(int device) : c(dev_ctx(device)), lk(c.op_mu) {
        CK(cudaSetDevice(device));
        CK(cudaMemsetAsync(c.op_ctl, 0, sizeof(Ctl), c.op_stream));
    }
    template <class T>
    T* put(const T* src, size_t n) {
        T* d = mem.alloc<T>(n);
        if (n) CK(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, c.op_stream));
        return d;
    }
    int8_t* put_padded(const dimg_qtensor& w, uint32_t row_stride, uint32_t rows_total,
                       uint32_t row0, int8_t* dst = nullptr) {
        const uint32_t Kp = pad16(w.cols);
        if (!dst) {
            dst = mem.alloc<int8_t>(size_t(rows_total) * Kp);
            CK(cudaMemsetAsync(dst, 0, size_t(rows_total) * Kp, c.op_stream));
        }
        put_rows(dst, Kp, row0, row_stride, w.data, w.rows, w.cols, c.op_stream);
        return dst;
    }
    template <class T>
    void get(T* dst, const T* src, size_t n) {
        CK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, c.op_stream));
        CK(cudaStreamSynchronize(c.op_stream));
        uint32_t err[2] = {0, 0};
        CK(cudaMemcpy(err, &c.op_ctl->err, 8, cudaMemcpyDeviceToHost));
        if (err[0] & 1u) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
        if (err[1] & 2u) fail(DIMG_EDOMAIN, "exp_neg_lut: argument outside [0, 8]");
    }
    GemvArgs args() {
        GemvArgs a{};
        a.ctl = c.op_ctl;
        a.exp_lut = c.exp_lut;
        a.seeds = c.seeds;
        return a;
    }
};

__global__ void rmsnorm_op_kernel(GemvArgs a, int64_t* out) {
    __shared__ u128 scratch[32];
    int64_t r = norm_factor<MODE_NORM>(a, 0, nullptr, scratch);
    for (uint32_t j = threadIdx.x; j < a.K; j += blockDim.x)
        out[j] = input_elem<MODE_NORM>(a, j, r, 0, nullptr);
}

__global__ void softmax_op_kernel(int64_t* s, uint32_t n, const int64_t* exp_lut) {
    __shared__ u128 red[32];
    softmax_strip(s, n, exp_lut, red);
}

__global__ void set_pos_kernel(Ctl* ctl, uint32_t pos) { ctl->pos = pos; }

}  // namespace

extern "C" {

dimg_status dimg_op_dense(int device, const dimg_qtensor* w, const int64_t* x, int64_t* out) {
    // dense_forward (proj/src/kernels.cpp:18-30)
    DIMG_API_GUARD({
        OpScope o(device);
        GemvArgs a = o.args();
        a.W = o.put_padded(*w, 1, w->rows, 0);
        a.scales = o.put(w->scales, w->rows);
        a.rows = w->rows; a.K = w->cols; a.Kp = pad16(w->cols);
        a.x = o.put(x, w->cols);
        a.y = o.mem.alloc<int64_t>(w->rows);
        launch_gemv<EPI_STORE, MODE_PLAIN>(a, o.c, o.c.op_stream);
        CK(cudaGetLastError());
        o.get(out, a.y, w->rows);
    })
}

// BLAKE3 of len device bytes on stream st: the chunk kernel folds 256
// chunks per CTA, each further launch 256 nodes, until the root
// (kernels/blake3.cuh). ms (optional): CUDA-event time of the kernels.
static void blake3_device_run(const uint8_t* d, size_t len, uint8_t out[32], cudaStream_t st, DevBuf& mem,
                              float* ms) {
    if (len == 0) {  // one empty chunk: nothing to stream
        const auto h = b3::hash(nullptr, 0, 1);
        std::memcpy(out, h.data(), 32);
        if (ms) *ms = 0.f;
        return;
    }
    const uint64_t n_chunks = (len + 1023) / 1024;
    uint64_t g = (n_chunks + B3_FOLD - 1) / B3_FOLD;
    uint32_t* a = mem.alloc<uint32_t>(g * 8);
    uint32_t* b = mem.alloc<uint32_t>(((g + B3_FOLD - 1) / B3_FOLD) * 8 + 8);
    uint32_t* root = mem.alloc<uint32_t>(8);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ms) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, st));
    }
    b3_chunks_kernel<<<uint32_t(g), B3_FOLD, 0, st>>>(d, len, a, root);
    for (uint64_t cnt = g; cnt > 1; cnt = (cnt + B3_FOLD - 1) / B3_FOLD) {
        b3_fold_kernel<<<uint32_t((cnt + B3_FOLD - 1) / B3_FOLD), B3_FOLD, 0, st>>>(a, cnt, b, root);
        std::swap(a, b);
    }
    CK(cudaGetLastError());
    if (ms) {
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    CK(cudaMemcpyAsync(out, root, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

dimg_status dimg_blake3_device(int device, const void* data, size_t len, uint8_t out[32], float* ms) {
    // weight_hash / deserialize (proj/src/model.cpp:310-316) on device-resident bytes
    DIMG_API_GUARD({
        if (!data && len) fail(DIMG_EINVAL, "blake3_device: null data");
        OpScope o(device);
        blake3_device_run(static_cast<const uint8_t*>(data), len, out, o.c.op_stream, o.mem, ms);
    })
}

dimg_status dimg_generation_counter(uint64_t* out) { DIMG_API_GUARD(*out = g_generations.load()) }

dimg_status dimg_make_attestation(int device, const uint8_t* model_bytes, size_t n_bytes, const uint32_t* prompt,
                                  size_t n_prompt, const uint8_t output_hash[32], uint64_t bond,
                                  uint64_t challenge_period, dimg_attestation* out) {
    // make_attestation (proj/src/attest.cpp:68-78)
    DIMG_API_GUARD({
        const dimg_status st = dimg_blake3_gpu(device, model_bytes, n_bytes, out->model_id);
        if (st != DIMG_OK) return st;
        const auto ih = b3::hash(prompt, n_prompt * 4, 1);  // hash_token_ids (u32 LE)
        std::memcpy(out->input_hash, ih.data(), 32);
        std::memcpy(out->output_hash, output_hash, 32);
        out->bond = bond;
        out->challenge_period = challenge_period;
    })
}

dimg_status dimg_verify_by_reexecution(int device, const dimg_attestation* att, const uint8_t* model_bytes,
                                       size_t n_bytes, const uint32_t* prompt, size_t n_prompt, uint32_t max_new,
                                       dimg_verify_outcome* out) {
    // verify_by_reexecution (proj/src/attest.cpp:89-117): the first stage whose
    // recomputed digest differs refutes; only an intact model and prompt are
    // re-executed (once).
    DIMG_API_GUARD({
        *out = dimg_verify_outcome{};
        auto refute = [&](uint32_t stage, const uint8_t* expected, const uint8_t* found) {
            out->refuted_stage = stage;
            std::memcpy(out->expected, expected, 32);
            std::memcpy(out->found, found, 32);
        };
        uint8_t found[32];
        dimg_status st = dimg_blake3_gpu(device, model_bytes, n_bytes, found);
        if (st != DIMG_OK) return st;
        if (std::memcmp(found, att->model_id, 32)) {
            refute(0, att->model_id, found);
            return DIMG_OK;
        }
        const auto ih = b3::hash(prompt, n_prompt * 4, 1);
        if (std::memcmp(ih.data(), att->input_hash, 32)) {
            refute(1, att->input_hash, ih.data());
            return DIMG_OK;
        }
        dimg_host_model* hm = nullptr;
        if ((st = dimg_host_model_from_bytes(model_bytes, n_bytes, &hm)) != DIMG_OK) return st;  // ParseError
        std::unique_ptr<dimg_host_model, dimg_status (*)(dimg_host_model*)> keep_hm(hm, dimg_host_model_free);
        dimg_model_desc desc;
        if ((st = dimg_host_model_desc(hm, &desc)) != DIMG_OK) return st;
        dimg_model* dm = nullptr;
        if ((st = dimg_model_upload(device, &desc, 0, 1, &dm)) != DIMG_OK) return st;
        std::unique_ptr<dimg_model, dimg_status (*)(dimg_model*)> keep_dm(dm, dimg_model_free);
        dimg_session* s = nullptr;
        if ((st = dimg_session_create(dm, 0, &s)) != DIMG_OK) return st;
        std::unique_ptr<dimg_session, dimg_status (*)(dimg_session*)> keep_s(s, dimg_session_free);
        std::vector<uint32_t> toks(max_new);
        uint8_t oh[32];
        if ((st = dimg_generate_greedy(s, prompt, uint32_t(n_prompt), max_new, toks.data(), oh, nullptr)) != DIMG_OK)
            return st;
        if (std::memcmp(oh, att->output_hash, 32)) {
            refute(2, att->output_hash, oh);
            return DIMG_OK;
        }
        out->confirmed = 1;
    })
}

dimg_status dimg_dispute_game(int device, const dimg_attestation* att, const uint8_t* model_bytes, size_t n_bytes,
                              const uint32_t* prompt, size_t n_prompt, uint32_t max_new, uint32_t* winner,
                              dimg_verify_outcome* out) {
    // dispute_game (proj/src/attest.cpp:119-125): the challenger wins iff
    // re-execution refutes the attestation
    DIMG_API_GUARD({
        const dimg_status st =
            dimg_verify_by_reexecution(device, att, model_bytes, n_bytes, prompt, n_prompt, max_new, out);
        if (st != DIMG_OK) return st;
        *winner = out->confirmed ? 0 : 1;
    })
}

dimg_status dimg_sample_key(int device, const uint8_t* model_bytes, size_t n_bytes, const uint32_t* prompt,
                            size_t n_prompt, uint8_t key[32]) {
    // generate_sampled's RNG key (proj/src/engine.cpp:151-157): BLAKE3 of the
    // model bytes followed by the prompt ids (u32 LE), one device buffer
    DIMG_API_GUARD({
        OpScope o(device);
        uint8_t* d = o.mem.alloc<uint8_t>(n_bytes + 4 * n_prompt);
        if (n_bytes) CK(cudaMemcpyAsync(d, model_bytes, n_bytes, cudaMemcpyHostToDevice, o.c.op_stream));
        if (n_prompt)
            CK(cudaMemcpyAsync(d + n_bytes, prompt, 4 * n_prompt, cudaMemcpyHostToDevice, o.c.op_stream));
        blake3_device_run(d, n_bytes + 4 * n_prompt, key, o.c.op_stream, o.mem, nullptr);
    })
}

dimg_status dimg_op_sample(int device, const int64_t* logits, uint32_t V, int64_t temperature, uint32_t draw,
                           uint32_t* out) {
    // sample_from_logits (proj/src/engine.cpp:122-139) of one row with a given draw
    DIMG_API_GUARD({
        if (temperature <= 0) fail(DIMG_EINVAL, "sample: temperature must be positive");
        if (V == 0) fail(DIMG_EINVAL, "sample: empty logits");
        OpScope o(device);
        const int64_t* dl = o.put(logits, V);
        const uint32_t* dd = o.put(&draw, 1);
        int64_t* scratch = o.mem.alloc<int64_t>(V);
        uint32_t* tok = o.mem.alloc<uint32_t>(2);
        sample_kernel<<<1, SM_THREADS, 0, o.c.op_stream>>>(dl, V, temperature, dd, 0, o.c.exp_lut, scratch, tok, 0,
                                                           &o.c.op_ctl->serr);
        CK(cudaGetLastError());
        o.get(out, tok + 1, 1);
    })
}

dimg_status dimg_generate_sampled(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt, uint32_t max_new,
                                  int64_t temperature, const uint8_t key[32], uint32_t* tokens_out,
                                  uint8_t hash_out[32]) {
    // generate_sampled (proj/src/engine.cpp:148-163): run_generation with
    // sample_from_logits as the selection. The prompt prefill as for greedy;
    // then per step one decode step (logits to the session's scratch row)
    // and the sampling kernel, which writes the token the next step reads --
    // all enqueued back to back, no host round trip per token.
    DIMG_API_GUARD({
        if (temperature <= 0) fail(DIMG_EINVAL, "sample: temperature must be positive");
        const dimg_model& m = *s->m;
        begin(*s, prompt, n_prompt, max_new, false);
        g_generations.fetch_add(1, std::memory_order_relaxed);
        if (max_new > 0) {
            if (s->draws_cap < max_new) {
                CK(cudaStreamSynchronize(s->stream));
                s->draws = s->mem.alloc<uint32_t>(max_new);
                s->draws_cap = max_new;
            }
            if (!s->sample_scratch) s->sample_scratch = s->mem.alloc<int64_t>(m.V);
            chacha::Key k;
            for (int i = 0; i < 8; ++i)
                k[i] = uint32_t(key[4 * i]) | uint32_t(key[4 * i + 1]) << 8 | uint32_t(key[4 * i + 2]) << 16 |
                       uint32_t(key[4 * i + 3]) << 24;
            chacha::Stream rng(k);
            std::vector<uint32_t> dr(max_new);
            for (auto& d : dr) d = rng.u32();
            CK(cudaMemcpyAsync(s->draws, dr.data(), size_t(max_new) * 4, cudaMemcpyHostToDevice, s->stream));
            CK(cudaMemsetAsync(&s->ctl->serr, 0, 4, s->stream));
            run_prefill(*s);  // positions 0 .. P-2
            for (uint32_t step = 0; step < max_new; ++step) {
                const uint32_t pos = n_prompt - 1 + step;
                write_ctl(*s, pos, pos, 0);  // logits to the scratch row 0
                launch_pk(*s, s->stages, n_layer_stages(*s), 1, 0);
                sample_kernel<<<1, SM_THREADS, 0, s->stream>>>(s->logits, m.V, temperature, s->draws, step,
                                                                m.ctx->exp_lut, s->sample_scratch, s->tokens, pos,
                                                                &s->ctl->serr);
            }
            CK(cudaGetLastError());
            s->len = n_prompt - 1 + max_new;
            CK(cudaMemcpyAsync(tokens_out, s->tokens + n_prompt, size_t(max_new) * 4, cudaMemcpyDeviceToHost,
                               s->stream));
        }
        check_ctl_err(*s);
        if (max_new > 0) check_sample_err(*s);
        if (hash_out) {
            auto d = b3::hash(tokens_out, size_t(max_new) * 4, 1);
            std::memcpy(hash_out, d.data(), 32);
        }
    })
}

dimg_status dimg_blake3_gpu(int device, const void* data, size_t len, uint8_t out[32]) {
    // the same for host bytes: one upload, then the device tree hash
    DIMG_API_GUARD({
        if (!data && len) fail(DIMG_EINVAL, "blake3_gpu: null data");
        OpScope o(device);
        const uint8_t* d = o.put(static_cast<const uint8_t*>(data), len);
        blake3_device_run(d, len, out, o.c.op_stream, o.mem, nullptr);
    })
}

dimg_status dimg_op_dense_tokens(int device, const dimg_qtensor* w, const int64_t* x, uint32_t T, int64_t* out) {
    // dense_forward (proj/src/kernels.cpp:18-30) for T tokens: the tensor-core
    // limb GEMM (kind::i8); tokens with an activation beyond 3 limbs go
    // through the exact GEMV instead.
    DIMG_API_GUARD({
        if (T == 0) return DIMG_OK;
        OpScope o(device);
        const uint32_t N = w->rows, K = w->cols, Kp = pad16(K);
        const uint32_t Tp = (T + TG_BN - 1) / TG_BN * TG_BN;
        int8_t* Wr = o.put_padded(*w, 1, N, 0);
        const uint32_t kblk = (K + TG_BK - 1) / TG_BK, rows128 = (N + TG_BM - 1) / TG_BM * TG_BM;
        int8_t* W = o.mem.alloc<int8_t>(size_t(kblk) * rows128 * TG_BK);
        kmajor_kernel<<<1024, 256, 0, o.c.op_stream>>>(Wr, Kp, N, K, W, rows128, kblk);
        int64_t* sc = o.put(w->scales, N);
        int64_t* xd = o.put(x, size_t(T) * K);
        uint8_t* planes = o.mem.alloc<uint8_t>(size_t(3) * Tp * Kp);
        uint32_t* wide = o.mem.alloc<uint32_t>(1);
        CK(cudaMemsetAsync(planes, 0, size_t(3) * Tp * Kp, o.c.op_stream));
        CK(cudaMemsetAsync(wide, 0, 4, o.c.op_stream));
        limbs_kernel<<<1024, 256, 0, o.c.op_stream>>>(xd, T, K, K, planes, Tp, Kp, wide);
        CK(cudaGetLastError());
        int64_t* y = o.mem.alloc<int64_t>(size_t(T) * N);
        TgArgs a{};
        a.n_out = N;
        a.a_rows = rows128;
        a.n_tok = T;
        a.n_kblk = (K + TG_BK - 1) / TG_BK;
        a.limb_rows = Tp;
        a.epi = TG_STORE;
        a.scales = sc;
        a.y = y;
        a.ldy = N;
        const CUtensorMap ta = tmap_bytes(W, TG_BK, size_t(kblk) * rows128, TG_BK, TG_BM);
        const CUtensorMap tb = tmap_bytes(planes, K, size_t(3) * Tp, Kp, TG_BN);
        launch_limb_gemm(ta, tb, a, o.c.op_stream);
        uint32_t wide_h = 0;
        o.get(&wide_h, wide, 1);
        o.get(out, y, size_t(T) * N);
        if (wide_h)
            for (uint32_t t = 0; t < T; ++t) {
                const dimg_status s = dimg_op_dense(device, w, x + size_t(t) * K, out + size_t(t) * N);
                if (s != DIMG_OK) return s;
            }
    })
}

dimg_status dimg_op_rmsnorm(int device, const int64_t* x, const int64_t* g, uint32_t n, int64_t* out) {
    DIMG_API_GUARD({
        if (n == 0) fail(DIMG_EINVAL, "rmsnorm: empty vector");
        OpScope o(device);
        GemvArgs a = o.args();
        a.K = n;
        a.x = o.put(x, n);
        a.gamma = o.put(g, n);
        int64_t* d = o.mem.alloc<int64_t>(n);
        rmsnorm_op_kernel<<<1, 256, 0, o.c.op_stream>>>(a, d);
        CK(cudaGetLastError());
        o.get(out, d, n);
    })
}

dimg_status dimg_op_softmax(int device, const int64_t* s, uint32_t n, int64_t* out) {
    DIMG_API_GUARD({
        if (n == 0) fail(DIMG_EINVAL, "softmax_q16: empty input");
        OpScope o(device);
        int64_t* d = o.put(s, n);
        softmax_op_kernel<<<1, 256, 0, o.c.op_stream>>>(d, n, o.c.exp_lut);
        CK(cudaGetLastError());
        o.get(out, d, n);
    })
}

dimg_status dimg_op_attention(int device, uint32_t H, uint32_t dh, uint32_t max_ctx, double theta,
                              uint32_t steps, const int64_t* q, const int64_t* k, const int64_t* v,
                              int64_t* out) {
    // consecutive attention_step calls (proj/src/kernels.cpp:117-177)
    DIMG_API_GUARD({
        if (steps > max_ctx) fail(DIMG_ELENGTH, "attention_step: cache overflow");
        OpScope o(device);
        const size_t D = size_t(H) * dh;
        std::vector<int64_t> rc(size_t(max_ctx) * (dh / 2)), rs(rc.size());
        build_rope(theta, dh, max_ctx, rc.data(), rs.data());
        AttnArgs t{};
        t.rope_cos = o.put(rc.data(), rc.size());
        t.rope_sin = o.put(rs.data(), rs.size());
        int64_t* qkv = o.mem.alloc<int64_t>(3 * D);
        t.qkv = qkv;
        t.kc = o.mem.alloc<int64_t>(D * max_ctx);
        t.vc = o.mem.alloc<int64_t>(D * max_ctx);
        t.scores = o.mem.alloc<int64_t>(size_t(H) * max_ctx);
        int64_t* d_out = o.mem.alloc<int64_t>(D * steps);
        t.ctl = o.c.op_ctl;
        t.H = H; t.dh = dh; t.max_ctx = max_ctx;
        {
            int64_t x = int64_t(dh) * kOne;
            int b = 63 - __builtin_clzll(uint64_t(x));
            __int128 y = invsqrt_seed(b);
            for (int it = 0; it < 3; ++it) {
                __int128 tt = (y * y) >> 48;
                __int128 u = (__int128(x) * tt) >> 16;
                y = (y * ((__int128(3) << 48) - u)) >> 49;
            }
            t.inv_scale = int64_t((y + (__int128(1) << 31)) >> 32);
        }
        t.exp_lut = o.c.exp_lut;
        for (uint32_t p = 0; p < steps; ++p) {
            CK(cudaMemcpyAsync(qkv, q + p * D, D * 8, cudaMemcpyHostToDevice, o.c.op_stream));
            CK(cudaMemcpyAsync(qkv + D, k + p * D, D * 8, cudaMemcpyHostToDevice, o.c.op_stream));
            CK(cudaMemcpyAsync(qkv + 2 * D, v + p * D, D * 8, cudaMemcpyHostToDevice, o.c.op_stream));
            set_pos_kernel<<<1, 1, 0, o.c.op_stream>>>(o.c.op_ctl, p);
            t.out = d_out + p * D;
            attn_decode_kernel<<<H, ATTN_THREADS, attn_op_scratch_bytes(dh), o.c.op_stream>>>(t);
            CK(cudaGetLastError());
        }
        o.get(out, d_out, D * steps);
    })
}

dimg_status dimg_op_ffn(int device, const dimg_qtensor* gate, const dimg_qtensor* up,
                        const dimg_qtensor* down, const int64_t* x, int64_t* out) {
    // ffn_silu (proj/src/kernels.cpp:179-190): interleaved gate/up GEMV with
    // the silu*up epilogue, then the down GEMV
    DIMG_API_GUARD({
        if (gate->rows != up->rows || gate->cols != up->cols || down->cols != gate->rows)
            fail(DIMG_EINVAL, "ffn_silu: gate/up mismatch");
        OpScope o(device);
        const uint32_t F = gate->rows, D = gate->cols;
        GemvArgs a = o.args();
        int8_t* gu = o.put_padded(*gate, 2, 2 * F, 0);
        o.put_padded(*up, 2, 2 * F, 1, gu);
        std::vector<int64_t> gs(2 * size_t(F));
        for (uint32_t i = 0; i < F; ++i) {
            gs[2 * i] = gate->scales[i];
            gs[2 * i + 1] = up->scales[i];
        }
        a.W = gu; a.scales = o.put(gs.data(), gs.size());
        a.rows = 2 * F; a.K = D; a.Kp = pad16(D);
        a.x = o.put(x, D);
        int64_t* h = o.mem.alloc<int64_t>(F);
        a.y = h;
        launch_gemv<EPI_SILU, MODE_PLAIN>(a, o.c, o.c.op_stream);
        GemvArgs b = o.args();
        b.W = o.put_padded(*down, 1, down->rows, 0);
        b.scales = o.put(down->scales, down->rows);
        b.rows = down->rows; b.K = F; b.Kp = pad16(F);
        b.x = h;
        b.y = o.mem.alloc<int64_t>(down->rows);
        launch_gemv<EPI_STORE, MODE_PLAIN>(b, o.c, o.c.op_stream);
        CK(cudaGetLastError());
        o.get(out, b.y, down->rows);
    })
}

}  // extern "C"

#include "tp_engine.cuh"
