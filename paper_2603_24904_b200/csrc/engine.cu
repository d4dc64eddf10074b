// Device half of include/dimg.h: model upload (HBM layout), sessions (KV
// cache + control block), the per-token step as a CUDA graph, and the
// reference-shaped entry points generate_greedy / forward.
//
// One decode step (InferenceSession::forward + select_greedy,
// proj/src/engine.cpp:80-102,113-120) is 5L+1 kernels:
//   per layer: QKV GEMV (rmsnorm prologue; layer 0 also embeds the token)
//              -> attention step -> WO GEMV (+residual clamp)
//              -> GATE/UP GEMV (rmsnorm prologue, silu*up epilogue)
//              -> DOWN GEMV (+residual clamp)
//   head:      LM_HEAD GEMV (final rmsnorm prologue, argmax epilogue that
//              appends the next token on the device)
// The position and the token ring live in device memory, so the same
// instantiated graph is replayed for every token and nothing returns to the
// host until the caller asks for the tokens.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host/blake3.hpp"
#include "host/common.hpp"
#include "host/model.hpp"
#include "kernels/attention.cuh"
#include "kernels/gemv.cuh"

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
    Ctl* op_ctl = nullptr;  // control block for the operator-level exports
    cudaStream_t op_stream = nullptr;
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
    set_gemv_attrs<EPI_STORE, MODE_EMBED>();
    set_gemv_attrs<EPI_RESID, MODE_PLAIN>();
    set_gemv_attrs<EPI_SILU, MODE_NORM>();
    set_gemv_attrs<EPI_SILU, MODE_PLAIN>();
    set_gemv_attrs<EPI_ARGMAX, MODE_NORM>();
    set_gemv_attrs<EPI_RAW, MODE_PLAIN>();
    CK(cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            64 * 1024));
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

}  // namespace

// ---------------------------------------------------------------------------
// Model in HBM
// ---------------------------------------------------------------------------
struct dimg_model {
    int device;
    DevCtx* ctx;
    dimg_config cfg;
    uint32_t D, F, V, H, dh, L, Kd, Kf;
    int tp_rank, tp_size;
    struct Layer {
        int8_t* qkv;   // [3D][Kd]: wq rows, wk rows, wv rows
        int64_t* qkv_s;
        int8_t* wo;    // [D][Kd]
        int64_t* wo_s;
        int8_t* gu;    // [2F][Kd]: gate_i at row 2i, up_i at row 2i+1
        int64_t* gu_s;
        int8_t* down;  // [D][Kf]
        int64_t* down_s;
        int64_t* attn_norm;
        int64_t* ffn_norm;
    };
    std::vector<Layer> layers;
    int8_t* embd;      // [V][D] (gathered row by row, unpadded)
    int64_t* embd_s;
    int8_t* out_w;     // [V][Kd]
    int64_t* out_s;
    int64_t* final_norm;
    int64_t* rope_cos;
    int64_t* rope_sin;
    int64_t inv_scale;
    DevBuf mem;
};

namespace {

// Copies rows x cols int8 (row-major, pitch cols) into a device buffer with
// row pitch dpitch, starting at row offset `row0` with row stride `rstride`.
void put_rows(int8_t* dst, size_t dpitch, size_t row0, size_t rstride, const int8_t* src,
              uint32_t rows, uint32_t cols) {
    if (rows == 0) return;
    CK(cudaMemcpy2D(dst + row0 * dpitch, dpitch * rstride, src, cols, cols, rows,
                    cudaMemcpyHostToDevice));
}

template <class T>
T* upload(DevBuf& mem, const T* src, size_t n) {
    T* d = mem.alloc<T>(n);
    CK(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

}  // namespace

// ---------------------------------------------------------------------------
// Session: one sequence (KV cache, control block, token ring, graphs)
// ---------------------------------------------------------------------------
struct dimg_session {
    dimg_model* m;
    cudaStream_t stream = nullptr;
    DevBuf mem;
    int64_t *x, *qkv, *att, *h, *kc, *vc, *scores, *logits;
    ArgPart* parts;
    uint32_t* tokens;  // [max_ctx + 1]
    Ctl* ctl;
    uint32_t keep_cap = 0;
    uint32_t len = 0;              // host mirror of the cache length
    uint32_t n_prompt = 0, max_new = 0;
    uint32_t gemv_blocks = 0;
    cudaGraphExec_t g_prefill = nullptr, g_decode = nullptr;
    uint32_t launches_decode = 0, launches_prefill = 0;
    ~dimg_session() {
        if (g_prefill) cudaGraphExecDestroy(g_prefill);
        if (g_decode) cudaGraphExecDestroy(g_decode);
        if (stream) cudaStreamDestroy(stream);
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

GemvArgs base_args(const dimg_model& m, Ctl* ctl) {
    GemvArgs a{};
    a.ctl = ctl;
    a.exp_lut = m.ctx->exp_lut;
    a.seeds = m.ctx->seeds;
    return a;
}

void launch_qkv(dimg_session& s, uint32_t l) {
    const dimg_model& m = *s.m;
    const auto& lw = m.layers[l];
    GemvArgs a = base_args(m, s.ctl);
    a.W = lw.qkv; a.scales = lw.qkv_s; a.rows = 3 * m.D; a.K = m.D; a.Kp = m.Kd;
    a.x = s.x; a.gamma = lw.attn_norm; a.y = s.qkv;
    if (l == 0) {
        a.embd = m.embd; a.embd_scales = m.embd_s; a.tokens = s.tokens; a.x_out = s.x;
        launch_gemv<EPI_STORE, MODE_EMBED>(a, *m.ctx, s.stream);
    } else {
        launch_gemv<EPI_STORE, MODE_NORM>(a, *m.ctx, s.stream);
    }
}

void launch_attn(dimg_session& s, uint32_t l) {
    const dimg_model& m = *s.m;
    AttnArgs t{};
    t.qkv = s.qkv;
    t.kc = s.kc + size_t(l) * m.H * m.cfg.max_ctx * m.dh;
    t.vc = s.vc + size_t(l) * m.H * m.cfg.max_ctx * m.dh;
    t.rope_cos = m.rope_cos; t.rope_sin = m.rope_sin;
    t.scores = s.scores; t.out = s.att; t.ctl = s.ctl;
    t.H = m.H; t.dh = m.dh; t.max_ctx = m.cfg.max_ctx; t.inv_scale = m.inv_scale;
    t.exp_lut = m.ctx->exp_lut;
    attn_decode_kernel<<<m.H, ATTN_THREADS, m.dh * sizeof(int64_t), s.stream>>>(t);
}

void launch_wo(dimg_session& s, uint32_t l) {
    const dimg_model& m = *s.m;
    const auto& lw = m.layers[l];
    GemvArgs a = base_args(m, s.ctl);
    a.W = lw.wo; a.scales = lw.wo_s; a.rows = m.D; a.K = m.D; a.Kp = m.Kd;
    a.x = s.att; a.y = s.x;
    launch_gemv<EPI_RESID, MODE_PLAIN>(a, *m.ctx, s.stream);
}

void launch_gate_up(dimg_session& s, uint32_t l) {
    const dimg_model& m = *s.m;
    const auto& lw = m.layers[l];
    GemvArgs a = base_args(m, s.ctl);
    a.W = lw.gu; a.scales = lw.gu_s; a.rows = 2 * m.F; a.K = m.D; a.Kp = m.Kd;
    a.x = s.x; a.gamma = lw.ffn_norm; a.y = s.h;
    launch_gemv<EPI_SILU, MODE_NORM>(a, *m.ctx, s.stream);
}

void launch_down(dimg_session& s, uint32_t l) {
    const dimg_model& m = *s.m;
    const auto& lw = m.layers[l];
    GemvArgs a = base_args(m, s.ctl);
    a.W = lw.down; a.scales = lw.down_s; a.rows = m.D; a.K = m.F; a.Kp = m.Kf;
    a.x = s.h; a.y = s.x;
    launch_gemv<EPI_RESID, MODE_PLAIN>(a, *m.ctx, s.stream);
}

void launch_head(dimg_session& s) {
    const dimg_model& m = *s.m;
    GemvArgs a = base_args(m, s.ctl);
    a.W = m.out_w; a.scales = m.out_s; a.rows = m.V; a.K = m.D; a.Kp = m.Kd;
    a.x = s.x; a.gamma = m.final_norm; a.logits = s.logits; a.parts = s.parts;
    a.tokens_out = s.tokens;
    launch_gemv<EPI_ARGMAX, MODE_NORM>(a, *m.ctx, s.stream, s.gemv_blocks);
}

// Enqueues one forward step; `head` adds the lm_head + greedy selection,
// otherwise the position is just advanced (a prompt token whose logits the
// reference computes and discards, engine.cpp:40-42).
uint32_t enqueue_step(dimg_session& s, bool head) {
    const dimg_model& m = *s.m;
    for (uint32_t l = 0; l < m.L; ++l) {
        launch_qkv(s, l);
        launch_attn(s, l);
        launch_wo(s, l);
        launch_gate_up(s, l);
        launch_down(s, l);
    }
    if (head) launch_head(s);
    else advance_pos_kernel<<<1, 1, 0, s.stream>>>(s.ctl);
    CK(cudaGetLastError());
    return 5 * m.L + 1;
}

cudaGraphExec_t capture(dimg_session& s, bool head, uint32_t* launches) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal));
    try {
        *launches = enqueue_step(s, head);
    } catch (...) {
        cudaStreamEndCapture(s.stream, &g);
        throw;
    }
    CK(cudaStreamEndCapture(s.stream, &g));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    return ex;
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
    if (err & 1u) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
}

void ensure_keep(dimg_session& s, uint32_t need) {
    if (need <= s.keep_cap) return;
    CK(cudaStreamSynchronize(s.stream));
    void* p = nullptr;
    CK(cudaMalloc(&p, size_t(need + 1) * s.m->V * sizeof(int64_t)));
    s.mem.ptrs.push_back(p);
    s.logits = static_cast<int64_t*>(p);
    s.keep_cap = need;
    // the decode graph bakes the logits pointer in: recapture
    if (s.g_decode) CK(cudaGraphExecDestroy(s.g_decode));
    s.g_decode = capture(s, true, &s.launches_decode);
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

void run_prefill(dimg_session& s) {
    for (uint32_t i = 0; i + 1 < s.n_prompt; ++i) CK(cudaGraphLaunch(s.g_prefill, s.stream));
    s.len = s.n_prompt - 1;
}

void run_decode(dimg_session& s, uint32_t steps) {
    for (uint32_t i = 0; i < steps; ++i) CK(cudaGraphLaunch(s.g_decode, s.stream));
    s.len += steps;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

dimg_status dimg_device_count(int* n) { DIMG_API_GUARD(CK(cudaGetDeviceCount(n))) }

dimg_status dimg_model_upload(int device, const dimg_model_desc* d, int tp_rank, int tp_size,
                              dimg_model** out) {
    DIMG_API_GUARD({
        validate_config(d->cfg);
        if (tp_size != 1 || tp_rank != 0)
            fail(DIMG_EINVAL, "model_upload: tensor-parallel sharding is not built yet");
        DevCtx& c = dev_ctx(device);
        CK(cudaSetDevice(device));
        auto m = std::make_unique<dimg_model>();
        m->device = device;
        m->ctx = &c;
        m->cfg = d->cfg;
        m->D = d->cfg.d_model; m->F = d->cfg.d_ffn; m->V = d->cfg.vocab; m->H = d->cfg.n_heads;
        m->dh = m->D / m->H; m->L = d->cfg.n_layers; m->Kd = pad16(m->D); m->Kf = pad16(m->F);
        m->tp_rank = tp_rank; m->tp_size = tp_size;
        if (size_t(8) * std::max(m->Kd, m->Kf) > 200 * 1024)
            fail(DIMG_EINVAL, "model_upload: d_ffn above 25600 needs the tiled-limb GEMV (not built)");
        if (size_t(m->dh) * 8 > 64 * 1024) fail(DIMG_EINVAL, "model_upload: d_head above 8192");
        const uint32_t D = m->D, F = m->F, V = m->V;
        auto check_qt = [&](const dimg_qtensor& t, uint32_t r, uint32_t k, const char* what) {
            if (t.rows != r || t.cols != k) fail(DIMG_EINVAL, std::string("model_upload: bad shape of ") + what);
        };
        m->layers.resize(m->L);
        for (uint32_t l = 0; l < m->L; ++l) {
            const dimg_qtensor* t = d->layers + 7 * size_t(l);
            const char* names[7] = {"wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"};
            for (int i = 0; i < 7; ++i)
                check_qt(t[i], i < 4 ? D : (i < 6 ? F : D), i < 6 ? D : F, names[i]);
            auto& lw = m->layers[l];
            lw.qkv = m->mem.alloc<int8_t>(size_t(3) * D * m->Kd);
            CK(cudaMemset(lw.qkv, 0, size_t(3) * D * m->Kd));
            for (int i = 0; i < 3; ++i) put_rows(lw.qkv, m->Kd, size_t(i) * D, 1, t[i].data, D, D);
            std::vector<int64_t> s(3 * size_t(D));
            for (int i = 0; i < 3; ++i) std::copy(t[i].scales, t[i].scales + D, s.begin() + i * D);
            lw.qkv_s = upload(m->mem, s.data(), s.size());
            lw.wo = m->mem.alloc<int8_t>(size_t(D) * m->Kd);
            CK(cudaMemset(lw.wo, 0, size_t(D) * m->Kd));
            put_rows(lw.wo, m->Kd, 0, 1, t[3].data, D, D);
            lw.wo_s = upload(m->mem, t[3].scales, D);
            lw.gu = m->mem.alloc<int8_t>(size_t(2) * F * m->Kd);
            CK(cudaMemset(lw.gu, 0, size_t(2) * F * m->Kd));
            put_rows(lw.gu, m->Kd, 0, 2, t[4].data, F, D);
            put_rows(lw.gu, m->Kd, 1, 2, t[5].data, F, D);
            std::vector<int64_t> gs(2 * size_t(F));
            for (uint32_t i = 0; i < F; ++i) {
                gs[2 * i] = t[4].scales[i];
                gs[2 * i + 1] = t[5].scales[i];
            }
            lw.gu_s = upload(m->mem, gs.data(), gs.size());
            lw.down = m->mem.alloc<int8_t>(size_t(D) * m->Kf);
            CK(cudaMemset(lw.down, 0, size_t(D) * m->Kf));
            put_rows(lw.down, m->Kf, 0, 1, t[6].data, D, F);
            lw.down_s = upload(m->mem, t[6].scales, D);
            lw.attn_norm = upload(m->mem, d->norms + size_t(2 * l) * D, D);
            lw.ffn_norm = upload(m->mem, d->norms + size_t(2 * l + 1) * D, D);
        }
        check_qt(d->tok_embd, V, D, "tok_embd");
        check_qt(d->output, V, D, "output");
        m->embd = upload(m->mem, d->tok_embd.data, size_t(V) * D);
        m->embd_s = upload(m->mem, d->tok_embd.scales, V);
        m->out_w = m->mem.alloc<int8_t>(size_t(V) * m->Kd);
        CK(cudaMemset(m->out_w, 0, size_t(V) * m->Kd));
        put_rows(m->out_w, m->Kd, 0, 1, d->output.data, V, D);
        m->out_s = upload(m->mem, d->output.scales, V);
        m->final_norm = upload(m->mem, d->norms + size_t(2 * m->L) * D, D);
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
        *out = m.release();
    })
}

dimg_status dimg_model_free(dimg_model* m) {
    DIMG_API_GUARD({
        if (m) {
            cudaSetDevice(m->device);
            delete m;
        }
    })
}

dimg_status dimg_model_bytes_on_device(const dimg_model* m, uint64_t* bytes) {
    DIMG_API_GUARD(*bytes = m->mem.bytes)
}

dimg_status dimg_session_create(dimg_model* m, uint32_t keep_logits_cap, dimg_session** out) {
    DIMG_API_GUARD({
        CK(cudaSetDevice(m->device));
        auto s = std::make_unique<dimg_session>();
        s->m = m;
        CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        const size_t ctx = m->cfg.max_ctx;
        s->x = s->mem.alloc<int64_t>(m->D);
        s->qkv = s->mem.alloc<int64_t>(3 * size_t(m->D));
        s->att = s->mem.alloc<int64_t>(m->D);
        s->h = s->mem.alloc<int64_t>(m->F);
        size_t kv = size_t(m->L) * m->H * ctx * m->dh;
        s->kc = s->mem.alloc<int64_t>(kv);
        s->vc = s->mem.alloc<int64_t>(kv);
        s->scores = s->mem.alloc<int64_t>(size_t(m->H) * ctx);
        s->keep_cap = keep_logits_cap;
        s->logits = s->mem.alloc<int64_t>(size_t(keep_logits_cap + 1) * m->V);
        s->gemv_blocks = gemv_grid(*m->ctx, m->V, 1);
        s->parts = s->mem.alloc<ArgPart>(s->gemv_blocks);
        s->tokens = s->mem.alloc<uint32_t>(ctx + 1);
        s->ctl = s->mem.alloc<Ctl>(1);
        CK(cudaMemsetAsync(s->ctl, 0, sizeof(Ctl), s->stream));
        CK(cudaMemsetAsync(s->tokens, 0, (ctx + 1) * 4, s->stream));
        s->g_prefill = capture(*s, false, &s->launches_prefill);
        s->g_decode = capture(*s, true, &s->launches_decode);
        CK(cudaStreamSynchronize(s->stream));
        *out = s.release();
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
        // keep slot 0 for this position's logits; the head appends the argmax
        // at tokens[pos + 1], which the next forward overwrites
        write_ctl(*s, pos, pos, 1 <= s->keep_cap ? 1 : 0);
        CK(cudaGraphLaunch(s->g_decode, s->stream));
        s->len = pos + 1;
        if (logits)  // slot 0 (kept) or row 0 = scratch when keep_cap == 0
            CK(cudaMemcpyAsync(logits, s->logits, size_t(m.V) * 8, cudaMemcpyDeviceToHost, s->stream));
        check_ctl_err(*s);
    })
}

dimg_status dimg_generate_greedy(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt,
                                 uint32_t max_new, uint32_t* tokens_out, uint8_t hash_out[32],
                                 int64_t* logits_out) {
    // run_generation (proj/src/engine.cpp:31-54): P + N - 1 forwards, the
    // lm_head only where a selection follows.
    DIMG_API_GUARD({
        begin(*s, prompt, n_prompt, max_new, logits_out != nullptr);
        if (max_new > 0) {
            run_prefill(*s);
            run_decode(*s, max_new);
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
    })
}

dimg_status dimg_session_time_kernel(dimg_session* s, int which, uint32_t n, float* ms_per_launch,
                                    uint64_t* bytes_per_launch) {
    // Replays one kernel class n times (cycling layers so weights come from
    // HBM, not L2) between CUDA events on the session stream. Algorithmic
    // bytes = int8 weights + int64 scales + int64 gains + activation I/O.
    DIMG_API_GUARD({
        const dimg_model& m = *s->m;
        CK(cudaSetDevice(m.device));
        const uint64_t D = m.D, F = m.F, V = m.V;
        uint64_t bytes = 0;
        switch (which) {
            case 0: bytes = 3 * D * D + 3 * D * 8 + D * 8 + D * 8 + 3 * D * 8; break;   // qkv
            case 1: bytes = D * D + D * 8 + D * 8 + 2 * D * 8; break;                   // wo
            case 2: bytes = 2 * F * D + 2 * F * 8 + D * 8 + D * 8 + F * 8; break;       // gate/up
            case 3: bytes = D * F + D * 8 + F * 8 + 2 * D * 8; break;                   // down
            case 4: bytes = V * D + V * 8 + D * 8 + D * 8; break;                       // lm_head
            default: fail(DIMG_EINVAL, "time_kernel: which in 0..4");
        }
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(s->stream));
        // the head's argmax appends tokens: keep pos fixed by restoring it after
        uint32_t pos_save = 0;
        CK(cudaMemcpy(&pos_save, &s->ctl->pos, 4, cudaMemcpyDeviceToHost));
        CK(cudaEventRecord(e0, s->stream));
        for (uint32_t i = 0; i < n; ++i) {
            uint32_t l = i % m.L;
            if (which == 0) launch_qkv(*s, l);
            else if (which == 1) launch_wo(*s, l);
            else if (which == 2) launch_gate_up(*s, l);
            else if (which == 3) launch_down(*s, l);
            else launch_head(*s);
        }
        CK(cudaEventRecord(e1, s->stream));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        CK(cudaMemcpy(&s->ctl->pos, &pos_save, 4, cudaMemcpyHostToDevice));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_per_launch = ms / float(n);
        *bytes_per_launch = bytes;
    })
}

dimg_status dimg_session_launches(const dimg_session* s, uint32_t* per_decode, uint32_t* per_prefill) {
    DIMG_API_GUARD({
        *per_decode = s->launches_decode;
        *per_prefill = s->launches_prefill;
    })
}

dimg_status dimg_session_stats(dimg_session* s, uint64_t out[4]) {
    DIMG_API_GUARD({
        Ctl c;
        CK(cudaMemcpyAsync(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        out[0] = c.stats[0];
        out[1] = c.err;
        out[2] = c.stats[2];
        out[3] = c.stats[3];
    })
}

}  // extern "C"

// ---- operator-level exports ------------------------------------------------
// Each runs the engine's own device code on host buffers (upload, one launch,
// download) so proj/src/kernels.cpp's operators can be checked one by one.

namespace {

struct OpScope {
    DevCtx& c;
    DevBuf mem;
    explicit OpScope(int device) : c(dev_ctx(device)) {
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
        CK(cudaStreamSynchronize(c.op_stream));
        put_rows(dst, Kp, row0, row_stride, w.data, w.rows, w.cols);
        return dst;
    }
    template <class T>
    void get(T* dst, const T* src, size_t n) {
        CK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, c.op_stream));
        CK(cudaStreamSynchronize(c.op_stream));
        uint32_t err = 0;
        CK(cudaMemcpy(&err, &c.op_ctl->err, 4, cudaMemcpyDeviceToHost));
        if (err & 1u) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
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
            attn_decode_kernel<<<H, ATTN_THREADS, dh * 8, o.c.op_stream>>>(t);
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
