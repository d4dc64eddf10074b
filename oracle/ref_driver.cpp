// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-linkage shim over the UNMODIFIED reference library (the sources under
// /root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libdimref.so). It lets Python tests, the golden-vector script
// and bench.py's cpu_baseline / --impl reference legs drive the reference's
// own public API (dim::generate_greedy, dim::InferenceSession, the kernels in
// proj/include/dim/kernels.hpp) without its CLI. Nothing here reimplements
// reference behaviour; it only marshals plain buffers into dim:: types.
#include <array>
#include <cstdint>
#include <cstdio>
#include <string>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "dim/attest.hpp"
#include "dim/blake3.hpp"
#include "dim/chacha20.hpp"
#include "dim/engine.hpp"
#include "dim/kernels.hpp"
#include "dim/model.hpp"
#include "dim/q16.hpp"
#include "dim/rope.hpp"
#include "dim/serial.hpp"

using namespace dim;

namespace {

// Exceptions -> codes (the same mapping the B200 C ABI uses, include/dimg.h).
int code_of(const std::exception& e) {
    if (dynamic_cast<const ContextOverflow*>(&e)) return 4;
    if (dynamic_cast<const ParseError*>(&e)) return 7;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
    if (dynamic_cast<const std::length_error*>(&e)) return 5;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 6;  // DIMG_EDOMAIN
    if (dynamic_cast<const std::logic_error*>(&e)) return 3;
    return 99;
}

#define GUARD(...)                                    \
    try {                                             \
        __VA_ARGS__;                                  \
        return 0;                                     \
    } catch (const std::exception& e) {               \
        return code_of(e);                            \
    }

ModelConfig make_cfg(const uint32_t* c, double theta) {
    ModelConfig cfg;
    cfg.n_layers = c[0];
    cfg.d_model = c[1];
    cfg.n_heads = c[2];
    cfg.d_ffn = c[3];
    cfg.vocab = c[4];
    cfg.max_ctx = c[5];
    cfg.rope_theta = theta;
    return cfg;
}

std::vector<QuantTensor*> quant_order(ModelFile& m) {
    std::vector<QuantTensor*> v{&m.tok_embd};
    for (auto& l : m.layers) {
        for (QuantTensor* t : {&l.wq, &l.wk, &l.wv, &l.wo, &l.w_gate, &l.w_up, &l.w_down})
            v.push_back(t);
    }
    v.push_back(&m.output);
    return v;
}

std::vector<std::vector<q16>*> norm_order(ModelFile& m) {
    std::vector<std::vector<q16>*> v;
    for (auto& l : m.layers) {
        v.push_back(&l.attn_norm);
        v.push_back(&l.ffn_norm);
    }
    v.push_back(&m.final_norm);
    return v;
}

QuantTensor make_qt(uint32_t rows, uint32_t cols, const int8_t* data, const int64_t* scales) {
    QuantTensor t;
    t.rows = rows;
    t.cols = cols;
    t.data.assign(data, data + size_t(rows) * cols);
    t.scales.assign(scales, scales + rows);
    return t;
}

std::vector<q16> to_q16(const int64_t* x, size_t n) {
    std::vector<q16> v(n);
    for (size_t i = 0; i < n; ++i) v[i].raw = x[i];
    return v;
}

} // namespace

extern "C" {

// ---- primitives ---------------------------------------------------------
void ref_blake3(const void* data, size_t len, uint8_t out[32]) {
    Digest d = blake3(data, len);
    std::memcpy(out, d.bytes.data(), 32);
}
void ref_exp_lut(int64_t out[257]) {
    const auto& e = ExpLut::instance().entries;
    for (int i = 0; i < 257; ++i) out[i] = e[i];
}
int ref_inv_sqrt(int64_t x, int64_t* out) { GUARD(*out = inv_sqrt_q16(q16{x}).raw) }
int ref_exp_neg(int64_t t, int64_t* out) { GUARD(*out = exp_neg_lut(q16{t}).raw) }
int64_t ref_sigmoid(int64_t x) { return sigmoid_q16(q16{x}).raw; }
int64_t ref_silu(int64_t x) { return silu_q16(q16{x}).raw; }
int ref_q16_from_ratio(int64_t n, int64_t d, int64_t* out) { GUARD(*out = q16_from_ratio(n, d).raw) }
int ref_rope_tables(double theta, uint32_t dh, uint32_t ctx, int64_t* cos_out, int64_t* sin_out) {
    GUARD({
        RopeTables t = build_rope_tables(theta, dh, ctx);
        std::memcpy(cos_out, t.cos_raw.data(), t.cos_raw.size() * 8);
        std::memcpy(sin_out, t.sin_raw.data(), t.sin_raw.size() * 8);
    })
}
void ref_chacha_stream(uint64_t seed, uint8_t* out, size_t n) {
    ChaCha20Rng r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.next_u8();
}
void ref_prompt(uint64_t seed, uint32_t vocab, uint32_t n, uint32_t* out) {
    // prompt[i] = ChaCha20Rng(seed).next_u32() % V (proj/tests/acceptance.cpp:80-82)
    ChaCha20Rng r(seed);
    for (uint32_t i = 0; i < n; ++i) out[i] = r.next_u32() % vocab;
}

// ---- operators (proj/src/kernels.cpp) ------------------------------------
int ref_dense(uint32_t rows, uint32_t cols, const int8_t* w, const int64_t* s, const int64_t* x,
              size_t chunk, int64_t* out) {
    GUARD({
        QuantTensor t = make_qt(rows, cols, w, s);
        auto y = dense_dispatch(t, to_q16(x, cols), chunk);
        for (uint32_t r = 0; r < rows; ++r) out[r] = y[r].raw;
    })
}
int ref_rmsnorm(const int64_t* x, const int64_t* g, uint32_t n, int64_t* out) {
    GUARD({
        auto y = rmsnorm(to_q16(x, n), to_q16(g, n));
        for (uint32_t i = 0; i < n; ++i) out[i] = y[i].raw;
    })
}
int ref_softmax(const int64_t* s, uint32_t n, int64_t* out) {
    GUARD({
        auto y = softmax_q16(to_q16(s, n));
        for (uint32_t i = 0; i < n; ++i) out[i] = y[i].raw;
    })
}
// Runs `steps` consecutive attention_step calls (pos 0..steps-1) on one fresh
// LayerKv; q/k/v are [steps][H*dh]; out receives every step's output.
int ref_attention(uint32_t H, uint32_t dh, uint32_t max_ctx, double theta, uint32_t steps,
                  const int64_t* q, const int64_t* k, const int64_t* v, int threads,
                  int64_t* out) {
    GUARD({
        RopeTables tabs = build_rope_tables(theta, dh, max_ctx);
        LayerKv cache(H, dh, max_ctx);
        size_t D = size_t(H) * dh;
        for (uint32_t t = 0; t < steps; ++t) {
            auto y = attention_step(to_q16(q + t * D, D), to_q16(k + t * D, D),
                                    to_q16(v + t * D, D), cache, t, tabs, threads);
            for (size_t i = 0; i < D; ++i) out[t * D + i] = y[i].raw;
        }
    })
}
int ref_ffn(uint32_t d, uint32_t f, const int8_t* wg, const int64_t* sg, const int8_t* wu,
            const int64_t* su, const int8_t* wd, const int64_t* sd, const int64_t* x,
            int64_t* out) {
    GUARD({
        QuantTensor g = make_qt(f, d, wg, sg), u = make_qt(f, d, wu, su), dn = make_qt(d, f, wd, sd);
        auto y = ffn_silu(to_q16(x, d), g, u, dn);
        for (uint32_t i = 0; i < d; ++i) out[i] = y[i].raw;
    })
}

// ---- model ----------------------------------------------------------------
// cfg = {n_layers, d_model, n_heads, d_ffn, vocab, max_ctx}
int ref_gen_toy_model(uint64_t seed, const uint32_t* cfg, double theta, void** out) {
    GUARD(*out = new ModelFile(gen_toy_model(seed, make_cfg(cfg, theta))))
}
// Builds a ModelFile straight from directory-order buffers (the bench's fast
// path: the reference's own generator costs 83 s at 7B). bytes/weight_hash
// are left empty; the forward pass never reads them.
int ref_model_from_arrays(const uint32_t* cfg, double theta, const int8_t* weights,
                          const int64_t* scales, const int64_t* norms, void** out) {
    GUARD({
        auto* m = new ModelFile();
        m->config = make_cfg(cfg, theta);
        m->config.validate();
        m->layers.resize(m->config.n_layers);
        const uint32_t D = m->config.d_model, F = m->config.d_ffn, V = m->config.vocab;
        size_t wo = 0, so = 0, i = 0;
        for (QuantTensor* t : quant_order(*m)) {
            uint32_t rows, cols;
            if (i == 0 || t == &m->output) { rows = V; cols = D; }
            else {
                int k = int((i - 1) % 7);
                rows = k < 4 ? D : (k < 6 ? F : D);
                cols = k < 6 ? D : F;
            }
            *t = make_qt(rows, cols, weights + wo, scales + so);
            wo += size_t(rows) * cols;
            so += rows;
            ++i;
        }
        size_t no = 0;
        for (auto* n : norm_order(*m)) {
            *n = to_q16(norms + no, D);
            no += D;
        }
        *out = m;
    })
}
int ref_deserialize(const uint8_t* bytes, size_t n, void** out) {
    GUARD(*out = new ModelFile(deserialize(std::span<const uint8_t>(bytes, n))))
}
void ref_model_free(void* m) { delete static_cast<ModelFile*>(m); }
void ref_model_weight_hash(void* m, uint8_t out[32]) {
    std::memcpy(out, static_cast<ModelFile*>(m)->weight_hash.bytes.data(), 32);
}
size_t ref_model_bytes(void* m, uint8_t* out) {
    auto& b = static_cast<ModelFile*>(m)->bytes;
    if (out) std::memcpy(out, b.data(), b.size());
    return b.size();
}
// Copies weights/scales/norms out in directory order.
void ref_model_export(void* mp, int8_t* weights, int64_t* scales, int64_t* norms) {
    auto& m = *static_cast<ModelFile*>(mp);
    size_t wo = 0, so = 0, no = 0;
    for (QuantTensor* t : quant_order(m)) {
        std::memcpy(weights + wo, t->data.data(), t->data.size());
        std::memcpy(scales + so, t->scales.data(), t->scales.size() * 8);
        wo += t->data.size();
        so += t->scales.size();
    }
    for (auto* n : norm_order(m)) {
        for (auto& v : *n) norms[no++] = v.raw;
    }
}

// ---- engine (proj/src/engine.cpp) -----------------------------------------
int ref_generate_greedy(void* m, const uint32_t* prompt, uint32_t p, uint32_t n, int threads,
                        size_t chunk, uint32_t* tokens_out, uint8_t hash_out[32],
                        int64_t* logits_out) {
    GUARD({
        EngineOptions o;
        o.threads = threads;
        o.chunk = chunk;
        o.keep_logits = logits_out != nullptr;
        auto r = generate_greedy(*static_cast<ModelFile*>(m),
                                 std::span<const uint32_t>(prompt, p), n, o);
        for (size_t i = 0; i < r.token_ids.size(); ++i) tokens_out[i] = r.token_ids[i];
        std::memcpy(hash_out, r.output_hash.bytes.data(), 32);
        if (logits_out) {
            size_t V = static_cast<ModelFile*>(m)->config.vocab;
            for (size_t i = 0; i < r.logits.size(); ++i)
                for (size_t j = 0; j < V; ++j) logits_out[i * V + j] = r.logits[i][j].raw;
        }
    })
}
int ref_session_new(void* m, int threads, void** out) {
    GUARD({
        EngineOptions o;
        o.threads = threads;
        *out = new InferenceSession(*static_cast<ModelFile*>(m), o);
    })
}
void ref_session_free(void* s) { delete static_cast<InferenceSession*>(s); }
int ref_session_forward(void* s, uint32_t token, uint32_t pos, int64_t* logits, uint32_t* argmax) {
    GUARD({
        auto y = static_cast<InferenceSession*>(s)->forward(token, pos);
        if (logits)
            for (size_t i = 0; i < y.size(); ++i) logits[i] = y[i].raw;
        if (argmax) *argmax = select_greedy(y);
    })
}
uint64_t ref_generation_counter() { return generation_counter().load(); }
// generate_sampled (proj/src/engine.cpp:148-163) with the per-step logits
int ref_generate_sampled(void* m, const uint32_t* prompt, uint32_t p, uint32_t n, int64_t temperature,
                         uint32_t* tokens_out, uint8_t hash_out[32], int64_t* logits_out) {
    GUARD({
        EngineOptions o;
        o.keep_logits = logits_out != nullptr;
        auto r = generate_sampled(*static_cast<ModelFile*>(m), std::span<const uint32_t>(prompt, p), n,
                                  q16{temperature}, o);
        for (size_t i = 0; i < r.token_ids.size(); ++i) tokens_out[i] = r.token_ids[i];
        std::memcpy(hash_out, r.output_hash.bytes.data(), 32);
        if (logits_out) {
            size_t V = static_cast<ModelFile*>(m)->config.vocab;
            for (size_t i = 0; i < r.logits.size(); ++i)
                for (size_t j = 0; j < V; ++j) logits_out[i * V + j] = r.logits[i][j].raw;
        }
    })
}

// sample_from_logits (proj/src/engine.cpp:122-139) of one row, the draw being
// the first u32 of ChaCha20Rng(key) (the caller recomputes it)
int ref_sample_from_logits(const int64_t* logits, uint32_t V, int64_t temperature, const uint8_t key[32],
                           uint32_t* out) {
    GUARD({
        std::vector<q16> row(V);
        for (uint32_t i = 0; i < V; ++i) row[i].raw = logits[i];
        std::array<uint8_t, 32> k;
        std::memcpy(k.data(), key, 32);
        ChaCha20Rng rng(k);
        *out = sample_from_logits(std::span<const q16>(row.data(), row.size()), q16{temperature}, rng);
    })
}

// RTAB codec (proj/src/rope.cpp:41-93): the reference's bytes for built
// tables, and the ParseError kind (or 0) of deserializing arbitrary bytes
int ref_rtab_serialize(double theta, uint32_t dh, uint32_t ctx, uint8_t* out, size_t cap, size_t* n) {
    GUARD({
        const auto b = serialize_rope_tables(build_rope_tables(theta, dh, ctx));
        *n = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    })
}
int ref_rtab_parse(const uint8_t* bytes, size_t n, int* kind) {
    *kind = -1;
    try {
        (void)deserialize_rope_tables(std::span<const uint8_t>(bytes, n));
        return 0;
    } catch (const ParseError& e) {
        *kind = int(e.kind);
        return 7;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// ---- attestation (proj/src/attest.cpp) ----------------------------------------
// make_attestation of a fresh greedy generation: wire bytes + to_text
int ref_attestation(void* m, const uint32_t* prompt, uint32_t p, uint32_t n, uint64_t bond, uint64_t period,
                    uint8_t wire[112], char* text, size_t cap) {
    GUARD({
        auto& mf = *static_cast<ModelFile*>(m);
        const std::span<const uint32_t> pr(prompt, p);
        const auto a = make_attestation(mf.bytes, pr, generate_greedy(mf, pr, n), bond, period);
        const auto w = a.encode();
        std::memcpy(wire, w.data(), 112);
        const std::string t = a.to_text();
        std::snprintf(text, cap, "%s", t.c_str());
    })
}
// verify_by_reexecution of wire bytes: the outcome's to_text
int ref_verify(const uint8_t* wire, void* m, const uint32_t* prompt, uint32_t p, uint32_t n, char* text,
               size_t cap) {
    GUARD({
        auto& mf = *static_cast<ModelFile*>(m);
        const auto a = Attestation::decode(std::span<const uint8_t>(wire, 112));
        const auto o = verify_by_reexecution(a, mf.bytes, std::span<const uint32_t>(prompt, p), n);
        std::snprintf(text, cap, "%s", o.to_text().c_str());
    })
}

} // extern "C"
