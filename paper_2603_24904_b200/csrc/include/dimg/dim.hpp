// dim.hpp -- the reference's C++ engine API (proj/include/dim/{engine,model}.hpp)
// re-expressed over the B200 C ABI (include/dimg.h). Header-only: link
// libdimg.so. Same names, argument meaning and exception types as dim::, so a
// caller of dim::generate_greedy / dim::InferenceSession switches by changing
// the namespace. Every forward pass runs on the GPU; there is no CPU path.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dimg.h"

namespace dimg {

// ---- exceptions (proj/include/dim/engine.hpp:16-18, serial.hpp:10-15) -------
struct ContextOverflow : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    enum class Kind { bad_magic, bad_version, truncated, invariant };
    ParseError(Kind k, const std::string& w) : std::runtime_error(w), kind(k) {}
    Kind kind;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(dimg_status s) {
    if (s == DIMG_OK) return;
    const std::string msg = dimg_last_error();
    switch (s) {
        case DIMG_EINVAL: throw std::invalid_argument(msg);
        case DIMG_ERANGE: throw std::out_of_range(msg);
        case DIMG_ELOGIC: throw std::logic_error(msg);
        case DIMG_ECTX: throw ContextOverflow(msg);
        case DIMG_ELENGTH: throw std::length_error(msg);
        case DIMG_EDOMAIN: throw std::domain_error(msg);
        case DIMG_EPARSE: throw ParseError(ParseError::Kind(dimg_last_parse_kind()), msg);
        case DIMG_ENOMEM: throw std::bad_alloc();
        default: throw CudaError(msg);
    }
}

// ---- values ------------------------------------------------------------------
struct Digest {
    std::array<uint8_t, 32> bytes{};
    std::string hex() const {
        static const char* k = "0123456789abcdef";
        std::string s;
        for (uint8_t b : bytes) {
            s.push_back(k[b >> 4]);
            s.push_back(k[b & 15]);
        }
        return s;
    }
    friend bool operator==(const Digest&, const Digest&) = default;
};

struct ModelConfig {  // proj/include/dim/model.hpp:15-29
    uint32_t n_layers = 0, d_model = 0, n_heads = 0, d_ffn = 0, vocab = 0, max_ctx = 0;
    double rope_theta = 10000.0;
    uint32_t d_head() const { return d_model / n_heads; }
    dimg_config c() const { return {n_layers, d_model, n_heads, d_ffn, vocab, max_ctx, rope_theta}; }
    void validate() const {
        dimg_config cc = c();
        check(dimg_config_validate(&cc));
    }
};

struct EngineOptions {  // proj/include/dim/engine.hpp:20-24 (+ device)
    int threads = 1;    // head-thread pool in the reference; output-invariant, ignored here
    size_t chunk = 0;   // chunked matvec in the reference; output-invariant, ignored here
    bool keep_logits = false;
    int device = 0;
};

struct GenerationResult {  // proj/include/dim/engine.hpp:26-30
    std::vector<uint32_t> token_ids;
    Digest output_hash;
    std::vector<std::vector<int64_t>> logits;
};

// ---- model ---------------------------------------------------------------------
class ModelFile {  // proj/include/dim/model.hpp:50-60
  public:
    static ModelFile gen_toy(uint64_t seed, const ModelConfig& cfg, int threads = 0) {
        dimg_config c = cfg.c();
        dimg_host_model* h = nullptr;
        check(dimg_host_model_gen_toy(seed, &c, threads, &h));
        return ModelFile(h);
    }
    static ModelFile deserialize(std::span<const uint8_t> bytes) {
        dimg_host_model* h = nullptr;
        check(dimg_host_model_from_bytes(bytes.data(), bytes.size(), &h));
        return ModelFile(h);
    }
    static ModelFile load(const std::string& path) {
        dimg_host_model* h = nullptr;
        check(dimg_host_model_load(path.c_str(), &h));
        return ModelFile(h);
    }
    void save(const std::string& path) const { check(dimg_host_model_save(h_.get(), path.c_str())); }

    std::span<const uint8_t> bytes() const {
        const uint8_t* p = nullptr;
        size_t n = 0;
        check(dimg_host_model_bytes(h_.get(), &p, &n));
        return {p, n};
    }
    Digest weight_hash() const {
        Digest d;
        check(dimg_host_model_weight_hash(h_.get(), d.bytes.data()));
        return d;
    }
    ModelConfig config() const {
        dimg_model_desc d;
        check(dimg_host_model_desc(h_.get(), &d));
        return {d.cfg.n_layers, d.cfg.d_model, d.cfg.n_heads, d.cfg.d_ffn, d.cfg.vocab, d.cfg.max_ctx,
                d.cfg.rope_theta};
    }
    // The model re-laid out in one GPU's HBM, uploaded on first use.
    dimg_model* device_model(int device) const {
        auto& slot = (*devs_)[device];
        if (!slot) {
            dimg_model_desc d;
            check(dimg_host_model_desc(h_.get(), &d));
            dimg_model* m = nullptr;
            check(dimg_model_upload(device, &d, 0, 1, &m));
            slot = std::shared_ptr<dimg_model>(m, [](dimg_model* p) { dimg_model_free(p); });
        }
        return slot.get();
    }

  private:
    explicit ModelFile(dimg_host_model* h)
        : h_(h, [](dimg_host_model* p) { dimg_host_model_free(p); }),
          devs_(std::make_shared<std::map<int, std::shared_ptr<dimg_model>>>()) {}
    std::shared_ptr<dimg_host_model> h_;
    std::shared_ptr<std::map<int, std::shared_ptr<dimg_model>>> devs_;
};

inline ModelFile gen_toy_model(uint64_t seed, const ModelConfig& cfg) { return ModelFile::gen_toy(seed, cfg); }
inline ModelFile load_model(const std::string& path) { return ModelFile::load(path); }
inline ModelFile deserialize(std::span<const uint8_t> b) { return ModelFile::deserialize(b); }

// ---- engine --------------------------------------------------------------------
inline Digest hash_token_ids(std::span<const uint32_t> ids) {  // engine.cpp:104-111
    Digest d;
    check(dimg_hash_token_ids(ids.data(), ids.size(), d.bytes.data()));
    return d;
}

// ---- RoPE tables and the RTAB artifact (proj/include/dim/rope.hpp:15-39) -----
struct RopeTables {
    uint32_t max_ctx = 0;
    uint32_t half_dim = 0;
    double theta_base = 10000.0;
    std::vector<int64_t> cos_raw;  // max_ctx * half_dim, row-major
    std::vector<int64_t> sin_raw;
    int64_t cos_at(uint32_t pos, uint32_t k) const { return cos_raw[size_t(pos) * half_dim + k]; }
    int64_t sin_at(uint32_t pos, uint32_t k) const { return sin_raw[size_t(pos) * half_dim + k]; }
    friend bool operator==(const RopeTables&, const RopeTables&) = default;
};

inline RopeTables build_rope_tables(double theta_base, uint32_t d_head, uint32_t max_ctx) {  // rope.cpp:17-39
    if (d_head == 0 || d_head % 2 != 0) throw std::invalid_argument("rope: d_head must be even");
    RopeTables t;
    t.max_ctx = max_ctx;
    t.half_dim = d_head / 2;
    t.theta_base = theta_base;
    t.cos_raw.resize(size_t(max_ctx) * t.half_dim);
    t.sin_raw.resize(t.cos_raw.size());
    check(dimg_rope_tables(theta_base, d_head, max_ctx, t.cos_raw.data(), t.sin_raw.data()));
    return t;
}

inline std::vector<uint8_t> serialize_rope_tables(const RopeTables& t) {  // rope.cpp:41-51
    size_t n = 0;
    check(dimg_rtab_serialize(t.theta_base, t.max_ctx, t.half_dim, t.cos_raw.data(), t.sin_raw.data(), nullptr, 0, &n));
    std::vector<uint8_t> out(n);
    check(dimg_rtab_serialize(t.theta_base, t.max_ctx, t.half_dim, t.cos_raw.data(), t.sin_raw.data(), out.data(),
                              out.size(), &n));
    return out;
}

inline RopeTables deserialize_rope_tables(std::span<const uint8_t> bytes) {  // rope.cpp:53-78
    RopeTables t;
    check(dimg_rtab_deserialize(bytes.data(), bytes.size(), &t.max_ctx, &t.half_dim, &t.theta_base, nullptr, nullptr,
                                0));
    const size_t cells = size_t(t.max_ctx) * t.half_dim;
    t.cos_raw.resize(cells);
    t.sin_raw.resize(cells);
    check(dimg_rtab_deserialize(bytes.data(), bytes.size(), &t.max_ctx, &t.half_dim, &t.theta_base, t.cos_raw.data(),
                                t.sin_raw.data(), cells));
    return t;
}

inline void save_rope_tables(const RopeTables& t, const std::string& path) {  // rope.cpp:80-86
    const dimg_status s = dimg_rtab_save(path.c_str(), t.theta_base, t.max_ctx, t.half_dim, t.cos_raw.data(),
                                         t.sin_raw.data());
    if (s == DIMG_EIO) throw std::runtime_error(dimg_last_error());
    check(s);
}

inline RopeTables load_rope_tables(const std::string& path) {  // rope.cpp:88-93
    size_t n = 0;
    dimg_status s = dimg_rtab_load(path.c_str(), nullptr, 0, &n);
    if (s == DIMG_EIO) throw std::runtime_error(dimg_last_error());
    check(s);
    std::vector<uint8_t> b(n);
    check(dimg_rtab_load(path.c_str(), b.data(), b.size(), &n));
    return deserialize_rope_tables(b);
}

inline uint32_t select_greedy(std::span<const int64_t> logits) {  // engine.cpp:113-120
    uint32_t i = 0;
    check(dimg_select_greedy(logits.data(), logits.size(), &i));
    return i;
}

class InferenceSession {  // proj/include/dim/engine.hpp:41-57
  public:
    explicit InferenceSession(const ModelFile& model, EngineOptions opts = {}, uint32_t keep_logits_cap = 0)
        : model_(model), vocab_(model.config().vocab) {
        model.config().validate();
        dimg_session* s = nullptr;
        check(dimg_session_create(model.device_model(opts.device), keep_logits_cap, &s));
        s_.reset(s);
    }
    // Runs token at position pos (== cache length); returns the logits.
    std::vector<int64_t> forward(uint32_t token, uint32_t pos) {
        std::vector<int64_t> out(vocab_);
        check(dimg_session_forward(s_.get(), token, pos, out.data()));
        return out;
    }
    uint32_t cache_len() const {
        uint32_t n = 0;
        check(dimg_session_len(s_.get(), &n));
        return n;
    }
    GenerationResult generate_greedy(std::span<const uint32_t> prompt, size_t max_new, bool keep_logits) {
        GenerationResult r;
        r.token_ids.resize(max_new);
        std::vector<int64_t> flat(keep_logits ? max_new * vocab_ : 0);
        check(dimg_generate_greedy(s_.get(), prompt.data(), uint32_t(prompt.size()), uint32_t(max_new),
                                   r.token_ids.data(), r.output_hash.bytes.data(),
                                   keep_logits ? flat.data() : nullptr));
        for (size_t i = 0; keep_logits && i < max_new; ++i)
            r.logits.emplace_back(flat.begin() + i * vocab_, flat.begin() + (i + 1) * vocab_);
        return r;
    }

  private:
    struct Free {
        void operator()(dimg_session* p) const { dimg_session_free(p); }
    };
    ModelFile model_;
    uint32_t vocab_;
    std::unique_ptr<dimg_session, Free> s_;
};

// generate_greedy (proj/include/dim/engine.hpp:70-72): prompt + greedy
// continuation + BLAKE3 output hash, one persistent GPU launch.
inline GenerationResult generate_greedy(const ModelFile& model, std::span<const uint32_t> prompt,
                                        size_t max_new, EngineOptions opts = {}) {
    InferenceSession s(model, opts, opts.keep_logits ? uint32_t(max_new) : 0);
    return s.generate_greedy(prompt, max_new, opts.keep_logits);
}

}  // namespace dimg
