// extern "C" host half of include/dimg.h: hashing, RNG, prompt parsing,
// tables and the DIM1 container.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "blake3.hpp"
#include "chacha20.hpp"
#include "common.hpp"
#include "model.hpp"

namespace dimg {
namespace {
thread_local std::string g_err;
thread_local int g_parse_kind = -1;
}  // namespace

void set_last_error(dimg_status code, const char* msg, int parse_kind) {
    g_err = code == DIMG_OK ? std::string() : std::string(msg);
    g_parse_kind = parse_kind;
}
}  // namespace dimg

struct dimg_host_model {
    dimg::HostModel m;
};

using namespace dimg;

extern "C" {

const char* dimg_last_error(void) { return g_err.c_str(); }
int dimg_last_parse_kind(void) { return g_parse_kind; }
const char* dimg_version(void) { return "dimg 0.1 (sm_100a)"; }

dimg_status dimg_config_validate(const dimg_config* cfg) { DIMG_API_GUARD(validate_config(*cfg)) }

dimg_status dimg_blake3(const void* data, size_t len, uint8_t out[32]) {
    DIMG_API_GUARD({
        auto d = b3::hash(data, len, 0);
        std::memcpy(out, d.data(), 32);
    })
}

dimg_status dimg_hash_token_ids(const uint32_t* ids, size_t n, uint8_t out[32]) {
    // BLAKE3 over u32-LE ids (proj/src/engine.cpp:104-111); x86 is LE already
    DIMG_API_GUARD({
        auto d = b3::hash(ids, n * 4, 1);
        std::memcpy(out, d.data(), 32);
    })
}

dimg_status dimg_select_greedy(const int64_t* logits, size_t n, uint32_t* out) {
    DIMG_API_GUARD({
        if (n == 0) fail(DIMG_EINVAL, "select_greedy: empty logits");
        size_t best = 0;
        for (size_t i = 1; i < n; ++i)
            if (logits[i] > logits[best]) best = i;
        *out = uint32_t(best);
    })
}

dimg_status dimg_prompt_from_seed(uint64_t seed, uint32_t vocab, uint32_t n, uint32_t* out) {
    DIMG_API_GUARD({
        if (vocab == 0) fail(DIMG_EINVAL, "prompt: vocab must be positive");
        chacha::Stream s(chacha::key_from_seed(seed));
        for (uint32_t i = 0; i < n; ++i) out[i] = s.u32() % vocab;
    })
}

dimg_status dimg_parse_prompt(const char* csv, const char* bytes, uint32_t* out, size_t cap,
                              size_t* n) {
    // proj/tools/dim_cli.cpp:56-70
    DIMG_API_GUARD({
        size_t k = 0;
        auto push = [&](uint32_t v) {
            if (k < cap) out[k] = v;
            ++k;
        };
        if (bytes && *bytes) {
            for (const unsigned char* p = reinterpret_cast<const unsigned char*>(bytes); *p; ++p)
                push(uint32_t(*p));
        } else {
            std::string s = csv ? csv : "";
            size_t start = 0;
            while (start <= s.size()) {
                size_t comma = s.find(',', start);
                std::string item = s.substr(start, comma == std::string::npos ? std::string::npos
                                                                             : comma - start);
                if (!item.empty()) {
                    // uint32_t(std::stoul(item)), truncation included
                    unsigned long v;
                    try {
                        v = std::stoul(item);
                    } catch (const std::out_of_range&) {
                        fail(DIMG_ERANGE, "stoul: '" + item + "' out of range");
                    } catch (const std::invalid_argument&) {
                        fail(DIMG_EINVAL, "stoul: bad token id '" + item + "'");
                    }
                    push(uint32_t(v));
                }
                if (comma == std::string::npos) break;
                start = comma + 1;
            }
            if (k == 0) fail(DIMG_EINVAL, "prompt: no token ids given");
        }
        *n = k;
    })
}

dimg_status dimg_rope_tables(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out,
                             int64_t* sin_out) {
    DIMG_API_GUARD(build_rope(theta, d_head, max_ctx, cos_out, sin_out))
}

dimg_status dimg_exp_lut(int64_t out[257]) {
    DIMG_API_GUARD(for (int i = 0; i <= 256; ++i) out[i] = exp_lut_entry(i))
}

dimg_status dimg_invsqrt_seeds(int64_t out[64]) {
    DIMG_API_GUARD(for (int b = 0; b < 64; ++b) out[b] = invsqrt_seed(b))
}

dimg_status dimg_host_model_gen_toy(uint64_t seed, const dimg_config* cfg, int threads,
                                    dimg_host_model** out) {
    DIMG_API_GUARD(*out = new dimg_host_model{gen_toy_model(seed, *cfg, threads)})
}

dimg_status dimg_host_model_gen_toy_gpu(int device, uint64_t seed, const dimg_config* cfg, dimg_host_model** out) {
    // gen_toy_model with the ChaCha20 weight stream synthesised on the GPU
    DIMG_API_GUARD(*out = new dimg_host_model{gen_toy_model(seed, *cfg, 1, device)})
}

dimg_status dimg_host_model_from_bytes(const uint8_t* bytes, size_t n, dimg_host_model** out) {
    DIMG_API_GUARD(*out = new dimg_host_model{deserialize(bytes, n)})
}

dimg_status dimg_host_model_load(const char* path, dimg_host_model** out) {
    DIMG_API_GUARD({
        std::ifstream f(path, std::ios::binary);
        if (!f) fail(DIMG_EIO, std::string("cannot open ") + path);
        f.seekg(0, std::ios::end);
        size_t n = size_t(f.tellg());
        f.seekg(0);
        std::vector<uint8_t> b(n);
        f.read(reinterpret_cast<char*>(b.data()), std::streamsize(n));
        if (!f) fail(DIMG_EIO, std::string("read failed: ") + path);
        *out = new dimg_host_model{deserialize(b.data(), n)};
    })
}

dimg_status dimg_host_model_save(const dimg_host_model* m, const char* path) {
    DIMG_API_GUARD({
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) fail(DIMG_EIO, std::string("model: cannot open ") + path);
        f.write(reinterpret_cast<const char*>(m->m.bytes.data()), std::streamsize(m->m.bytes.size()));
        if (!f) fail(DIMG_EIO, std::string("model: write failed: ") + path);
    })
}

dimg_status dimg_host_model_from_desc(const dimg_model_desc* d, dimg_host_model** out) {
    DIMG_API_GUARD(*out = new dimg_host_model{serialize_desc(*d)})
}

dimg_status dimg_host_model_bytes(const dimg_host_model* m, const uint8_t** bytes, size_t* n) {
    DIMG_API_GUARD({
        *bytes = m->m.bytes.data();
        *n = m->m.bytes.size();
    })
}

dimg_status dimg_host_model_weight_hash(const dimg_host_model* m, uint8_t out[32]) {
    DIMG_API_GUARD({
        auto d = b3::hash(m->m.bytes.data(), m->m.bytes.size(), 0);
        std::memcpy(out, d.data(), 32);
    })
}

dimg_status dimg_host_model_desc(const dimg_host_model* m, dimg_model_desc* out) {
    DIMG_API_GUARD(*out = m->m.desc())
}

dimg_status dimg_host_model_free(dimg_host_model* m) { DIMG_API_GUARD(delete m) }

}  // extern "C"
