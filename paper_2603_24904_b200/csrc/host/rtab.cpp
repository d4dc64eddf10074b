// RTAB: the reference's byte-exact RoPE table artifact
// (proj/src/rope.cpp:41-93, proj/include/dim/rope.hpp:28-39):
//   "RTAB" | u32 version (1) | u32 max_ctx | u32 half_dim | f64 theta_base |
//   cos_raw i64[max_ctx*half_dim] | sin_raw i64[max_ctx*half_dim]
// all little-endian. Parse errors carry the reference's ParseError kinds:
// bad magic, bad version, truncated (a read past the end, wire.hpp:89),
// invariant (empty dimensions, trailing bytes). Imported tables feed
// dimg_model_desc.rope_cos/rope_sin (InferenceSession's imported_tables).
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "common.hpp"

namespace {

constexpr char kMagic[4] = {'R', 'T', 'A', 'B'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 4 + 4 + 4 + 4 + 8;

template <class T>
void put_le(uint8_t*& p, T v) {
    std::memcpy(p, &v, sizeof v);  // x86-64 is little-endian, as the wire format
    p += sizeof v;
}

struct Reader {
    const uint8_t* p;
    size_t n, pos = 0;
    template <class T>
    T get() {
        if (n - pos < sizeof(T)) dimg::fail_parse(DIMG_PARSE_TRUNCATED, "truncated input");
        T v;
        std::memcpy(&v, p + pos, sizeof v);
        pos += sizeof v;
        return v;
    }
};

size_t rtab_bytes(uint32_t max_ctx, uint32_t half_dim) {
    return kHeader + size_t(2) * max_ctx * half_dim * 8;
}

// Header fields of an RTAB, checked in deserialize_rope_tables' order (magic,
// version, dims, then the payload length: short = truncated, long = trailing).
void parse_header(const uint8_t* b, size_t n, uint32_t* max_ctx, uint32_t* half_dim, double* theta) {
    Reader r{b, n};
    char magic[4];
    for (char& c : magic) c = char(r.get<uint8_t>());
    if (std::memcmp(magic, kMagic, 4) != 0) dimg::fail_parse(DIMG_PARSE_BAD_MAGIC, "rope tables: bad magic");
    if (r.get<uint32_t>() != kVersion)
        dimg::fail_parse(DIMG_PARSE_BAD_VERSION, "rope tables: unsupported version");
    *max_ctx = r.get<uint32_t>();
    *half_dim = r.get<uint32_t>();
    *theta = r.get<double>();
    if (*max_ctx == 0 || *half_dim == 0) dimg::fail_parse(DIMG_PARSE_INVARIANT, "rope tables: empty dimensions");
    const unsigned __int128 want = kHeader + (unsigned __int128)(2 * 8) * *max_ctx * *half_dim;
    if (n < want) dimg::fail_parse(DIMG_PARSE_TRUNCATED, "truncated input");
    if (n > want) dimg::fail_parse(DIMG_PARSE_INVARIANT, "rope tables: trailing bytes");
}

}  // namespace

extern "C" {

dimg_status dimg_rtab_serialize(double theta, uint32_t max_ctx, uint32_t half_dim, const int64_t* cos_raw,
                                const int64_t* sin_raw, uint8_t* out, size_t cap, size_t* n) {
    DIMG_API_GUARD({
        const size_t need = rtab_bytes(max_ctx, half_dim);
        *n = need;
        if (!out) return DIMG_OK;  // size query
        if (cap < need) dimg::fail(DIMG_ELENGTH, "rtab: output buffer too small");
        uint8_t* p = out;
        std::memcpy(p, kMagic, 4);
        p += 4;
        put_le<uint32_t>(p, kVersion);
        put_le<uint32_t>(p, max_ctx);
        put_le<uint32_t>(p, half_dim);
        put_le<double>(p, theta);
        const size_t cells = size_t(max_ctx) * half_dim;
        std::memcpy(p, cos_raw, cells * 8);
        std::memcpy(p + cells * 8, sin_raw, cells * 8);
    })
}

dimg_status dimg_rtab_deserialize(const uint8_t* bytes, size_t n, uint32_t* max_ctx, uint32_t* half_dim,
                                  double* theta, int64_t* cos_out, int64_t* sin_out, size_t cap_cells) {
    DIMG_API_GUARD({
        parse_header(bytes, n, max_ctx, half_dim, theta);
        const size_t cells = size_t(*max_ctx) * *half_dim;
        if (!cos_out && !sin_out) return DIMG_OK;  // header query
        if (cap_cells < cells) dimg::fail(DIMG_ELENGTH, "rtab: table buffers too small");
        std::memcpy(cos_out, bytes + kHeader, cells * 8);
        std::memcpy(sin_out, bytes + kHeader + cells * 8, cells * 8);
    })
}

dimg_status dimg_rtab_save(const char* path, double theta, uint32_t max_ctx, uint32_t half_dim,
                           const int64_t* cos_raw, const int64_t* sin_raw) {
    // save_rope_tables (rope.cpp:80-86): runtime_error -> DIMG_EIO
    DIMG_API_GUARD({
        std::vector<uint8_t> b(rtab_bytes(max_ctx, half_dim));
        size_t n = 0;
        const dimg_status st = dimg_rtab_serialize(theta, max_ctx, half_dim, cos_raw, sin_raw, b.data(), b.size(), &n);
        if (st != DIMG_OK) return st;
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) dimg::fail(DIMG_EIO, std::string("rope tables: cannot open ") + path);
        f.write(reinterpret_cast<const char*>(b.data()), std::streamsize(n));
        if (!f) dimg::fail(DIMG_EIO, std::string("rope tables: write failed: ") + path);
    })
}

dimg_status dimg_rtab_load(const char* path, uint8_t* out, size_t cap, size_t* n) {
    // load_rope_tables (rope.cpp:88-93) as bytes: the caller deserializes
    // (size query with out == NULL)
    DIMG_API_GUARD({
        std::ifstream f(path, std::ios::binary);
        if (!f) dimg::fail(DIMG_EIO, std::string("rope tables: cannot open ") + path);
        std::vector<uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        *n = b.size();
        if (!out) return DIMG_OK;
        if (cap < b.size()) dimg::fail(DIMG_ELENGTH, "rtab: output buffer too small");
        std::memcpy(out, b.data(), b.size());
    })
}

}  // extern "C"
