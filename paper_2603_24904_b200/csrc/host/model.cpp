// DIM1 container build / parse and the FP64-built tables.
#include "model.hpp"

#include <algorithm>
#include <thread>
#include <atomic>
#include <cmath>
#include <cstring>

#include "chacha20.hpp"

namespace dimg {
namespace {

constexpr uint32_t kVersion = 1;

struct DirEntry {
    std::string name;
    uint32_t rows, cols;
    uint8_t kind;  // 0 int8 + scales, 1 dense q16
};

// Fixed directory order (proj/src/model.cpp:41-61).
std::vector<DirEntry> directory(const dimg_config& c) {
    std::vector<DirEntry> d;
    d.push_back({"tok_embd", c.vocab, c.d_model, 0});
    for (uint32_t i = 0; i < c.n_layers; ++i) {
        std::string p = "layers." + std::to_string(i) + ".";
        d.push_back({p + "attn_norm", 1, c.d_model, 1});
        d.push_back({p + "wq", c.d_model, c.d_model, 0});
        d.push_back({p + "wk", c.d_model, c.d_model, 0});
        d.push_back({p + "wv", c.d_model, c.d_model, 0});
        d.push_back({p + "wo", c.d_model, c.d_model, 0});
        d.push_back({p + "ffn_norm", 1, c.d_model, 1});
        d.push_back({p + "w_gate", c.d_ffn, c.d_model, 0});
        d.push_back({p + "w_up", c.d_ffn, c.d_model, 0});
        d.push_back({p + "w_down", c.d_model, c.d_ffn, 0});
    }
    d.push_back({"final_norm", 1, c.d_model, 1});
    d.push_back({"output", c.vocab, c.d_model, 0});
    return d;
}

struct Writer {
    uint8_t* p;
    void raw(const void* s, size_t n) {
        std::memcpy(p, s, n);
        p += n;
    }
    template <class T>
    void le(T v) {
        for (size_t i = 0; i < sizeof(T); ++i) *p++ = uint8_t(uint64_t(v) >> (8 * i));
    }
};

struct Reader {
    const uint8_t* p;
    size_t n, off = 0;
    void need(size_t k) const {
        if (n - off < k) fail_parse(DIMG_PARSE_TRUNCATED, "truncated input");
    }
    template <class T>
    T le() {
        need(sizeof(T));
        uint64_t v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= uint64_t(p[off + i]) << (8 * i);
        off += sizeof(T);
        return T(v);
    }
    std::string str(size_t k) {
        need(k);
        std::string s(reinterpret_cast<const char*>(p + off), k);
        off += k;
        return s;
    }
};

size_t header_size(const std::vector<DirEntry>& dir) {
    size_t n = 4 + 4 + 6 * 4 + 8 + 4;
    for (auto& e : dir) n += 2 + e.name.size() + 4 + 4 + 1;
    return n;
}

uint32_t isqrt_floor(uint32_t v) {
    uint32_t r = uint32_t(std::sqrt(double(v)));
    while (uint64_t(r + 1) * (r + 1) <= v) ++r;
    while (uint64_t(r) * r > v) --r;
    return r;
}

// Lays out header + directory and records every payload offset; payloads
// are left for the caller to fill.
void layout(HostModel& m) {
    auto dir = directory(m.cfg);
    size_t total = header_size(dir);
    for (auto& e : dir) total += e.kind == 0 ? size_t(e.rows) * 8 + size_t(e.rows) * e.cols
                                             : size_t(e.cols) * 8;
    m.bytes.assign(total, 0);
    Writer w{m.bytes.data()};
    w.raw("DIM1", 4);
    w.le<uint32_t>(kVersion);
    for (uint32_t v : {m.cfg.n_layers, m.cfg.d_model, m.cfg.n_heads, m.cfg.d_ffn, m.cfg.vocab,
                       m.cfg.max_ctx})
        w.le<uint32_t>(v);
    uint64_t tb;
    std::memcpy(&tb, &m.cfg.rope_theta, 8);
    w.le<uint64_t>(tb);
    w.le<uint32_t>(uint32_t(dir.size()));
    for (auto& e : dir) {
        w.le<uint16_t>(uint16_t(e.name.size()));
        w.raw(e.name.data(), e.name.size());
        w.le<uint32_t>(e.rows);
        w.le<uint32_t>(e.cols);
        w.le<uint8_t>(e.kind);
    }
    size_t off = size_t(w.p - m.bytes.data());
    m.q_rows.clear(); m.q_cols.clear(); m.q_scale_off.clear(); m.q_data_off.clear();
    m.norm_off.clear();
    for (auto& e : dir) {
        if (e.kind == 0) {
            m.q_rows.push_back(e.rows);
            m.q_cols.push_back(e.cols);
            m.q_scale_off.push_back(off);
            off += size_t(e.rows) * 8;
            m.q_data_off.push_back(off);
            off += size_t(e.rows) * e.cols;
        } else {
            m.norm_off.push_back(off);
            off += size_t(e.cols) * 8;
        }
    }
}

void gather_aligned(HostModel& m) {
    size_t ns = 0;
    for (size_t r : m.q_rows) ns += r;
    m.scales.resize(ns);
    size_t o = 0;
    for (size_t i = 0; i < m.q_rows.size(); ++i) {
        std::memcpy(m.scales.data() + o, m.bytes.data() + m.q_scale_off[i], m.q_rows[i] * 8);
        o += m.q_rows[i];
    }
    m.norms.resize(m.norm_off.size() * size_t(m.cfg.d_model));
    for (size_t i = 0; i < m.norm_off.size(); ++i)
        std::memcpy(m.norms.data() + i * m.cfg.d_model, m.bytes.data() + m.norm_off[i],
                    size_t(m.cfg.d_model) * 8);
    m.layer_desc.resize(size_t(m.cfg.n_layers) * 7);
}

}  // namespace

void validate_config(const dimg_config& c) {
    if (c.n_layers < 1) fail(DIMG_EINVAL, "config: n_layers must be >= 1");
    if (c.n_heads < 1) fail(DIMG_EINVAL, "config: n_heads must be >= 1");
    if (c.d_model == 0 || c.d_model % c.n_heads != 0)
        fail(DIMG_EINVAL, "config: d_model must be a positive multiple of n_heads");
    if (c.d_model > 8192) fail(DIMG_EINVAL, "config: d_model exceeds 8192");
    if ((c.d_model / c.n_heads) % 2 != 0) fail(DIMG_EINVAL, "config: d_head must be even");
    if (c.d_ffn < 1) fail(DIMG_EINVAL, "config: d_ffn must be >= 1");
    if (c.vocab < 2) fail(DIMG_EINVAL, "config: vocab must be >= 2");
    if (c.max_ctx < 1) fail(DIMG_EINVAL, "config: max_ctx must be >= 1");
    if (!(c.rope_theta > 0.0) || !std::isfinite(c.rope_theta))
        fail(DIMG_EINVAL, "config: rope_theta must be positive and finite");
}

dimg_model_desc HostModel::desc() const {
    dimg_model_desc d{};
    d.cfg = cfg;
    auto qt = [&](size_t i, size_t so) {
        dimg_qtensor t;
        t.rows = uint32_t(q_rows[i]);
        t.cols = uint32_t(q_cols[i]);
        t.data = reinterpret_cast<const int8_t*>(bytes.data() + q_data_off[i]);
        t.scales = scales.data() + so;
        return t;
    };
    size_t so = 0;
    auto& ld = const_cast<std::vector<dimg_qtensor>&>(layer_desc);
    for (size_t i = 0; i < q_rows.size(); ++i) {
        dimg_qtensor t = qt(i, so);
        so += q_rows[i];
        if (i == 0) d.tok_embd = t;
        else if (i + 1 == q_rows.size()) d.output = t;
        else ld[i - 1] = t;
    }
    d.layers = layer_desc.data();
    d.norms = norms.data();
    return d;
}

int64_t q16_from_ratio(int64_t num, int64_t den) {
    // round half away from zero of num*65536/den (proj/src/q16.cpp:13-24,47-50)
    if (den == 0) fail(DIMG_EINVAL, "q16_from_ratio: zero denominator");
    __int128 n = __int128(num) * 65536, d = den;
    __int128 q = n / d, r = n % d;
    if (r != 0) {
        __int128 ad = d < 0 ? -d : d, ar = r < 0 ? -r : r;
        if (2 * ar >= ad) q += ((n < 0) != (d < 0)) ? -1 : 1;
    }
    return int64_t(q);
}

HostModel gen_toy_model(uint64_t seed, const dimg_config& cfg, int threads, int device) {
    validate_config(cfg);
    HostModel m;
    m.cfg = cfg;
    layout(m);
    std::vector<chacha::Span> spans;
    for (size_t i = 0; i < m.q_rows.size(); ++i) {
        // scale = 1 / (127 * floor(sqrt(cols))) in Q16 (proj/src/model.cpp:70-77)
        int64_t s = q16_from_ratio(1, 127ll * isqrt_floor(uint32_t(m.q_cols[i])));
        uint8_t* sp = m.bytes.data() + m.q_scale_off[i];
        for (size_t r = 0; r < m.q_rows[i]; ++r) Writer{sp + 8 * r}.le<uint64_t>(uint64_t(s));
        spans.push_back({reinterpret_cast<int8_t*>(m.bytes.data() + m.q_data_off[i]),
                         m.q_rows[i] * m.q_cols[i]});
    }
    for (size_t off : m.norm_off)  // gains = ONE
        for (uint32_t j = 0; j < cfg.d_model; ++j) Writer{m.bytes.data() + off + 8 * j}.le<uint64_t>(kOne);
    if (device >= 0) chacha::gpu_weight_stream(device, seed, spans.data(), spans.size());
    else chacha::weight_stream(seed, spans.data(), spans.size(), threads);
    gather_aligned(m);
    return m;
}

namespace {

// Splits [0, n) over the host threads (one piece each for small n).
template <class F>
void parallel_ranges(size_t n, F&& f) {
    const size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t parts = n < (size_t(16) << 20) ? 1 : std::min<size_t>(hw, n >> 20);
    if (parts <= 1) {
        f(size_t(0), n);
        return;
    }
    std::vector<std::thread> ts;
    for (size_t t = 0; t < parts; ++t) ts.emplace_back([&, t] { f(n * t / parts, n * (t + 1) / parts); });
    for (auto& th : ts) th.join();
}

// Does any byte equal 0x80 (int8 -128)? Eight bytes at a time: a byte of
// v ^ 0x80..80 is zero exactly where v held 0x80.
bool has_minus128(const uint8_t* p, size_t n) {
    std::atomic<bool> hit{false};
    parallel_ranges(n, [&](size_t a, size_t b) {
        size_t i = a;
        for (; i < b && (reinterpret_cast<uintptr_t>(p + i) & 7); ++i)
            if (p[i] == 0x80) { hit = true; return; }
        constexpr uint64_t k80 = 0x8080808080808080ull, k01 = 0x0101010101010101ull;
        for (; i + 8 <= b; i += 8) {
            if ((i & ((1u << 20) - 1)) == 0 && hit.load(std::memory_order_relaxed)) return;
            uint64_t v;
            std::memcpy(&v, p + i, 8);
            const uint64_t x = v ^ k80;
            if ((x - k01) & ~x & k80) { hit = true; return; }
        }
        for (; i < b; ++i)
            if (p[i] == 0x80) { hit = true; return; }
    });
    return hit.load();
}

}  // namespace

HostModel deserialize(const uint8_t* bytes, size_t n) {
    // strict parse (proj/src/model.cpp:251-312)
    Reader r{bytes, n};
    if (r.str(4) != "DIM1") fail_parse(DIMG_PARSE_BAD_MAGIC, "model: bad magic");
    if (r.le<uint32_t>() != kVersion) fail_parse(DIMG_PARSE_BAD_VERSION, "model: unsupported version");
    HostModel m;
    m.cfg.n_layers = r.le<uint32_t>();
    m.cfg.d_model = r.le<uint32_t>();
    m.cfg.n_heads = r.le<uint32_t>();
    m.cfg.d_ffn = r.le<uint32_t>();
    m.cfg.vocab = r.le<uint32_t>();
    m.cfg.max_ctx = r.le<uint32_t>();
    uint64_t tb = r.le<uint64_t>();
    std::memcpy(&m.cfg.rope_theta, &tb, 8);
    try {
        validate_config(m.cfg);
    } catch (const Error& e) {
        fail_parse(DIMG_PARSE_INVARIANT, e.what());
    }
    auto dir = directory(m.cfg);
    if (r.le<uint32_t>() != dir.size()) fail_parse(DIMG_PARSE_INVARIANT, "model: unexpected tensor count");
    for (auto& e : dir) {
        uint16_t nl = r.le<uint16_t>();
        std::string name = r.str(nl);
        uint32_t rows = r.le<uint32_t>(), cols = r.le<uint32_t>();
        uint8_t kind = r.le<uint8_t>();
        if (name != e.name || rows != e.rows || cols != e.cols || kind != e.kind)
            fail_parse(DIMG_PARSE_INVARIANT, "model: directory entry mismatch at " + e.name);
    }
    for (auto& e : dir) {
        size_t need = e.kind == 0 ? size_t(e.rows) * 8 + size_t(e.rows) * e.cols : size_t(e.cols) * 8;
        if (e.kind == 0) {
            // whole tensor read first, then invariants: -128 before scales
            // (check_quant_invariants, proj/src/model.cpp:79-93)
            r.need(size_t(e.rows) * 8);
            bool bad_scale = false;
            for (uint32_t i = 0; i < e.rows; ++i) bad_scale |= r.le<int64_t>() <= 0;
            r.need(size_t(e.rows) * e.cols);
            if (has_minus128(bytes + r.off, size_t(e.rows) * e.cols))
                fail_parse(DIMG_PARSE_INVARIANT, e.name + ": weight value -128");
            if (bad_scale) fail_parse(DIMG_PARSE_INVARIANT, e.name + ": non-positive scale");
            r.off += size_t(e.rows) * e.cols;
        } else {
            r.need(need);
            r.off += need;
        }
    }
    if (r.off != n) fail_parse(DIMG_PARSE_INVARIANT, "model: trailing bytes");
    layout(m);  // offsets are a pure function of the config
    parallel_ranges(n, [&](size_t a, size_t b) { std::memcpy(m.bytes.data() + a, bytes + a, b - a); });
    gather_aligned(m);
    return m;
}

HostModel serialize_desc(const dimg_model_desc& d) {
    validate_config(d.cfg);
    HostModel m;
    m.cfg = d.cfg;
    layout(m);
    for (size_t i = 0; i < m.q_rows.size(); ++i) {
        const dimg_qtensor& t = i == 0 ? d.tok_embd
                                : (i + 1 == m.q_rows.size() ? d.output : d.layers[i - 1]);
        if (t.rows != m.q_rows[i] || t.cols != m.q_cols[i])
            fail(DIMG_EINVAL, "model: tensor shape does not match the config");
        for (size_t r = 0; r < t.rows; ++r) {
            if (t.scales[r] <= 0) fail(DIMG_EINVAL, "model: non-positive scale");
            Writer{m.bytes.data() + m.q_scale_off[i] + 8 * r}.le<uint64_t>(uint64_t(t.scales[r]));
        }
        std::memcpy(m.bytes.data() + m.q_data_off[i], t.data, m.q_rows[i] * m.q_cols[i]);
    }
    for (size_t i = 0; i < m.norm_off.size(); ++i)
        for (uint32_t j = 0; j < d.cfg.d_model; ++j)
            Writer{m.bytes.data() + m.norm_off[i] + 8 * j}.le<uint64_t>(
                uint64_t(d.norms[i * d.cfg.d_model + j]));
    gather_aligned(m);
    return m;
}

void build_rope(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out, int64_t* sin_out) {
    // angle = pos * theta^(-2k/d_head) in FP64, llround(v * 65536)
    // (proj/src/rope.cpp:17-39, q16_from_real proj/src/q16.cpp:52-54)
    if (d_head == 0 || d_head % 2 != 0) fail(DIMG_EINVAL, "rope: d_head must be even");
    if (max_ctx == 0) fail(DIMG_EINVAL, "rope: max_ctx must be >= 1");
    if (!(theta > 0.0) || !std::isfinite(theta)) fail(DIMG_EINVAL, "rope: theta_base must be positive and finite");
    const uint32_t half = d_head / 2;
    for (uint32_t k = 0; k < half; ++k) {
        double freq = std::pow(theta, -2.0 * double(k) / double(d_head));
        for (uint32_t pos = 0; pos < max_ctx; ++pos) {
            double a = double(pos) * freq;
            cos_out[size_t(pos) * half + k] = int64_t(std::llround(std::cos(a) * 65536.0));
            sin_out[size_t(pos) * half + k] = int64_t(std::llround(std::sin(a) * 65536.0));
        }
    }
}

int64_t exp_lut_entry(int i) {
    // round(exp(-8 + i/32) * 65536) (proj/src/q16.cpp:70-79)
    return int64_t(std::llround(std::exp(-8.0 + double(i) / 32.0) * 65536.0));
}

int64_t invsqrt_seed(int b) {
    // Q48 seed at the geometric midpoint of octave [2^b, 2^(b+1)) (q16.cpp:28-43)
    double mid = std::ldexp(1.0, b - 16) * std::sqrt(2.0);
    double raw = (1.0 / std::sqrt(mid)) * 0x1.0p48;
    return raw >= 1.0 ? int64_t(std::llround(raw)) : 1;
}

}  // namespace dimg
