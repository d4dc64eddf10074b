/*
 * dim_oracle.c -- TEST INFRASTRUCTURE ONLY (see dim_oracle.h).
 *
 * Plain-C restatement of the reference's integer forward pass. Scalar loops,
 * __int128 wherever the reference widens, and unsigned arithmetic wherever
 * the reference's int64/int128 sums could wrap (the reference relies on the
 * two's-complement wrap of its accumulators; unsigned arithmetic gives the
 * same bits without C undefined behaviour).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp). The FP64
 * table builders must see the same libm and no FMA contraction as the
 * reference (proj/CMakeLists.txt:13 sets -ffp-contract=off).
 */
#include "dim_oracle.h"

#include <stdio.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

#define ONE ((int64_t)65536)
#define ACT_CLAMP (256 * ONE) /* proj/include/dim/kernels.hpp:16 */

/* ======================================================================= */
/* BLAKE3 (spec restated; reference: proj/src/blake3.cpp)                   */
/* ======================================================================= */

static const uint32_t B3_IV[8] = {0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au,
                                  0x510E527Fu, 0x9B05688Cu, 0x1F83D9ABu, 0x5BE0CD19u};
static const uint8_t B3_PERM[16] = {2, 6, 3, 10, 7, 0, 4, 13, 1, 11, 12, 5, 9, 14, 15, 8};
enum { B3_CHUNK_START = 1, B3_CHUNK_END = 2, B3_PARENT = 4, B3_ROOT = 8 };

static inline uint32_t rotr32(uint32_t v, int n) { return (v >> n) | (v << (32 - n)); }

static void b3_g(uint32_t* v, int a, int b, int c, int d, uint32_t x, uint32_t y) {
    v[a] += v[b] + x;
    v[d] = rotr32(v[d] ^ v[a], 16);
    v[c] += v[d];
    v[b] = rotr32(v[b] ^ v[c], 12);
    v[a] += v[b] + y;
    v[d] = rotr32(v[d] ^ v[a], 8);
    v[c] += v[d];
    v[b] = rotr32(v[b] ^ v[c], 7);
}

/* compression function: 7 rounds, message permuted between rounds */
static void b3_compress(const uint32_t cv[8], const uint32_t msg[16], uint64_t counter,
                        uint32_t len, uint32_t flags, uint32_t out[16]) {
    uint32_t v[16] = {cv[0], cv[1], cv[2], cv[3], cv[4], cv[5], cv[6], cv[7],
                      B3_IV[0], B3_IV[1], B3_IV[2], B3_IV[3],
                      (uint32_t)counter, (uint32_t)(counter >> 32), len, flags};
    uint32_t m[16], t[16];
    memcpy(m, msg, sizeof m);
    for (int r = 0; r < 7; ++r) {
        b3_g(v, 0, 4, 8, 12, m[0], m[1]);
        b3_g(v, 1, 5, 9, 13, m[2], m[3]);
        b3_g(v, 2, 6, 10, 14, m[4], m[5]);
        b3_g(v, 3, 7, 11, 15, m[6], m[7]);
        b3_g(v, 0, 5, 10, 15, m[8], m[9]);
        b3_g(v, 1, 6, 11, 12, m[10], m[11]);
        b3_g(v, 2, 7, 8, 13, m[12], m[13]);
        b3_g(v, 3, 4, 9, 14, m[14], m[15]);
        for (int i = 0; i < 16; ++i) t[i] = m[B3_PERM[i]];
        memcpy(m, t, sizeof m);
    }
    for (int i = 0; i < 8; ++i) {
        out[i] = v[i] ^ v[i + 8];
        out[i + 8] = v[i + 8] ^ cv[i];
    }
}

static void b3_words(const uint8_t* p, uint32_t w[16]) {
    for (int i = 0; i < 16; ++i)
        w[i] = (uint32_t)p[4 * i] | (uint32_t)p[4 * i + 1] << 8 | (uint32_t)p[4 * i + 2] << 16 |
               (uint32_t)p[4 * i + 3] << 24;
}

static void b3_parent_cv(const uint32_t l[8], const uint32_t r[8], uint32_t flags,
                         uint32_t out[16]) {
    uint32_t m[16];
    memcpy(m, l, 32);
    memcpy(m + 8, r, 32);
    b3_compress(B3_IV, m, 0, 64, B3_PARENT | flags, out);
}

void orc_blake3_init(orc_blake3* h) {
    memset(h, 0, sizeof *h);
    memcpy(h->cv, B3_IV, 32);
}

void orc_blake3_update(orc_blake3* h, const void* data, size_t len) {
    const uint8_t* p = (const uint8_t*)data;
    while (len > 0) {
        if (h->blocks_done == 15 && h->block_len == 64) {
            /* a full chunk is buffered and more input follows: close it */
            uint32_t w[16], o[16];
            b3_words(h->block, w);
            b3_compress(h->cv, w, h->chunk_counter, 64, B3_CHUNK_END, o);
            uint32_t cv[8];
            memcpy(cv, o, 32);
            uint64_t total = h->chunk_counter + 1;
            while ((total & 1) == 0) {
                b3_parent_cv(h->stack[--h->stack_len], cv, 0, o);
                memcpy(cv, o, 32);
                total >>= 1;
            }
            memcpy(h->stack[h->stack_len++], cv, 32);
            h->chunk_counter++;
            memcpy(h->cv, B3_IV, 32);
            memset(h->block, 0, 64);
            h->block_len = 0;
            h->blocks_done = 0;
        }
        if (h->block_len == 64) {
            uint32_t w[16], o[16];
            b3_words(h->block, w);
            b3_compress(h->cv, w, h->chunk_counter, 64, h->blocks_done == 0 ? B3_CHUNK_START : 0,
                        o);
            memcpy(h->cv, o, 32);
            h->blocks_done++;
            memset(h->block, 0, 64);
            h->block_len = 0;
        }
        size_t take = 64 - h->block_len;
        if (take > len) take = len;
        memcpy(h->block + h->block_len, p, take);
        h->block_len += (uint32_t)take;
        p += take;
        len -= take;
    }
}

void orc_blake3_final(const orc_blake3* h, uint8_t out[32]) {
    uint32_t w[16], o[16];
    b3_words(h->block, w);
    uint32_t flags = B3_CHUNK_END | (h->blocks_done == 0 ? B3_CHUNK_START : 0);
    /* the output node: (cv, words, counter, len, flags) */
    uint32_t node_cv[8], node_m[16];
    uint64_t node_counter = h->chunk_counter;
    uint32_t node_len = h->block_len, node_flags = flags;
    memcpy(node_cv, h->cv, 32);
    memcpy(node_m, w, 64);
    for (uint32_t i = h->stack_len; i-- > 0;) {
        b3_compress(node_cv, node_m, node_counter, node_len, node_flags, o);
        memcpy(node_m, h->stack[i], 32);
        memcpy(node_m + 8, o, 32);
        memcpy(node_cv, B3_IV, 32);
        node_counter = 0;
        node_len = 64;
        node_flags = B3_PARENT;
    }
    b3_compress(node_cv, node_m, 0, node_len, node_flags | B3_ROOT, o);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)o[i];
        out[4 * i + 1] = (uint8_t)(o[i] >> 8);
        out[4 * i + 2] = (uint8_t)(o[i] >> 16);
        out[4 * i + 3] = (uint8_t)(o[i] >> 24);
    }
}

void orc_blake3_oneshot(const void* data, size_t len, uint8_t out[32]) {
    orc_blake3 h;
    orc_blake3_init(&h);
    orc_blake3_update(&h, data, len);
    orc_blake3_final(&h, out);
}

/* ======================================================================= */
/* ChaCha20 (RFC 8439) + keystream RNG (proj/src/chacha20.cpp:20-96)        */
/* ======================================================================= */

static inline uint32_t rotl32(uint32_t v, int n) { return (v << n) | (v >> (32 - n)); }
#define QR(a, b, c, d)                  \
    a += b; d ^= a; d = rotl32(d, 16);  \
    c += d; b ^= c; b = rotl32(b, 12);  \
    a += b; d ^= a; d = rotl32(d, 8);   \
    c += d; b ^= c; b = rotl32(b, 7);

void orc_chacha20_block(const uint32_t key[8], const uint32_t nonce[3], uint32_t counter,
                        uint8_t out[64]) {
    uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                       key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                       counter, nonce[0], nonce[1], nonce[2]};
    uint32_t x[16];
    memcpy(x, in, sizeof x);
    for (int i = 0; i < 10; ++i) {
        QR(x[0], x[4], x[8], x[12]);
        QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]);
        QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]);
        QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]);
        QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; ++i) {
        uint32_t w = x[i] + in[i];
        out[4 * i] = (uint8_t)w;
        out[4 * i + 1] = (uint8_t)(w >> 8);
        out[4 * i + 2] = (uint8_t)(w >> 16);
        out[4 * i + 3] = (uint8_t)(w >> 24);
    }
}

void orc_rng_from_key(orc_rng* r, const uint8_t key[32]) {
    for (int i = 0; i < 8; ++i)
        r->key[i] = (uint32_t)key[4 * i] | (uint32_t)key[4 * i + 1] << 8 |
                    (uint32_t)key[4 * i + 2] << 16 | (uint32_t)key[4 * i + 3] << 24;
    r->counter = 0;
    r->pos = 64;
}

void orc_rng_from_seed(orc_rng* r, uint64_t seed) {
    uint8_t le[8], key[32];
    for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(seed >> (8 * i));
    orc_blake3_oneshot(le, 8, key);
    orc_rng_from_key(r, key);
}

uint8_t orc_rng_u8(orc_rng* r) {
    if (r->pos >= 64) {
        static const uint32_t zero_nonce[3] = {0, 0, 0};
        orc_chacha20_block(r->key, zero_nonce, r->counter++, r->buf);
        r->pos = 0;
    }
    return r->buf[r->pos++];
}

uint32_t orc_rng_u32(orc_rng* r) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)orc_rng_u8(r) << (8 * i);
    return v;
}

uint64_t orc_rng_u64(orc_rng* r) {
    uint64_t lo = orc_rng_u32(r);
    return lo | (uint64_t)orc_rng_u32(r) << 32;
}

int8_t orc_rng_weight(orc_rng* r) {
    for (;;) {
        uint8_t b = orc_rng_u8(r);
        if (b != 255) return (int8_t)((int)b - 127);
    }
}

/* ======================================================================= */
/* Q16 primitives (proj/src/q16.cpp, proj/include/dim/q16.hpp)              */
/* ======================================================================= */

int64_t orc_q16_from_ratio(int64_t num, int64_t den) {
    /* round-half-away-from-zero of num*65536/den (q16.cpp:13-24,47-50) */
    i128 n = (i128)num * 65536, d = den;
    i128 q = n / d, rem = n % d;
    if (rem != 0) {
        i128 ad = d < 0 ? -d : d, ar = rem < 0 ? -rem : rem;
        if (2 * ar >= ad) q += ((n < 0) != (d < 0)) ? -1 : 1;
    }
    return (int64_t)q;
}

int64_t orc_q16_mul(int64_t a, int64_t b) { return (int64_t)(((i128)a * (i128)b) >> 16); }

int64_t orc_invsqrt_seed(int b) {
    /* seed at the geometric midpoint of raw octave [2^b, 2^(b+1)) in Q48 */
    double mid = ldexp(1.0, b - 16) * sqrt(2.0);
    double raw = (1.0 / sqrt(mid)) * 0x1.0p48;
    return raw >= 1.0 ? (int64_t)llround(raw) : 1;
}

int64_t orc_inv_sqrt(int64_t x) {
    /* three Newton steps y <- y(3 - x y^2)/2 at Q48 (q16.cpp:56-68) */
    int b = 63 - __builtin_clzll((uint64_t)x);
    i128 y = orc_invsqrt_seed(b);
    for (int it = 0; it < 3; ++it) {
        i128 t = (y * y) >> 48;
        i128 u = ((i128)x * t) >> 16;
        y = (y * (((i128)3 << 48) - u)) >> 49;
    }
    return (int64_t)((y + ((i128)1 << 31)) >> 32);
}

int64_t orc_exp_entry(int i) { return (int64_t)llround(exp(-8.0 + (double)i / 32.0) * 65536.0); }

static int64_t g_exp[257];
static int g_exp_ready = 0;
static const int64_t* exp_table(void) {
    if (!g_exp_ready) {
        for (int i = 0; i <= 256; ++i) g_exp[i] = orc_exp_entry(i);
        __atomic_store_n(&g_exp_ready, 1, __ATOMIC_RELEASE);
    }
    return g_exp;
}

/* exp_neg_lut's std::domain_error for t outside [0, 8] (q16.cpp:82): the
 * restatement raises a sticky thread-local flag instead of throwing
 * (orc_domain_error reads and clears it); the weight is then 0. */
static _Thread_local int g_domain_error;
int orc_domain_error(void) {
    int e = g_domain_error;
    g_domain_error = 0;
    return e;
}

int64_t orc_exp_neg(int64_t t) {
    /* 2048 raw units per cell, round-half-up interpolation (q16.cpp:81-92) */
    const int64_t* e = exp_table();
    if (t < 0 || t > 8 * ONE) {
        g_domain_error = 1;
        return 0;
    }
    int64_t cell = t >> 11, frac = t & 2047;
    if (cell == 256) return e[0];
    int64_t hi = e[256 - cell], lo = e[255 - cell];
    return hi - (((hi - lo) * frac + 1024) >> 11);
}

int64_t orc_sigmoid(int64_t x) {
    /* exact symmetry sigma(x) = ONE - sigma(-x) for x > 0 (q16.cpp:94-101) */
    if (x > 0) return ONE - orc_sigmoid(-x);
    int64_t t = x <= -8 * ONE ? 8 * ONE : -x;
    int64_t e = orc_exp_neg(t);
    int64_t den = ONE + e;
    return ((e << 16) + den / 2) / den;
}

int64_t orc_silu(int64_t x) { return orc_q16_mul(x, orc_sigmoid(x)); }

void orc_rope_tables(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out,
                     int64_t* sin_out) {
    /* angle = pos * theta^(-2k/d_head) in FP64 (rope.cpp:17-39) */
    uint32_t half = d_head / 2;
    for (uint32_t k = 0; k < half; ++k) {
        double freq = pow(theta, -2.0 * (double)k / (double)d_head);
        for (uint32_t p = 0; p < max_ctx; ++p) {
            double a = (double)p * freq;
            cos_out[(size_t)p * half + k] = (int64_t)llround(cos(a) * 65536.0);
            sin_out[(size_t)p * half + k] = (int64_t)llround(sin(a) * 65536.0);
        }
    }
}

/* ======================================================================= */
/* model directory, toy generation, DIM1 serialization                     */
/* ======================================================================= */

/* directory walk: fn(kind, name, rows, cols, tensor index or norm index) */
typedef struct {
    char name[48];
    uint32_t rows, cols;
    uint8_t kind;    /* 0 int8+scales, 1 dense q16 */
    int idx;         /* quant: 0 tok_embd, 1..7L layer tensors, 7L+1 output; dense: norm idx */
} dir_entry;

static size_t dir_build(const orc_model* m, dir_entry* d) {
    size_t n = 0;
    uint32_t L = m->n_layers, D = m->d_model, F = m->d_ffn, V = m->vocab;
#define ADD(nm, r, c, k, i)                                  \
    do {                                                      \
        snprintf(d[n].name, sizeof d[n].name, "%s", nm);      \
        d[n].rows = r; d[n].cols = c; d[n].kind = k; d[n].idx = i; ++n; \
    } while (0)
    char buf[48];
    ADD("tok_embd", V, D, 0, 0);
    static const char* qn[7] = {"wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"};
    for (uint32_t l = 0; l < L; ++l) {
        snprintf(buf, sizeof buf, "layers.%u.attn_norm", l);
        ADD(buf, 1, D, 1, (int)(2 * l));
        for (int t = 0; t < 4; ++t) {
            snprintf(buf, sizeof buf, "layers.%u.%s", l, qn[t]);
            ADD(buf, D, D, 0, (int)(1 + 7 * l + t));
        }
        snprintf(buf, sizeof buf, "layers.%u.ffn_norm", l);
        ADD(buf, 1, D, 1, (int)(2 * l + 1));
        snprintf(buf, sizeof buf, "layers.%u.w_gate", l);
        ADD(buf, F, D, 0, (int)(1 + 7 * l + 4));
        snprintf(buf, sizeof buf, "layers.%u.w_up", l);
        ADD(buf, F, D, 0, (int)(1 + 7 * l + 5));
        snprintf(buf, sizeof buf, "layers.%u.w_down", l);
        ADD(buf, D, F, 0, (int)(1 + 7 * l + 6));
    }
    ADD("final_norm", 1, D, 1, (int)(2 * L));
    ADD("output", V, D, 0, (int)(1 + 7 * L));
#undef ADD
    return n;
}

#include <stdio.h>

static void quant_dims(const orc_model* m, int idx, uint32_t* rows, uint32_t* cols) {
    uint32_t L = m->n_layers, D = m->d_model, F = m->d_ffn, V = m->vocab;
    if (idx == 0 || idx == (int)(1 + 7 * L)) { *rows = V; *cols = D; return; }
    int t = (idx - 1) % 7;
    if (t < 4) { *rows = D; *cols = D; }
    else if (t < 6) { *rows = F; *cols = D; }
    else { *rows = D; *cols = F; }
}

uint64_t orc_model_weight_count(const orc_model* m) {
    uint64_t n = 0;
    for (uint32_t i = 0; i < 2 + 7 * m->n_layers; ++i) {
        uint32_t r, c;
        quant_dims(m, (int)i, &r, &c);
        n += (uint64_t)r * c;
    }
    return n;
}

uint64_t orc_model_scale_count(const orc_model* m) {
    uint64_t n = 0;
    for (uint32_t i = 0; i < 2 + 7 * m->n_layers; ++i) {
        uint32_t r, c;
        quant_dims(m, (int)i, &r, &c);
        n += r;
    }
    return n;
}

static uint32_t isqrt32(uint32_t v) {
    uint32_t r = (uint32_t)sqrt((double)v);
    while ((uint64_t)(r + 1) * (r + 1) <= v) ++r;
    while ((uint64_t)r * r > v) --r;
    return r;
}

void orc_gen_toy(uint64_t seed, const orc_model* m, int8_t* weights, int64_t* scales) {
    /* tensors drawn in directory order, one rejection draw per weight;
     * scale = q16_from_ratio(1, 127*floor(sqrt(cols))) (model.cpp:63-77,189-215) */
    orc_rng r;
    orc_rng_from_seed(&r, seed);
    uint64_t wo = 0, so = 0;
    for (uint32_t i = 0; i < 2 + 7 * m->n_layers; ++i) {
        uint32_t rows, cols;
        quant_dims(m, (int)i, &rows, &cols);
        uint64_t n = (uint64_t)rows * cols;
        for (uint64_t j = 0; j < n; ++j) weights[wo + j] = orc_rng_weight(&r);
        int64_t s = orc_q16_from_ratio(1, 127LL * isqrt32(cols));
        for (uint32_t j = 0; j < rows; ++j) scales[so + j] = s;
        wo += n;
        so += rows;
    }
}

void orc_bind(orc_model* m, orc_qtensor* layer_desc, const int8_t* weights,
              const int64_t* scales) {
    uint64_t wo = 0, so = 0;
    for (uint32_t i = 0; i < 2 + 7 * m->n_layers; ++i) {
        orc_qtensor t;
        quant_dims(m, (int)i, &t.rows, &t.cols);
        t.data = weights + wo;
        t.scales = scales + so;
        wo += (uint64_t)t.rows * t.cols;
        so += t.rows;
        if (i == 0) m->tok_embd = t;
        else if (i == 1 + 7 * m->n_layers) m->output = t;
        else layer_desc[i - 1] = t;
    }
    m->layers = layer_desc;
}

static const orc_qtensor* quant_at(const orc_model* m, int idx) {
    if (idx == 0) return &m->tok_embd;
    if (idx == (int)(1 + 7 * m->n_layers)) return &m->output;
    return &m->layers[idx - 1];
}

typedef void (*sink_fn)(void* ctx, const void* p, size_t n);

static void put_u32(sink_fn f, void* c, uint32_t v) {
    uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
    f(c, b, 4);
}

static void put_i64_array(sink_fn f, void* c, const int64_t* v, size_t n) {
    uint8_t b[4096];
    size_t k = 0;
    for (size_t i = 0; i < n; ++i) {
        uint64_t u = (uint64_t)v[i];
        for (int j = 0; j < 8; ++j) b[k++] = (uint8_t)(u >> (8 * j));
        if (k == sizeof b) { f(c, b, k); k = 0; }
    }
    if (k) f(c, b, k);
}

/* canonical DIM1 byte stream (model.cpp:217-249; README "File formats") */
static void emit_dim1(const orc_model* m, sink_fn f, void* c) {
    size_t cap = 2 + 9 * (size_t)m->n_layers + 2;
    dir_entry* d = (dir_entry*)malloc(cap * sizeof *d);
    size_t n = dir_build(m, d);
    f(c, "DIM1", 4);
    put_u32(f, c, 1);
    put_u32(f, c, m->n_layers);
    put_u32(f, c, m->d_model);
    put_u32(f, c, m->n_heads);
    put_u32(f, c, m->d_ffn);
    put_u32(f, c, m->vocab);
    put_u32(f, c, m->max_ctx);
    uint64_t tb;
    memcpy(&tb, &m->rope_theta, 8);
    uint8_t b8[8];
    for (int j = 0; j < 8; ++j) b8[j] = (uint8_t)(tb >> (8 * j));
    f(c, b8, 8);
    put_u32(f, c, (uint32_t)n);
    for (size_t i = 0; i < n; ++i) {
        uint16_t nl = (uint16_t)strlen(d[i].name);
        uint8_t b2[2] = {(uint8_t)nl, (uint8_t)(nl >> 8)};
        f(c, b2, 2);
        f(c, d[i].name, nl);
        put_u32(f, c, d[i].rows);
        put_u32(f, c, d[i].cols);
        f(c, &d[i].kind, 1);
    }
    for (size_t i = 0; i < n; ++i) {
        if (d[i].kind == 0) {
            const orc_qtensor* t = quant_at(m, d[i].idx);
            put_i64_array(f, c, t->scales, t->rows);
            f(c, t->data, (size_t)t->rows * t->cols);
        } else {
            put_i64_array(f, c, m->norms + (size_t)d[i].idx * m->d_model, m->d_model);
        }
    }
    free(d);
}

static void sink_hash(void* c, const void* p, size_t n) { orc_blake3_update((orc_blake3*)c, p, n); }
static void sink_count(void* c, const void* p, size_t n) { (void)p; *(uint64_t*)c += n; }
static void sink_copy(void* c, const void* p, size_t n) {
    uint8_t** dst = (uint8_t**)c;
    memcpy(*dst, p, n);
    *dst += n;
}

void orc_weight_hash(const orc_model* m, uint8_t out[32]) {
    orc_blake3* h = (orc_blake3*)malloc(sizeof *h);
    orc_blake3_init(h);
    emit_dim1(m, sink_hash, h);
    orc_blake3_final(h, out);
    free(h);
}

uint64_t orc_serialized_size(const orc_model* m) {
    uint64_t n = 0;
    emit_dim1(m, sink_count, &n);
    return n;
}

void orc_serialize(const orc_model* m, uint8_t* buf) { emit_dim1(m, sink_copy, &buf); }

/* ======================================================================= */
/* operators (proj/src/kernels.cpp)                                        */
/* ======================================================================= */

static int g_threads = 0;
void orc_set_threads(int n) { g_threads = n; }

void orc_dense(const orc_qtensor* w, const int64_t* x, int64_t* out) {
    /* acc = sum_j w[r,j]*x[j] in a wrapping 64-bit accumulator, then
     * (int128(acc) * scale) >> 16 (kernels.cpp:18-30) */
    long rows = (long)w->rows;
#ifdef _OPENMP
    int nt = g_threads > 0 ? g_threads : omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nt) if (rows >= 256)
#endif
    for (long r = 0; r < rows; ++r) {
        const int8_t* row = w->data + (size_t)r * w->cols;
        uint64_t acc = 0;
        for (uint32_t j = 0; j < w->cols; ++j) acc += (uint64_t)(int64_t)row[j] * (uint64_t)x[j];
        out[r] = (int64_t)(((i128)(int64_t)acc * w->scales[r]) >> 16);
    }
}

void orc_rmsnorm(const int64_t* x, const int64_t* g, uint32_t n, int64_t* out) {
    /* ms = (sum x^2 / n) >> 16 in int128; r = inv_sqrt(ms + 1);
     * out = mul16(mul16(x, r), g) (kernels.cpp:56-68) */
    u128 sum = 0;
    for (uint32_t i = 0; i < n; ++i) sum += (u128)((i128)x[i] * x[i]);
    int64_t ms = (int64_t)(((i128)sum / (i128)n) >> 16);
    int64_t r = orc_inv_sqrt(ms + 1);
    for (uint32_t i = 0; i < n; ++i) out[i] = orc_q16_mul(orc_q16_mul(x[i], r), g[i]);
}

void orc_rope_apply(int64_t* x, uint32_t half, const int64_t* c, const int64_t* s) {
    /* paired halves (kernels.cpp:70-82) */
    for (uint32_t k = 0; k < half; ++k) {
        int64_t a = x[k], b = x[k + half];
        x[k] = (int64_t)((uint64_t)orc_q16_mul(a, c[k]) - (uint64_t)orc_q16_mul(b, s[k]));
        x[k + half] = (int64_t)((uint64_t)orc_q16_mul(a, s[k]) + (uint64_t)orc_q16_mul(b, c[k]));
    }
}

void orc_softmax(const int64_t* s, uint32_t n, int64_t* p) {
    /* LUT weights against the max, truncating division (kernels.cpp:90-107) */
    int64_t m = s[0];
    for (uint32_t i = 1; i < n; ++i) if (s[i] > m) m = s[i];
    int64_t* w = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t total = 0;
    for (uint32_t i = 0; i < n; ++i) {
        int64_t d = (int64_t)((uint64_t)m - (uint64_t)s[i]);
        if (d > 8 * ONE) d = 8 * ONE;
        w[i] = orc_exp_neg(d);
        total += w[i];
    }
    for (uint32_t i = 0; i < n; ++i) p[i] = (w[i] << 16) / total;
    free(w);
}

void orc_attention_step(const int64_t* q, const int64_t* k, const int64_t* v, uint32_t H,
                        uint32_t dh, uint32_t max_ctx, int64_t* kc, int64_t* vc, uint32_t pos,
                        const int64_t* rope_cos, const int64_t* rope_sin, int64_t* out) {
    /* per head: RoPE q,k at pos; append k,v; scores = mul16(int128 dot >> 16,
     * inv_sqrt(dh)); softmax; out_j = sum_t mul16(p_t, v_tj) (kernels.cpp:117-177) */
    (void)max_ctx;
    const size_t D = (size_t)H * dh;
    const uint32_t half = dh / 2;
    const int64_t inv_scale = orc_inv_sqrt((int64_t)dh * ONE);
    const int64_t* cr = rope_cos + (size_t)pos * half;
    const int64_t* sr = rope_sin + (size_t)pos * half;
    int64_t* qh = (int64_t*)malloc(sizeof(int64_t) * dh);
    int64_t* scores = (int64_t*)malloc(sizeof(int64_t) * (pos + 1));
    int64_t* p = (int64_t*)malloc(sizeof(int64_t) * (pos + 1));
    for (uint32_t h = 0; h < H; ++h) {
        memcpy(qh, q + (size_t)h * dh, sizeof(int64_t) * dh);
        orc_rope_apply(qh, half, cr, sr);
        int64_t* krow = kc + (size_t)pos * D + (size_t)h * dh;
        memcpy(krow, k + (size_t)h * dh, sizeof(int64_t) * dh);
        orc_rope_apply(krow, half, cr, sr);
        memcpy(vc + (size_t)pos * D + (size_t)h * dh, v + (size_t)h * dh, sizeof(int64_t) * dh);
        for (uint32_t t = 0; t <= pos; ++t) {
            const int64_t* kt = kc + (size_t)t * D + (size_t)h * dh;
            u128 dot = 0;
            for (uint32_t j = 0; j < dh; ++j) dot += (u128)((i128)qh[j] * kt[j]);
            scores[t] = orc_q16_mul((int64_t)((i128)dot >> 16), inv_scale);
        }
        orc_softmax(scores, pos + 1, p);
        for (uint32_t j = 0; j < dh; ++j) {
            uint64_t acc = 0;
            for (uint32_t t = 0; t <= pos; ++t)
                acc += (uint64_t)orc_q16_mul(p[t], vc[(size_t)t * D + (size_t)h * dh + j]);
            out[(size_t)h * dh + j] = (int64_t)acc;
        }
    }
    free(qh);
    free(scores);
    free(p);
}

void orc_ffn(const orc_qtensor* gate, const orc_qtensor* up, const orc_qtensor* down,
             const int64_t* x, int64_t* out) {
    /* h = mul16(silu(gate x), up x); out = down h (kernels.cpp:179-190) */
    int64_t* g = (int64_t*)malloc(sizeof(int64_t) * gate->rows);
    int64_t* u = (int64_t*)malloc(sizeof(int64_t) * up->rows);
    orc_dense(gate, x, g);
    orc_dense(up, x, u);
    for (uint32_t i = 0; i < gate->rows; ++i) g[i] = orc_q16_mul(orc_silu(g[i]), u[i]);
    orc_dense(down, g, out);
    free(g);
    free(u);
}

static void residual_clamp(int64_t* x, const int64_t* y, uint32_t n) {
    /* kernels.cpp:192-200 */
    for (uint32_t i = 0; i < n; ++i) {
        int64_t s = (int64_t)((uint64_t)x[i] + (uint64_t)y[i]);
        x[i] = s > ACT_CLAMP ? ACT_CLAMP : (s < -ACT_CLAMP ? -ACT_CLAMP : s);
    }
}

/* ======================================================================= */
/* engine (proj/src/engine.cpp)                                            */
/* ======================================================================= */

struct orc_session {
    const orc_model* m;
    uint32_t len, cap;
    int64_t* rope_cos;
    int64_t* rope_sin;
    int64_t** kc; /* per layer [cap][D] */
    int64_t** vc;
};

orc_session* orc_session_new(const orc_model* m) {
    orc_session* s = (orc_session*)calloc(1, sizeof *s);
    s->m = m;
    uint32_t dh = m->d_model / m->n_heads;
    s->rope_cos = (int64_t*)malloc(sizeof(int64_t) * (size_t)m->max_ctx * (dh / 2));
    s->rope_sin = (int64_t*)malloc(sizeof(int64_t) * (size_t)m->max_ctx * (dh / 2));
    orc_rope_tables(m->rope_theta, dh, m->max_ctx, s->rope_cos, s->rope_sin);
    s->kc = (int64_t**)calloc(m->n_layers, sizeof(int64_t*));
    s->vc = (int64_t**)calloc(m->n_layers, sizeof(int64_t*));
    return s;
}

void orc_session_free(orc_session* s) {
    if (!s) return;
    for (uint32_t l = 0; l < s->m->n_layers; ++l) {
        free(s->kc[l]);
        free(s->vc[l]);
    }
    free(s->kc);
    free(s->vc);
    free(s->rope_cos);
    free(s->rope_sin);
    free(s);
}

static void session_reserve(orc_session* s, uint32_t need) {
    if (need <= s->cap) return;
    uint32_t cap = s->cap ? s->cap : 16;
    while (cap < need) cap *= 2;
    if (cap > s->m->max_ctx) cap = s->m->max_ctx;
    size_t bytes = sizeof(int64_t) * (size_t)cap * s->m->d_model;
    for (uint32_t l = 0; l < s->m->n_layers; ++l) {
        s->kc[l] = (int64_t*)realloc(s->kc[l], bytes);
        s->vc[l] = (int64_t*)realloc(s->vc[l], bytes);
    }
    s->cap = cap;
}

int orc_session_forward(orc_session* s, uint32_t token, uint32_t pos, int64_t* logits) {
    const orc_model* m = s->m;
    if (token >= m->vocab) return -1;
    if (pos >= m->max_ctx) return -2;
    if (pos != s->len) return -3;
    session_reserve(s, pos + 1);
    const uint32_t D = m->d_model, F = m->d_ffn, dh = D / m->n_heads;
    int64_t* x = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* xn = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* q = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* k = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* v = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* att = (int64_t*)malloc(sizeof(int64_t) * D);
    int64_t* y = (int64_t*)malloc(sizeof(int64_t) * D);
    (void)F;
    /* embed_token: int64(w) * scale, no shift (engine.cpp:10-19) */
    const int8_t* er = m->tok_embd.data + (size_t)token * D;
    int64_t es = m->tok_embd.scales[token];
    for (uint32_t j = 0; j < D; ++j) x[j] = (int64_t)((uint64_t)(int64_t)er[j] * (uint64_t)es);
    for (uint32_t l = 0; l < m->n_layers; ++l) {
        const orc_qtensor* lw = m->layers + 7 * (size_t)l;
        orc_rmsnorm(x, m->norms + (size_t)(2 * l) * D, D, xn);
        orc_dense(&lw[0], xn, q);
        orc_dense(&lw[1], xn, k);
        orc_dense(&lw[2], xn, v);
        orc_attention_step(q, k, v, m->n_heads, dh, m->max_ctx, s->kc[l], s->vc[l], pos,
                           s->rope_cos, s->rope_sin, att);
        orc_dense(&lw[3], att, y);
        residual_clamp(x, y, D);
        orc_rmsnorm(x, m->norms + (size_t)(2 * l + 1) * D, D, xn);
        orc_ffn(&lw[4], &lw[5], &lw[6], xn, y);
        residual_clamp(x, y, D);
    }
    s->len = pos + 1;
    if (logits) {
        orc_rmsnorm(x, m->norms + (size_t)(2 * m->n_layers) * D, D, xn);
        orc_dense(&m->output, xn, logits);
    }
    free(x); free(xn); free(q); free(k); free(v); free(att); free(y);
    return 0;
}

uint32_t orc_select_greedy(const int64_t* logits, uint32_t n) {
    /* strict '>' keeps the lowest index on ties (engine.cpp:113-120) */
    uint32_t best = 0;
    for (uint32_t i = 1; i < n; ++i) if (logits[i] > logits[best]) best = i;
    return best;
}

void orc_hash_tokens(const uint32_t* ids, size_t n, uint8_t out[32]) {
    orc_blake3 h;
    orc_blake3_init(&h);
    for (size_t i = 0; i < n; ++i) {
        uint8_t le[4] = {(uint8_t)ids[i], (uint8_t)(ids[i] >> 8), (uint8_t)(ids[i] >> 16),
                         (uint8_t)(ids[i] >> 24)};
        orc_blake3_update(&h, le, 4);
    }
    orc_blake3_final(&h, out);
}

int orc_generate_greedy(const orc_model* m, const uint32_t* prompt, uint32_t n_prompt,
                        uint32_t max_new, uint32_t* tokens_out, uint8_t hash_out[32],
                        int64_t* logits_out) {
    /* check_generate_pre (engine.cpp:21-29), then run_generation (:31-54) */
    if (n_prompt == 0) return -4;
    if ((uint64_t)n_prompt + max_new > m->max_ctx) return -2;
    for (uint32_t i = 0; i < n_prompt; ++i) if (prompt[i] >= m->vocab) return -1;
    orc_session* s = orc_session_new(m);
    int64_t* logits = (int64_t*)malloc(sizeof(int64_t) * m->vocab);
    uint32_t pos = 0;
    for (uint32_t i = 0; i < n_prompt; ++i, ++pos)
        orc_session_forward(s, prompt[i], pos, i + 1 == n_prompt ? logits : NULL);
    for (uint32_t n = 0; n < max_new; ++n) {
        uint32_t next = orc_select_greedy(logits, m->vocab);
        tokens_out[n] = next;
        if (logits_out) memcpy(logits_out + (size_t)n * m->vocab, logits, sizeof(int64_t) * m->vocab);
        if (n + 1 == max_new) break;
        orc_session_forward(s, next, pos++, logits);
    }
    orc_hash_tokens(tokens_out, max_new, hash_out);
    free(logits);
    orc_session_free(s);
    return 0;
}
