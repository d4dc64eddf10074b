/*
 * dim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference engine's integer forward pass
 * (/root/reference/proj, the C++20 `dim` engine). It is the parity checker
 * for the B200 engine: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * library (paper_2603_24904_b200/libdimg.so) never links or calls it.
 *
 * Every function cites the reference file:line whose behaviour it restates.
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   - the reference's own known-answer tests (proj/tests/test_*.cpp), and
 *   - golden vectors produced by the reference itself, compiled from its
 *     sources by oracle/Makefile into oracle/_ref/libdimref.so
 *     (tests/golden/make_golden.py).
 */
#ifndef DIM_ORACLE_H
#define DIM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- hashes / RNG ------------------------------------------------------ */

/* BLAKE3 plain hash, 32-byte output (proj/src/blake3.cpp:126-193). */
typedef struct {
    uint32_t cv[8];          /* chaining value of the current chunk */
    uint64_t chunk_counter;
    uint8_t block[64];
    uint32_t block_len;
    uint32_t blocks_done;    /* blocks compressed in the current chunk */
    uint32_t stack[54][8];
    uint32_t stack_len;
} orc_blake3;

void orc_blake3_init(orc_blake3* h);
void orc_blake3_update(orc_blake3* h, const void* data, size_t len);
void orc_blake3_final(const orc_blake3* h, uint8_t out[32]);
void orc_blake3_oneshot(const void* data, size_t len, uint8_t out[32]);

/* ChaCha20 block, RFC 8439 layout (proj/src/chacha20.cpp:20-46). */
void orc_chacha20_block(const uint32_t key[8], const uint32_t nonce[3], uint32_t counter,
                        uint8_t out[64]);

/* Keystream RNG keyed by BLAKE3(seed LE) (proj/src/chacha20.cpp:48-96). */
typedef struct {
    uint32_t key[8];
    uint32_t counter;
    uint8_t buf[64];
    uint32_t pos;
} orc_rng;

void orc_rng_from_seed(orc_rng* r, uint64_t seed);
void orc_rng_from_key(orc_rng* r, const uint8_t key[32]);
uint8_t orc_rng_u8(orc_rng* r);
uint32_t orc_rng_u32(orc_rng* r);
uint64_t orc_rng_u64(orc_rng* r);
int8_t orc_rng_weight(orc_rng* r);

/* ---- Q16 primitives (proj/src/q16.cpp) --------------------------------- */

int64_t orc_q16_from_ratio(int64_t num, int64_t den); /* q16.cpp:13-24,47-50 */
int64_t orc_q16_mul(int64_t a, int64_t b);             /* q16.hpp:28-30 */
int64_t orc_inv_sqrt(int64_t x);                       /* q16.cpp:56-68 (x>0) */
int64_t orc_invsqrt_seed(int b);                       /* q16.cpp:28-43 */
int64_t orc_exp_entry(int i);                          /* q16.cpp:70-79 */
int64_t orc_exp_neg(int64_t t);                        /* q16.cpp:81-92 (0<=t<=8*ONE) */
int orc_domain_error(void);                             /* exp_neg_lut domain_error since last call */
int64_t orc_sigmoid(int64_t x);                        /* q16.cpp:94-101 */
int64_t orc_silu(int64_t x);                           /* q16.cpp:103-105 */
/* RoPE tables [max_ctx][d_head/2] (proj/src/rope.cpp:17-39). */
void orc_rope_tables(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out,
                     int64_t* sin_out);

/* ---- model ------------------------------------------------------------- */

typedef struct {
    uint32_t rows, cols;
    const int8_t* data;    /* rows*cols row-major */
    const int64_t* scales; /* rows, Q16 raw */
} orc_qtensor;

/* Mirrors ModelConfig + the fixed tensor directory (proj/include/dim/model.hpp:15-29,
 * proj/src/model.cpp:41-61). layers = 7 tensors per layer in directory order
 * (wq, wk, wv, wo, w_gate, w_up, w_down). norms = (2L+1)*d_model values in
 * directory order (attn_norm[0], ffn_norm[0], ..., final_norm). */
typedef struct {
    uint32_t n_layers, d_model, n_heads, d_ffn, vocab, max_ctx;
    double rope_theta;
    orc_qtensor tok_embd;
    orc_qtensor output;
    const orc_qtensor* layers;
    const int64_t* norms;
} orc_model;

/* Total int8 weights / scale rows of a toy model in directory order. */
uint64_t orc_model_weight_count(const orc_model* cfg_only);
uint64_t orc_model_scale_count(const orc_model* cfg_only);

/* gen_toy_model's stream (proj/src/model.cpp:189-215): fills `weights` and
 * `scales` (directory order, contiguous) from ChaCha20Rng(seed). */
void orc_gen_toy(uint64_t seed, const orc_model* cfg_only, int8_t* weights, int64_t* scales);

/* Binds tensors of a contiguous directory-order weight/scale buffer into m
 * (m->layers must point to 7*n_layers writable descriptors). norms must be
 * provided by the caller. */
void orc_bind(orc_model* m, orc_qtensor* layer_desc, const int8_t* weights,
              const int64_t* scales);

/* BLAKE3 of the canonical DIM1 serialization (proj/src/model.cpp:217-249),
 * streamed (the container is never materialised). */
void orc_weight_hash(const orc_model* m, uint8_t out[32]);
/* Writes the DIM1 serialization into buf (size from orc_serialized_size). */
uint64_t orc_serialized_size(const orc_model* m);
void orc_serialize(const orc_model* m, uint8_t* buf);

/* ---- operators (proj/src/kernels.cpp) ---------------------------------- */

void orc_dense(const orc_qtensor* w, const int64_t* x, int64_t* out);          /* :18-30 */
void orc_rmsnorm(const int64_t* x, const int64_t* g, uint32_t n, int64_t* out); /* :56-68 */
void orc_rope_apply(int64_t* x, uint32_t half, const int64_t* cos_row,
                    const int64_t* sin_row);                                      /* :70-82 */
void orc_softmax(const int64_t* s, uint32_t n, int64_t* p);                       /* :90-107 */
/* attention_step for one layer (:117-177). kcache/vcache: position-major
 * [max_ctx][n_heads*dh] (the reference keeps one strip per head; the index
 * map differs, the values do not). */
void orc_attention_step(const int64_t* q, const int64_t* k, const int64_t* v, uint32_t n_heads,
                        uint32_t dh, uint32_t max_ctx, int64_t* kcache, int64_t* vcache,
                        uint32_t pos, const int64_t* rope_cos, const int64_t* rope_sin,
                        int64_t* out);
void orc_ffn(const orc_qtensor* gate, const orc_qtensor* up, const orc_qtensor* down,
             const int64_t* x, int64_t* out);                                     /* :179-190 */

/* ---- engine (proj/src/engine.cpp) -------------------------------------- */

typedef struct orc_session orc_session;
orc_session* orc_session_new(const orc_model* m); /* engine.cpp:58-78 */
void orc_session_free(orc_session* s);
/* forward(token, pos): returns 0 or a negative code mirroring the
 * reference's exceptions: -1 out_of_range, -2 ContextOverflow, -3 logic_error.
 * engine.cpp:80-102. logits may be NULL to skip the lm_head. */
int orc_session_forward(orc_session* s, uint32_t token, uint32_t pos, int64_t* logits);
uint32_t orc_select_greedy(const int64_t* logits, uint32_t n); /* engine.cpp:113-120 */
void orc_hash_tokens(const uint32_t* ids, size_t n, uint8_t out[32]); /* engine.cpp:104-111 */
/* run_generation with greedy select (engine.cpp:31-54,142-147). logits_out may
 * be NULL; else max_new*vocab int64. Returns 0, -4 invalid_argument (empty
 * prompt), -2 ContextOverflow, -1 out_of_range. */
int orc_generate_greedy(const orc_model* m, const uint32_t* prompt, uint32_t n_prompt,
                        uint32_t max_new, uint32_t* tokens_out, uint8_t hash_out[32],
                        int64_t* logits_out);

/* Worker threads used by orc_dense (OpenMP). Integer sums are exact in any
 * grouping, so this never changes a bit. */
void orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
