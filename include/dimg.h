/*
 * dimg.h -- C ABI of the B200-native integer transformer engine.
 *
 * The reference (`dim`, /root/reference/proj) is a C++20 library whose hot
 * path is InferenceSession::forward / generate_greedy
 * (proj/include/dim/engine.hpp:41-80). It has no FFI; this header is the
 * drop-in boundary a binding (ctypes, cgo, JNI, or the C++ wrapper in
 * paper_2603_24904_b200/csrc/include/dimg/dim.hpp) links against. Plain
 * pointers and sizes only; nothing throws across it. Every function returns a
 * dimg_status; dimg_last_error() gives the thread-local message.
 *
 * Status codes map one-to-one onto the reference's exception types
 * (SURVEY.md §8b "Errors"):
 *   DIMG_EINVAL  std::invalid_argument  (empty prompt engine.cpp:22, bad config model.cpp:95-109)
 *   DIMG_ERANGE  std::out_of_range      (token >= vocab engine.cpp:27,81)
 *   DIMG_ELOGIC  std::logic_error       (pos != cache length engine.cpp:83)
 *   DIMG_ECTX    dim::ContextOverflow   (engine.cpp:24,82)
 *   DIMG_ELENGTH std::length_error      (attention cache overflow kernels.cpp:126)
 *   DIMG_EDOMAIN std::domain_error      (inv_sqrt of a non-positive value q16.cpp:57)
 *   DIMG_EPARSE  dim::ParseError        (kind via dimg_last_parse_kind, serial.hpp:10-15)
 */
#ifndef DIMG_H
#define DIMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DIMG_OK = 0,
    DIMG_EINVAL = 1,
    DIMG_ERANGE = 2,
    DIMG_ELOGIC = 3,
    DIMG_ECTX = 4,
    DIMG_ELENGTH = 5,
    DIMG_EDOMAIN = 6,
    DIMG_EPARSE = 7,
    DIMG_ECUDA = 8,
    DIMG_ENCCL = 9,
    DIMG_ENOMEM = 10,
    DIMG_EIO = 11,
} dimg_status;

/* ParseError::Kind (proj/include/dim/serial.hpp:11) */
typedef enum { DIMG_PARSE_BAD_MAGIC = 0, DIMG_PARSE_BAD_VERSION = 1, DIMG_PARSE_TRUNCATED = 2,
               DIMG_PARSE_INVARIANT = 3 } dimg_parse_kind;

const char* dimg_last_error(void);
int dimg_last_parse_kind(void);
const char* dimg_version(void);

/* ModelConfig (proj/include/dim/model.hpp:15-29). */
typedef struct {
    uint32_t n_layers, d_model, n_heads, d_ffn, vocab, max_ctx;
    double rope_theta;
} dimg_config;

/* ModelConfig::validate (proj/src/model.cpp:95-109). */
dimg_status dimg_config_validate(const dimg_config* cfg);

/* QuantTensor (proj/include/dim/model.hpp:33-41): host pointers, borrowed. */
typedef struct {
    uint32_t rows, cols;
    const int8_t* data;    /* rows*cols row-major, values in [-127,127] */
    const int64_t* scales; /* rows, Q16 raw, > 0 */
} dimg_qtensor;

/* A model as plain host buffers, in the reference's directory order
 * (proj/src/model.cpp:41-61). layers: 7 per layer (wq wk wv wo w_gate w_up
 * w_down). norms: (2L+1)*d_model (attn_norm[l], ffn_norm[l], ..., final_norm).
 * rope_cos/rope_sin: optional imported RTAB tables [max_ctx][d_head/2]
 * (InferenceSession's imported_tables, engine.hpp:43-44); NULL = build them
 * (proj/src/rope.cpp:17-39). */
typedef struct {
    dimg_config cfg;
    dimg_qtensor tok_embd;
    dimg_qtensor output;
    const dimg_qtensor* layers;
    const int64_t* norms;
    const int64_t* rope_cos;
    const int64_t* rope_sin;
    uint32_t rope_max_ctx; /* rows of the imported tables (>= cfg.max_ctx) */
} dimg_model_desc;

/* ------------------------------------------------------------------------ */
/* Host side: hashes, RNG, container (the reference's L0/L1, kept on host)   */
/* ------------------------------------------------------------------------ */

/* BLAKE3 (proj/src/blake3.cpp); multi-threaded over 1 MiB subtrees when large. */
dimg_status dimg_blake3(const void* data, size_t len, uint8_t out[32]);
/* hash_token_ids: BLAKE3 over u32-LE ids (proj/src/engine.cpp:104-111). */
dimg_status dimg_hash_token_ids(const uint32_t* ids, size_t n, uint8_t out[32]);
/* select_greedy: argmax, lowest index on ties (proj/src/engine.cpp:113-120). */
dimg_status dimg_select_greedy(const int64_t* logits, size_t n, uint32_t* out);
/* prompt[i] = ChaCha20Rng(seed).next_u32() % vocab (acceptance.cpp:80-82). */
dimg_status dimg_prompt_from_seed(uint64_t seed, uint32_t vocab, uint32_t n, uint32_t* out);
/* parse_prompt (proj/tools/dim_cli.cpp:56-70): bytes != NULL maps each byte
 * to an id; else comma-separated ids. Writes up to cap ids, *n = count. */
dimg_status dimg_parse_prompt(const char* csv, const char* bytes, uint32_t* out, size_t cap,
                              size_t* n);
/* RoPE tables [max_ctx][d_head/2] in Q16 (proj/src/rope.cpp:17-39). */
dimg_status dimg_rope_tables(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out,
                             int64_t* sin_out);
/* RTAB, the reference's byte-exact RoPE table artifact (serialize_rope_tables /
 * deserialize_rope_tables / save_rope_tables / load_rope_tables,
 * proj/src/rope.cpp:41-93, proj/include/dim/rope.hpp:28-39): "RTAB", u32
 * version 1, u32 max_ctx, u32 half_dim, f64 theta_base, cos then sin as i64,
 * little-endian. serialize with out == NULL: *n = the size. deserialize with
 * cos_out == sin_out == NULL: header only (dims and theta, fully validated);
 * errors are DIMG_EPARSE with the reference's ParseError kind (bad magic, bad
 * version, truncated, invariant = empty dims or trailing bytes). The tables
 * feed dimg_model_desc.rope_cos/rope_sin. save/load: DIMG_EIO when the file
 * cannot be opened/written; load returns the file's bytes (out == NULL: size). */
dimg_status dimg_rtab_serialize(double theta, uint32_t max_ctx, uint32_t half_dim, const int64_t* cos_raw,
                                const int64_t* sin_raw, uint8_t* out, size_t cap, size_t* n);
dimg_status dimg_rtab_deserialize(const uint8_t* bytes, size_t n, uint32_t* max_ctx, uint32_t* half_dim,
                                  double* theta, int64_t* cos_out, int64_t* sin_out, size_t cap_cells);
dimg_status dimg_rtab_save(const char* path, double theta, uint32_t max_ctx, uint32_t half_dim,
                           const int64_t* cos_raw, const int64_t* sin_raw);
dimg_status dimg_rtab_load(const char* path, uint8_t* out, size_t cap, size_t* n);
/* The 257-entry exp LUT (q16.cpp:70-79) and 64 Q48 inv-sqrt seeds (:28-43). */
dimg_status dimg_exp_lut(int64_t out[257]);
dimg_status dimg_invsqrt_seeds(int64_t out[64]);
/* inv_sqrt_q16 (proj/src/q16.cpp:56-68) as the device kernels compute it
 * (kernels/q16.cuh), on the host: parity checks of its 64-bit fast path. */
dimg_status dimg_inv_sqrt_q16(int64_t x, int64_t* out);

/* Host model container: the canonical DIM1 bytes (ModelFile::bytes) plus
 * views into them (proj/include/dim/model.hpp:50-60). */
typedef struct dimg_host_model dimg_host_model;
/* gen_toy_model (proj/src/model.cpp:189-215); threads <= 0 = all cores. */
dimg_status dimg_host_model_gen_toy(uint64_t seed, const dimg_config* cfg, int threads,
                                    dimg_host_model** out);
/* gen_toy_model with its weight stream (ChaCha20 keystream, 0xFF rejected)
 * synthesised on GPU `device` and copied into the container: the same bytes. */
dimg_status dimg_host_model_gen_toy_gpu(int device, uint64_t seed, const dimg_config* cfg, dimg_host_model** out);
/* deserialize (proj/src/model.cpp:251-312) / load_model (:332-334). */
dimg_status dimg_host_model_from_bytes(const uint8_t* bytes, size_t n, dimg_host_model** out);
dimg_status dimg_host_model_load(const char* path, dimg_host_model** out);
dimg_status dimg_host_model_save(const dimg_host_model* m, const char* path);
/* Builds a container from plain buffers (serialize, model.cpp:217-249). */
dimg_status dimg_host_model_from_desc(const dimg_model_desc* d, dimg_host_model** out);
dimg_status dimg_host_model_bytes(const dimg_host_model* m, const uint8_t** bytes, size_t* n);
dimg_status dimg_host_model_weight_hash(const dimg_host_model* m, uint8_t out[32]);
dimg_status dimg_host_model_desc(const dimg_host_model* m, dimg_model_desc* out);
dimg_status dimg_host_model_free(dimg_host_model* m);

/* ------------------------------------------------------------------------ */
/* Device side (sm_100a)                                                     */
/* ------------------------------------------------------------------------ */

dimg_status dimg_device_count(int* n);

/* Uploads a model to one GPU, re-laid out for the decode GEMVs (rows padded
 * to 16 B, gate/up interleaved, q/k/v fused). tp_rank/tp_size shard it
 * Megatron-style; pass 0/1 for a whole model. */
typedef struct dimg_model dimg_model;
dimg_status dimg_model_upload(int device, const dimg_model_desc* desc, int tp_rank, int tp_size,
                              dimg_model** out);
dimg_status dimg_model_free(dimg_model* m);
dimg_status dimg_model_bytes_on_device(const dimg_model* m, uint64_t* bytes);

/* InferenceSession (engine.hpp:41-57): owns one sequence's KV cache on the
 * device; single writer. keep_logits_cap = how many logits vectors a
 * generate call may keep (EngineOptions::keep_logits). */
typedef struct dimg_session dimg_session;
dimg_status dimg_session_create(dimg_model* m, uint32_t keep_logits_cap, dimg_session** out);
dimg_status dimg_session_free(dimg_session* s);
dimg_status dimg_session_reset(dimg_session* s);
dimg_status dimg_session_len(const dimg_session* s, uint32_t* len);
/* forward(token, pos) -> logits (engine.cpp:80-102); logits may be NULL. */
dimg_status dimg_session_forward(dimg_session* s, uint32_t token, uint32_t pos, int64_t* logits);
/* generate_greedy (engine.cpp:31-54,142-147) on a reset session: prompt and
 * results in HOST memory. tokens_out: max_new ids; hash_out: BLAKE3 of them;
 * logits_out: NULL or max_new*vocab (the logits used for each selection). */
dimg_status dimg_generate_greedy(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt,
                                 uint32_t max_new, uint32_t* tokens_out, uint8_t hash_out[32],
                                 int64_t* logits_out);
/* generate_greedy for n_seqs independent sequences stepped together (C5):
 * prompts concatenated (p_lens[n_seqs] tokens each), tokens_out
 * [n_seqs][max_new], hashes_out [n_seqs][32] (nullable). Bit-identical to
 * n_seqs separate dimg_generate_greedy calls. *path (nullable) = 1 if the
 * tensor-core batch path produced them, 0 if the exact per-sequence path. */
dimg_status dimg_generate_greedy_batch(dimg_model* m, uint32_t n_seqs, const uint32_t* prompts,
                                       const uint32_t* p_lens, uint32_t max_new, uint32_t* tokens_out,
                                       uint8_t* hashes_out, uint32_t* path);

/* Device-resident stepping (bench / advanced callers). The prompt is staged
 * with dimg_session_begin; each decode step forwards the newest token and
 * appends its greedy successor on the device. Nothing is copied to the host
 * until dimg_session_tokens. */
dimg_status dimg_session_begin(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt,
                               uint32_t max_new);
dimg_status dimg_session_prefill(dimg_session* s);          /* all but the last prompt token */
dimg_status dimg_session_decode(dimg_session* s, uint32_t n_steps);
dimg_status dimg_session_sync(dimg_session* s);
dimg_status dimg_session_tokens(dimg_session* s, uint32_t* out, uint32_t n_generated);
/* cudaStream_t the session launches on (for CUDA-event timing by callers). */
dimg_status dimg_session_stream(dimg_session* s, void** stream);
/* Times n decode steps with CUDA events on the session stream. */
dimg_status dimg_session_time_decode(dimg_session* s, uint32_t n_steps, float* ms);
/* The prefill of the begun prompt between CUDA events; *tensor_cores = 1 if
 * it ran on the tensor-core prefill path (else the decode kernel). */
dimg_status dimg_session_time_prefill(dimg_session* s, float* ms, uint32_t* tensor_cores);
/* Replays one kernel class n times between CUDA events on the session
 * stream (layers cycled so weights stream from HBM): which = 0 QKV GEMV,
 * 1 WO, 2 GATE/UP, 3 DOWN, 4 LM_HEAD. Returns the mean launch time and the
 * algorithmic bytes of one launch (roofline numerator). */
dimg_status dimg_session_time_kernel(dimg_session* s, int which, uint32_t n, float* ms_per_launch,
                                     uint64_t* bytes_per_launch);
/* Tracing: n decode steps; out[DIMG_TRACE_WORDS*i + 0..3] = %globaltimer (ns)
 * of CTA 0 at stage i's start, after its prologue, after its chunk loop and
 * before its grid barrier; [4..7] = clock64 of prologue / attention sub-steps,
 * [8] = clock64 at the stage start, [9..31] = finer clock64 stamps of the
 * attention stage. cap stages recorded. */
#define DIMG_TRACE_WORDS 32
dimg_status dimg_session_trace(dimg_session* s, uint32_t n_steps, uint64_t* out, uint32_t cap);
/* Hand-off skew: n decode steps with every CTA stamping %globaltimer at the end
 * of each GEMV stage's prologue and of its chunk loop:
 * out[(i * grid + cta) * 2 + {0, 1}] for the first cap stages (grid = SMs). */
dimg_status dimg_session_trace_all(dimg_session* s, uint32_t n_steps, uint64_t* out, uint32_t cap);
/* Kernel launches per decode step / per prefill step (for the bench claim). */
dimg_status dimg_session_launches(const dimg_session* s, uint32_t* per_decode,
                                  uint32_t* per_prefill);

/* Counters: [0] GEMV CTAs that needed the 8-limb (full int64) path,
 * [1] device-side error bits (1: inv_sqrt of ms+1 <= 0, 4: barrier timeout),
 * [2] attention parts that read the int64 KV cache (a head holding values
 * beyond int32), [3] prompts prefilled on the tensor cores (low 32 bits) and
 * tensor-core prefills redone on the exact decode path (high 32 bits). */
dimg_status dimg_session_stats(dimg_session* s, uint64_t out[4]);

/* ---- tensor parallelism (BASELINE config C4) ----
 * One model sharded Megatron-style over tp_size ranks: q/k/v and the FFN
 * gate/up rows and lm_head vocab rows column-parallel, wo and w_down
 * row-parallel (input columns); the PRE-SCALE int64 accumulators of wo and
 * w_down (dense_forward's acc before (acc*s)>>16, proj/src/kernels.cpp:18-30)
 * are summed over the ranks (uint64: wrapping, order-free -- the reference's
 * chunk invariance, kernels.cpp:32-50) and the rescale, residual and clamp
 * run on every rank; the greedy pick gathers every rank's (max, lowest index)
 * pair (select_greedy, engine.cpp:113-120). Tokens and hashes are identical
 * to the single-GPU engine and the reference at every tp_size.
 * Backends:
 *   DIMG_TP_NCCL   this process is rank tp_rank (one process per GPU,
 *                  `device` its GPU); nccl_id from rank 0's
 *                  dimg_nccl_unique_id, distributed by the caller.
 *   DIMG_TP_LOCAL  all tp_size shards on `device` in this process, the sums
 *                  done by kernels (testing the sharded kernels on one GPU).
 *   (both: a chain of per-stage GEMV kernels + collectives per step)
 *   DIMG_TP_FUSED_IPC    this process is rank tp_rank; every rank runs the
 *                  persistent decode kernel on its shard and the sums happen
 *                  INSIDE it: the wo / w_down epilogues store their rows'
 *                  partials straight into every peer's inbox over NVLink
 *                  (peer memory from CUDA IPC handles) and poll their own.
 *                  After create: dimg_tp_exchange_handle on every rank, the
 *                  tp_size handles gathered by the caller, dimg_tp_connect.
 *   DIMG_TP_FUSED_LOCAL  the same kernel program for all tp_size shards on
 *                  `device`: one cooperative launch whose CTAs are split
 *                  between the ranks, exchanging through device memory (the
 *                  one-GPU test of the fused path; tp_size <= 8).
 * tp_size must divide n_heads. keep_logits_cap: logits vectors a generate
 * call may return (not with DIMG_TP_FUSED_IPC). */
typedef struct dimg_tp dimg_tp;
typedef enum { DIMG_TP_LOCAL = 0, DIMG_TP_NCCL = 1, DIMG_TP_FUSED_LOCAL = 2, DIMG_TP_FUSED_IPC = 3 } dimg_tp_backend;
dimg_status dimg_nccl_unique_id(uint8_t id[128]);
dimg_status dimg_tp_create(int device, const dimg_model_desc* desc, int backend, int tp_rank, int tp_size,
                           const uint8_t nccl_id[128], uint32_t keep_logits_cap, dimg_tp** out);
dimg_status dimg_tp_free(dimg_tp* t);
/* generate_greedy (engine.cpp:31-54,142-147) on the sharded model; host
 * buffers as dimg_generate_greedy; every rank returns the same tokens. */
dimg_status dimg_tp_generate_greedy(dimg_tp* t, const uint32_t* prompt, uint32_t n_prompt, uint32_t max_new,
                                    uint32_t* tokens_out, uint8_t hash_out[32], int64_t* logits_out);
/* The prompt steps, then n_steps decode steps between CUDA events on the
 * group's stream; the tokens through dimg_tp_tokens. */
dimg_status dimg_tp_time_decode(dimg_tp* t, const uint32_t* prompt, uint32_t n_prompt, uint32_t n_steps,
                                float* ms);
dimg_status dimg_tp_tokens(dimg_tp* t, uint32_t* out, uint32_t n_generated);
dimg_status dimg_tp_stream(dimg_tp* t, void** stream);
/* Device bytes of this process's shards; kernel launches + collectives per
 * decode step (after the first generation). */
dimg_status dimg_tp_info(dimg_tp* t, uint64_t* weight_bytes, uint64_t* launches_per_step);
/* DIMG_TP_FUSED_IPC: this rank's exchange-block handle (a cudaIpcMemHandle_t,
 * 64 bytes), and the group's handles in rank order (tp_size x 64 bytes) to
 * map the peers' blocks; generation needs a connected group. */
dimg_status dimg_tp_exchange_handle(dimg_tp* t, uint8_t handle[64]);
dimg_status dimg_tp_connect(dimg_tp* t, const uint8_t* handles);

/* ---- operator-level exports (host buffers in/out) for unit parity with
 *      proj/src/kernels.cpp; they run the engine's own device kernels. ---- */
dimg_status dimg_op_dense(int device, const dimg_qtensor* w, const int64_t* x, int64_t* out);
/* dense_forward (proj/src/kernels.cpp:18-30) applied to T tokens x[T][cols]
 * -> out[T][rows]: the prefill GEMM (tcgen05 kind::i8 over byte limbs). */
dimg_status dimg_op_dense_tokens(int device, const dimg_qtensor* w, const int64_t* x, uint32_t T, int64_t* out);
/* BLAKE3 (hash mode, 32 bytes) on the GPU: weight_hash / deserialize of the
 * model bytes (proj/src/model.cpp:310-316, attest.cpp:93) as a tree hash at
 * HBM speed. _device: `data` is a device pointer on `device` (ms, if not
 * NULL, receives the kernels' CUDA-event time); _gpu: host bytes, uploaded
 * first. Bit-identical to dimg_blake3. */
dimg_status dimg_blake3_device(int device, const void* data, size_t len, uint8_t out[32], float* ms);
dimg_status dimg_blake3_gpu(int device, const void* data, size_t len, uint8_t out[32]);

/* Attestation (proj/include/dim/attest.hpp:16-68, proj/src/attest.cpp). The
 * 112-byte wire format: model_id | input_hash | output_hash | bond (u64 LE) |
 * challenge_period (u64 LE). decode of any other size: DIMG_EPARSE with
 * parse kind DIMG_PARSE_TRUNCATED. */
typedef struct {
    uint8_t model_id[32];     /* BLAKE3 of the model bytes */
    uint8_t input_hash[32];   /* hash_token_ids(prompt) */
    uint8_t output_hash[32];  /* GenerationResult::output_hash */
    uint64_t bond, challenge_period;
} dimg_attestation;
/* VerifyOutcome: confirmed, or refuted at stage 0 model / 1 input / 2 output
 * with the claimed (expected) and recomputed (found) digests. */
typedef struct {
    uint32_t confirmed;
    uint32_t refuted_stage;
    uint8_t expected[32], found[32];
} dimg_verify_outcome;
dimg_status dimg_attestation_encode(const dimg_attestation* a, uint8_t out[112]);
dimg_status dimg_attestation_decode(const uint8_t* bytes, size_t n, dimg_attestation* out);
/* to_text (attest.cpp:54-62); writes at most cap-1 chars + NUL, *len = full length */
dimg_status dimg_attestation_text(const dimg_attestation* a, char* buf, size_t cap, size_t* len);
/* make_attestation (attest.cpp:68-78): the model id by the GPU BLAKE3 on `device`. */
dimg_status dimg_make_attestation(int device, const uint8_t* model_bytes, size_t n_bytes, const uint32_t* prompt,
                                  size_t n_prompt, const uint8_t output_hash[32], uint64_t bond,
                                  uint64_t challenge_period, dimg_attestation* out);
/* verify_by_reexecution (attest.cpp:89-117): model id (GPU BLAKE3), input hash,
 * then deserialize + one greedy re-execution on `device`; the first stage
 * that differs refutes. Unparseable model bytes: DIMG_EPARSE (no verdict). */
dimg_status dimg_verify_by_reexecution(int device, const dimg_attestation* att, const uint8_t* model_bytes,
                                       size_t n_bytes, const uint32_t* prompt, size_t n_prompt, uint32_t max_new,
                                       dimg_verify_outcome* out);
/* dispute_game (attest.cpp:119-125): *winner 0 = attester, 1 = challenger. */
dimg_status dimg_dispute_game(int device, const dimg_attestation* att, const uint8_t* model_bytes, size_t n_bytes,
                              const uint32_t* prompt, size_t n_prompt, uint32_t max_new, uint32_t* winner,
                              dimg_verify_outcome* out);
/* Seeded sampling (proj/src/engine.cpp:122-163). dimg_sample_key: the RNG key
 * BLAKE3(model bytes || prompt ids as u32 LE), hashed on the GPU.
 * dimg_generate_sampled: generate_sampled with that key and a Q16
 * temperature (> 0, else DIMG_EINVAL); each step's token is drawn on the
 * device (sample_from_logits with the step's ChaCha20 u32). dimg_op_sample:
 * sample_from_logits of one row with a given draw (parity tests). */
dimg_status dimg_sample_key(int device, const uint8_t* model_bytes, size_t n_bytes, const uint32_t* prompt,
                            size_t n_prompt, uint8_t key[32]);
dimg_status dimg_generate_sampled(dimg_session* s, const uint32_t* prompt, uint32_t n_prompt, uint32_t max_new,
                                  int64_t temperature, const uint8_t key[32], uint32_t* tokens_out,
                                  uint8_t hash_out[32]);
dimg_status dimg_op_sample(int device, const int64_t* logits, uint32_t V, int64_t temperature, uint32_t draw,
                           uint32_t* out);
/* generation_counter (engine.cpp:165-168): generation runs in this process. */
dimg_status dimg_generation_counter(uint64_t* out);
dimg_status dimg_op_rmsnorm(int device, const int64_t* x, const int64_t* g, uint32_t n,
                            int64_t* out);
dimg_status dimg_op_softmax(int device, const int64_t* s, uint32_t n, int64_t* out);
/* T consecutive attention_step calls at pos 0..T-1 on a fresh cache;
 * q/k/v/out are [T][n_heads*d_head]. */
dimg_status dimg_op_attention(int device, uint32_t n_heads, uint32_t d_head, uint32_t max_ctx,
                              double theta, uint32_t steps, const int64_t* q, const int64_t* k,
                              const int64_t* v, int64_t* out);
dimg_status dimg_op_ffn(int device, const dimg_qtensor* gate, const dimg_qtensor* up,
                        const dimg_qtensor* down, const int64_t* x, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
