// Persistent decode kernel: every forward step of a generation in ONE
// cooperative launch (one CTA per SM).
//
// Why: a batch-1 integer decode step is 5L+1 dependent matrix-vector stages.
// As separate kernels each stage pays launch + ramp-up + a serial prologue
// (rebuilding the input vector's limbs) + drain, and the HBM pipe idles in
// between (the multi-kernel v1 reached 25% of roofline). Here the stages are
// separated by grid barriers instead, and -- because weights never depend on
// activations -- every warp keeps streaming its NEXT weight chunks into a
// private shared-memory ring with cp.async.bulk (TMA bulk copies, mbarrier
// completion) while it waits at a barrier or builds the next input vector.
// The weight stream runs continuously across stage, layer and token
// boundaries. (tools/microbench.cu: rings of 4-8 KB chunks, 8 warps,
// 128-192 KB/SM stream ~7 TB/s on a B200 with the DP4A work on; in the
// kernel 4 KB chunks, as many per warp as shared memory leaves, measured best.)
//
// Weight layout in HBM ("row-group blocked", built at upload): each matrix is
// cut into groups of 4 rows and K-segments of <= PK_SEG bytes; chunk (group,
// segment) is one contiguous 4 x seg block = one bulk copy. CTAs own
// contiguous balanced group ranges; warp w of a CTA owns groups w, w+8, ...
// and walks all K-segments of a group, so its per-limb int32 partial sums stay
// in registers and each group needs one warp reduction. The dot products are
// the exact byte-limb DP4A scheme of gemv.cuh.
//
// Stage inputs are staged into shared memory with one vectorised L2 pass:
// rmsnorm inputs (the residual stream) are copied and normalised there;
// the attention output and the FFN hidden vector arrive as 3-limb byte planes
// written by their producers (attention / silu*up epilogues) plus a "needs
// more than 3 limbs" flag, so those prologues are a 12-33 KB copy.
#pragma once

#include <cstdint>

#include "attention.cuh"
#include "gemv.cuh"
#include "q16.cuh"

namespace dimg::dev {

constexpr int PK_THREADS = 256;
constexpr int PK_WARPS = PK_THREADS / 32;
#ifndef DIMG_PK_MAX_DEPTH
#define DIMG_PK_MAX_DEPTH 6
#endif
constexpr int PK_MAX_DEPTH = DIMG_PK_MAX_DEPTH;  // chunks in flight per warp (runtime depth <= this)
#ifndef DIMG_PK_SEG
#define DIMG_PK_SEG 1024
#endif
constexpr int PK_SEG = DIMG_PK_SEG;     // K-segment width (bytes; a multiple of 512)
constexpr int PK_ROWS = 4;              // rows per group
constexpr int PK_SCALES = PK_ROWS * 8;             // the group's 4 int64 row scales
constexpr int PK_SLOT = PK_ROWS * PK_SEG + PK_SCALES;  // chunk bytes incl. trailing scales

// Bytes of one row group in the blocked layout: 4 rows x Kp, then 4 scales.
__host__ __device__ constexpr size_t pk_group_bytes(uint32_t Kp) { return size_t(PK_ROWS) * Kp + PK_SCALES; }

enum { SK_GEMV = 0, SK_ATTN = 1 };

struct PkStage {
    uint32_t kind, mode, epi, layer;
    uint32_t rows, K, Kp, n_groups, n_segs, gamma_unit;
    const int8_t* W;          // blocked [n_groups][n_segs][4][seg] + 4 scales per group
    const int64_t* scales;    // [rows]
    const int64_t* x;         // input vector (K)
    const int64_t* gamma;     // norm gains (MODE_NORM / MODE_EMBED)
    int64_t* y;               // output
    const uint32_t* in_words; // MODE_PLAIN: the input as tagged limb words (nullptr: build from x)
    uint32_t* out_words;      // EPI_SILU / attention: publish y as tagged limb words
    uint32_t no_barrier;      // 1: the next stage consumes tagged words, no grid barrier after this one
    uint32_t tp_sum;          // EPI_RESID, tensor parallel: 1 + inbox buffer (WO 1, w_down 2); 0 none
    int32_t* x32_out;         // EPI_RESID: the clamped x also as int32 (|x| <= 2^24)
    const int32_t* x32_in;    // MODE_NORM after a RESID stage: read that copy (16 KB, not 32)
    // Residual stream as tagged words (no grid barrier after a RESID stage):
    // word = (x + 2^24) in bits 0-25 | 6-bit tag in 26-31; two alternating buffers.
    uint32_t* xw_out;         // EPI_RESID: publish the new x here (tag of the current layer)
    const uint32_t* xw_in;    // MODE_NORM: poll x from here; EPI_RESID: the residual input
    uint32_t xw_lag;          // its tag is the current layer's minus xw_lag
    uint32_t resid_embed;     // EPI_RESID on layer 0: the residual input is the token's embedding
    unsigned long long* ytag; // EPI_STORE: also publish y as tagged word pairs (attention inputs)
    unsigned long long* ssq_out;  // EPI_RESID: sum of the new x^2 (exact: |x| <= 2^24 after the clamp)
    const unsigned long long* ssq_in;  // MODE_NORM after a RESID stage: that sum (nullptr = compute it)
    unsigned long long* ssq_clear;     // accumulator the previous stage consumed: CTA 0 re-zeroes it
};

struct PkArgs {
    const PkStage* stages;    // [n_stages]: 5 per layer, then the head
    uint32_t n_layer_stages;  // 5L
    uint32_t n_steps;         // forward steps in this launch
    uint32_t n_prefill;       // the first n_prefill steps skip the head
    uint32_t planes_bytes;    // shared staging area (vector, 3 limb planes, attention)
    uint32_t ring_depth;      // weight-ring slots per warp (2 .. PK_MAX_DEPTH)
    uint32_t* wide_planes;    // [grid][wide_stride] words: 8-limb planes of out-of-range inputs
    uint32_t wide_stride;
    Ctl* ctl;
    unsigned int* bar;        // grid barrier counter (zeroed before launch)
    // embedding / head
    const int8_t* embd;
    const int64_t* embd_scales;
    uint32_t d_model, vocab;
    uint32_t* tokens;
    int64_t* logits;          // [keep_cap + 1][vocab]
    ArgPart* parts;           // [gridDim.x]
    int64_t* x_resid;         // residual stream (embedding target)
    // attention
    AttnArgs attn;            // per-layer kc/vc offsets applied in-kernel
    size_t kv_layer_stride;   // elements between layers in kc/vc
    const int64_t* exp_lut;   // repointed to a shared-memory copy inside the kernel
    const int64_t* seeds;     // idem
    unsigned long long* trace;  // optional: [stage_seq][32] stamps of CTA 0 (dimg_session_trace)
    uint32_t trace_cap;
    uint32_t attn_parts;      // CTAs per attention head (position blocks / dimension slices)
    uint32_t attn_dpp;        // dims per part (whole 4-dim quads)
    int32_t attn_np_shift;    // log2(attn_parts) if a power of two, else -1
    int32_t attn_nq_shift;    // log2(attn_dpp / 4) if a power of two, else -1
    unsigned long long* xg;   // [H][max_ctx][2] tagged score words exchanged by a head's parts
    unsigned long long* parts_w;  // [2][grid][3] tagged lm_head partials (value lo/hi, index)
    unsigned long long* qkv_x;  // [3D][2] tagged q | k | v words (QKV stage -> attention)
    uint32_t tag_base;        // attention stage k of this launch tags its words tag_base + k (never 0)
    int32_t* kc32;            // int32 mirror of kc / vc (same layout), read while kvwide is clear
    int32_t* vc32;
    uint32_t* kvwide;         // [L][H] some cached K/V value of the head needs more than 32 bits
    unsigned long long* trace_all;  // optional: [stage_seq][grid][2] every CTA's prologue end / chunk-loop end
    // Tensor parallel: this launch is rank tp_rank of tp_g,
    // holding its heads / FFN rows / vocab rows (vocab_off = its first vocab
    // row). The row-parallel stages' (WO, w_down) pre-scale accumulators are
    // summed across the ranks inside their epilogues: each CTA stores its rows'
    // partials straight into every peer's inbox (tagged words, peer memory over
    // NVLink or, for the one-device group, plain device memory) and polls its
    // own inbox for the peers' partials of the same rows; the lm_head's per-CTA
    // (max, index) partials go to every rank the same way. tp_g <= 1: none of it.
    uint32_t tp_g, tp_rank, vocab_off;
    unsigned long long* tp_in[8];     // every rank's inbox [2 (WO | down)][tp_g][d_model][2]
    unsigned long long* tp_parts[8];  // every rank's lm_head slots [2][tp_g * grid][4]
};

constexpr int PK_TP_MAX = 8;

// Scheduling constants, held in registers (never address kernel params or
// shared structs from hot code: local memory goes through L1, which each
// grid barrier's fence invalidates, turning every such read into an L2 trip).
// What a warp's weight stream needs of each stage, copied into shared memory
// at launch (reading the descriptors in global memory at every stage change
// cost an L2 round trip -- the grid fences keep L1 cold -- while the warp
// still had chunks to consume).
struct FetchInfo {
    const int8_t* W;
    uint32_t g_lo, g_hi;  // this CTA's row groups (empty: attention)
    uint32_t n_segs, Kp;
};

struct Sched {
    const PkStage* stages;
    uint32_t n_layer_stages, n_steps, n_prefill;
    const FetchInfo* fi;  // [n_layer_stages + 1], shared memory
};

// ---- small PTX helpers --------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D TMA bulk copy global -> shared, completion via the mbarrier's tx count.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const unsigned int* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// L2-coherent loads for data other CTAs wrote in this launch.
__device__ __forceinline__ int4 ld_cg4(const void* p) {
    int4 r;
    asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ int64_t ld_cg64(const int64_t* p) {
    int64_t r;
    asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_cg32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Tagged-word exchange (the LL-protocol idea): every 8-byte word carries 32
// bits of payload and a 32-bit stage tag; an aligned 8-byte access is
// single-copy atomic, so a reader that sees the current tag sees its payload
// -- no fence, no counter, one trip through L2.
__device__ __forceinline__ void st_tagged2(unsigned long long* p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_tagged2(const unsigned long long* p, uint64_t& a, uint64_t& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// The same at system scope: words another GPU stores into this one's memory
// (or this one into a peer's) over NVLink.
__device__ __forceinline__ void st_tagged2_sys(unsigned long long* p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_tagged2_sys(const unsigned long long* p, uint64_t& a, uint64_t& b) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Limb word of a MODE_PLAIN input element: bytes 0-2 = the three low limb
// bytes, byte 3 = wide bit (needs more than 3 limbs) << 7 | 7-bit stage tag.
__device__ __forceinline__ uint32_t limb_word(int64_t v, uint32_t tag7) {
    const uint32_t wide = (v < -(int64_t(1) << 23) || v >= (int64_t(1) << 23)) ? 0x80u : 0u;
    return (uint32_t(v) & 0xFFFFFFu) | ((wide | tag7) << 24);
}
__device__ __forceinline__ void st_word(uint32_t* p, uint32_t w) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 ld_words4(const uint32_t* p) {
    uint4 r;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}
// 1 + (tag mod 127): consecutive uses of a word buffer always differ.
__device__ __forceinline__ uint32_t tag7_of(uint32_t tag) { return 1u + tag % 127u; }
// Residual-stream words: |x| <= 2^24 after the clamp, so x + 2^24 fits 26
// bits; 6-bit tag 1 + (layer mod 63) above it.
__device__ __forceinline__ uint32_t tag6_of(uint32_t tag) { return 1u + tag % 63u; }
__device__ __forceinline__ uint32_t x_word(int64_t x, uint32_t tag6) {
    return uint32_t(x + (int64_t(1) << 24)) | (tag6 << 26);
}
__device__ __forceinline__ int32_t x_of_word(uint32_t w) { return int32_t(w & 0x3FFFFFFu) - (1 << 24); }
__device__ __forceinline__ uint32_t ld_word(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spins until the word's tag (bits >= shift) equals `tag`; a 4 s timeout
// (or another CTA's timeout) sets ctl->err bit 2 and returns the stale word:
// the launch then fails instead of hanging the GPU.
__device__ __noinline__ uint32_t poll_word(const uint32_t* p, uint32_t tag, int shift, Ctl* ctl) {
    uint64_t g0 = 0;
    for (uint32_t spins = 1;; ++spins) {
        const uint32_t w = ld_word(p);
        if ((w >> shift) == tag) return w;
        if ((spins & 1023) == 0) {
            const uint64_t now = globaltimer();
            if (!g0) g0 = now;
            if ((*((volatile uint32_t*)&ctl->err) & 4u) || now - g0 > 4000000000ull) {
                atomicOr(&ctl->err, 4u);
                return w;
            }
        }
    }
}

// Block-wide global -> shared copy of `bytes` (multiple of 16), many 16-B
// loads in flight per thread.
__device__ __forceinline__ void copy_g2s(void* dst, const void* src, uint32_t bytes) {
    const uint32_t n = bytes / 16;
    int4* d = static_cast<int4*>(dst);
    const char* s = static_cast<const char*>(src);
    uint32_t i = threadIdx.x;
    for (; i + 7 * PK_THREADS < n; i += 8 * PK_THREADS) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_cg4(s + size_t(i + u * PK_THREADS) * 16);
#pragma unroll
        for (int u = 0; u < 8; ++u) d[i + u * PK_THREADS] = v[u];
    }
    for (; i < n; i += PK_THREADS) d[i] = ld_cg4(s + size_t(i) * 16);
}

// Grid barrier #k (monotonic counter). Returns false if the wait timed out
// (a hung peer): the caller then unwinds instead of hanging the GPU.
// vg: the CTAs of this rank (gridDim.x, or the rank's share of a one-device
// tensor-parallel launch).
__device__ __forceinline__ bool grid_sync(unsigned int* bar, Ctl* ctl, uint32_t k, uint32_t vg) {
    __shared__ int ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        ok = 1;
        __threadfence();
        atomicAdd(bar, 1u);
        const uint32_t target = (k + 1) * vg;
        uint64_t t0 = globaltimer();
        while (ld_acquire(bar) < target) {
            if (*((volatile uint32_t*)&ctl->err) & 4u) { ok = 0; break; }
            if (globaltimer() - t0 > 4000000000ull) {  // 4 s
                atomicOr(&ctl->err, 4u);
                ok = 0;
                break;
            }
        }
    }
    __syncthreads();
    return ok != 0;
}

// CTA vb of vg: its share of n units.
__device__ __forceinline__ void cta_range(uint32_t n, uint32_t& lo, uint32_t& hi, uint32_t vb, uint32_t vg) {
    lo = uint32_t(uint64_t(n) * vb / vg);
    hi = uint32_t(uint64_t(n) * (vb + 1) / vg);
}

__device__ __forceinline__ uint32_t stages_in_step(const Sched& sc, uint32_t step) {
    return sc.n_layer_stages + (step >= sc.n_prefill ? 1u : 0u);
}

// ---- the warp's weight-chunk stream (same order as its consumption) -----------

struct Fetch {
    uint32_t step, stage, g, g_end, seg, n_segs, Kp;
    const int8_t* W;
    bool done;
};

__device__ __forceinline__ void fetch_load(const Sched& sc, Fetch& f) {
    const FetchInfo& fi = sc.fi[f.stage];
    f.g = fi.g_lo + (threadIdx.x >> 5);
    f.g_end = fi.g_hi;
    f.seg = 0;
    f.n_segs = fi.n_segs;
    f.Kp = fi.Kp;
    f.W = fi.W;
}

__device__ __forceinline__ void fetch_settle(const Sched& sc, Fetch& f) {
    while (!f.done && f.g >= f.g_end) {
        if (++f.stage >= stages_in_step(sc, f.step)) {
            f.stage = 0;
            if (++f.step >= sc.n_steps) {
                f.done = true;
                return;
            }
        }
        fetch_load(sc, f);
    }
}

__device__ __forceinline__ void fetch_advance(const Sched& sc, Fetch& f) {
    if (++f.seg == f.n_segs) {
        f.seg = 0;
        f.g += PK_WARPS;
    }
    fetch_settle(sc, f);
}

__device__ __forceinline__ uint32_t fetch_bytes(const Fetch& f) {
    return f.seg + 1 < f.n_segs ? PK_ROWS * PK_SEG
                                : PK_ROWS * (f.Kp - (f.n_segs - 1) * PK_SEG) + PK_SCALES;
}
__device__ __forceinline__ const int8_t* fetch_src(const Fetch& f) {
    return f.W + size_t(f.g) * pk_group_bytes(f.Kp) + size_t(f.seg) * PK_ROWS * PK_SEG;
}

__device__ __forceinline__ void fetch_issue(const Fetch& f, uint8_t* slot, uint64_t* bar) {
    mbar_expect_tx(bar, fetch_bytes(f));
    bulk_g2s(slot, fetch_src(f), fetch_bytes(f), bar);
}

#ifdef DIMG_CHUNK_TRACE
// Experiment build only (tools/chunk_trace.py): warp 0 of every CTA logs
// clock64 around each ring wait, plus stage markers.
constexpr int CT_MAX = 4096;
__device__ unsigned long long g_ct[148][CT_MAX][2];
#endif

struct Pipe {
#ifdef DIMG_CHUNK_TRACE
    uint32_t ctn;
#endif
    uint8_t* slots;     // this warp's ring
    uint64_t* bars;
    uint32_t slot;      // slot of the next chunk to consume
    uint32_t phase;     // its mbarrier parity
    uint32_t depth;     // slots in the ring (runtime: what shared memory allows)
    Fetch f;            // next chunk to load into the ring
};

// Waits for the next chunk of this warp; returns its slot.
__device__ __forceinline__ const uint8_t* pipe_wait(Pipe& p) {
#ifdef DIMG_CHUNK_TRACE
    const unsigned long long c0 = clock64();
    mbar_wait(&p.bars[p.slot], p.phase);
    if (threadIdx.x == 0 && blockIdx.x < 148 && p.ctn < CT_MAX) {
        g_ct[blockIdx.x][p.ctn][0] = c0;
        g_ct[blockIdx.x][p.ctn][1] = clock64();
        ++p.ctn;
    }
#else
    mbar_wait(&p.bars[p.slot], p.phase);
#endif
    return p.slots + p.slot * PK_SLOT;
}

// Releases the chunk just consumed and refills its slot with the next one.
__device__ __forceinline__ void pipe_release(const Sched& sc, Pipe& p) {
    const uint32_t sl = p.slot;
    if (++p.slot == p.depth) {
        p.slot = 0;
        p.phase ^= 1;
    }
    __syncwarp();
    if (!p.f.done) {
        if ((threadIdx.x & 31) == 0) {
#ifndef DIMG_EXP_NOFENCE
            fence_proxy_async();
#endif
            fetch_issue(p.f, p.slots + sl * PK_SLOT, &p.bars[sl]);
        }
        fetch_advance(sc, p.f);
    }
}

// ---- prologue: the stage's input vector as limb planes in shared memory -------
// Everything here runs once per stage: it is kept compact and out of line,
// because under a saturated HBM every instruction-cache miss is an L2 round
// trip (ncu: 46% of prologue stalls were stall_no_inst before this).

// Attention output / FFN hidden vector. Published by the producing stage as
// tagged limb words with no grid barrier in between: poll every word (16-byte
// loads) and unpack its three limb bytes into the planes. Every CTA reads
// every word, so "some element needs more than 3 limbs" is a grid-uniform
// decision: then (PLAIN_WIDE) all CTAs take one extra grid barrier and build
// 8 planes from the int64 vector (planes_from_x). words == nullptr (timing
// probes): planes straight from x.
constexpr int PLAIN_WIDE = 9;

// mul16(x, r) = (x r) >> 16 (proj/src/q16.cpp) for |x|, r <= 2^24 (the
// residual stream after the clamp and the rmsnorm factor): one IMAD.WIDE and
// one funnel shift give the low 32 bits of the result (its three limb bytes);
// fits &= the result lies in [-2^23, 2^23), i.e. x r in [-2^39, 2^39).
__device__ __forceinline__ uint32_t norm_lo32(int32_t x, int32_t r, int& fits) {
    int64_t p;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(p) : "r"(x), "r"(r));
    const int32_t hi = int32_t(p >> 32);
    fits &= uint32_t((hi >> 7) + 1) <= 1u;
    return __funnelshift_r(uint32_t(p), uint32_t(hi), 16);
}

// Bytes 0, 1, 2 of four elements -> one word per limb plane.
__device__ __forceinline__ void put_planes3(uint32_t* planes, uint32_t Kw, uint32_t w, const uint32_t (&lo)[4]) {
    planes[w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0040), __byte_perm(lo[2], lo[3], 0x0040), 0x5410);
    planes[Kw + w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0051), __byte_perm(lo[2], lo[3], 0x0051), 0x5410);
    planes[2 * Kw + w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0062), __byte_perm(lo[2], lo[3], 0x0062), 0x5410);
}

// 8-limb planes go to the CTA's global scratch (wplanes): shared memory only
// holds the usual 3.
__device__ __noinline__ int planes_from_x(uint32_t K, uint32_t Kp, const int64_t* x, uint32_t* splanes,
                                          uint32_t* wplanes, Ctl* ctl, bool wide) {
    const uint32_t Kw = Kp / 4;
    if (!wide) {
        int fits = 1;
        for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
            const int64_t v = ld_cg64(x + j);
            fits &= v >= -(int64_t(1) << 23) && v < (int64_t(1) << 23);
        }
        wide = !__syncthreads_and(fits);
    }
    const int L = wide ? 8 : 3;
    uint32_t* planes = wide ? wplanes : splanes;
#pragma unroll 1
    for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
        uint64_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = 4 * w + e < K ? uint64_t(ld_cg64(x + 4 * w + e)) : 0;
#pragma unroll 1
        for (int k = 0; k < L; ++k) {
            uint32_t word = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) word |= uint32_t((v[e] >> (8 * k)) & 0xFF) << (8 * e);
            planes[k * Kw + w] = word;
        }
    }
    if (L == 8 && threadIdx.x == 0) atomicAdd(&ctl->stats[0], 1ull);
    __syncthreads();
    return L;
}

__device__ __forceinline__ bool words_ready(uint4 q, uint32_t j, uint32_t K, uint32_t tag7) {
    return (j >= K || ((q.x >> 24) & 0x7Fu) == tag7) && (j + 1 >= K || ((q.y >> 24) & 0x7Fu) == tag7) &&
           (j + 2 >= K || ((q.z >> 24) & 0x7Fu) == tag7) && (j + 3 >= K || ((q.w >> 24) & 0x7Fu) == tag7);
}

__device__ __noinline__ int prologue_plain(uint32_t K, uint32_t Kp, const int64_t* x, const uint32_t* words,
                                           uint32_t tag7, uint32_t* planes, uint32_t* wplanes, Ctl* ctl) {
    const uint32_t Kw = Kp / 4;
    if (!words) return planes_from_x(K, Kp, x, planes, wplanes, ctl, false);
    constexpr int B = 8;  // 16-byte loads in flight per thread
    int wide = 0, ok = 1;
#pragma unroll 1
    for (uint32_t w0 = threadIdx.x; w0 < Kw && ok; w0 += B * PK_THREADS) {
        // the whole batch is reloaded until every word is published: one
        // round trip per retry, not one per late word
        uint4 q[B];
        uint64_t g0 = 0;
        for (uint32_t spins = 1;; ++spins) {
            bool ready = true;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t w = w0 + b * PK_THREADS;
                q[b] = w < Kw && 4 * w < K ? ld_words4(words + 4 * w) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t w = w0 + b * PK_THREADS;
                ready &= w >= Kw || 4 * w >= K || words_ready(q[b], 4 * w, K, tag7);
            }
            if (ready) break;
            if ((spins & 255) == 0) {
                const uint64_t now = globaltimer();
                if (!g0) g0 = now;
                if ((*((volatile uint32_t*)&ctl->err) & 4u) || now - g0 > 4000000000ull) {
                    atomicOr(&ctl->err, 4u);
                    ok = 0;
                    break;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const uint32_t w = w0 + b * PK_THREADS;
            if (w >= Kw) continue;
            uint4 v = q[b];
            if (4 * w < K) {
                if (4 * w + 1 >= K) v.y = 0;  // padding of the last word group
                if (4 * w + 2 >= K) v.z = 0;
                if (4 * w + 3 >= K) v.w = 0;
            }
            wide |= (v.x | v.y | v.z | v.w) >> 31;
            planes[w] = __byte_perm(__byte_perm(v.x, v.y, 0x0040), __byte_perm(v.z, v.w, 0x0040), 0x5410);
            planes[Kw + w] = __byte_perm(__byte_perm(v.x, v.y, 0x0051), __byte_perm(v.z, v.w, 0x0051), 0x5410);
            planes[2 * Kw + w] = __byte_perm(__byte_perm(v.x, v.y, 0x0062), __byte_perm(v.z, v.w, 0x0062), 0x5410);
        }
    }
    const int f = __syncthreads_or((ok ? 0 : 2) | (wide ? 1 : 0));  // one barrier for both decisions
    if (f & 2) return -1;
    return (f & 1) ? PLAIN_WIDE : 3;
}

// rmsnorm input: the residual stream (or the embedded token on layer 0)
// staged in shared memory, normalised there, packed into planes.
// erow != nullptr selects the embedding (engine.cpp:10-19).
__device__ __noinline__ int prologue_norm(uint32_t K, uint32_t Kp, bool gamma_unit, const int64_t* x,
                                          const int64_t* gamma, const int8_t* erow, int64_t es,
                                          int64_t* x_resid, int64_t* xb, uint32_t* planes, uint32_t* wplanes,
                                          u128* red, const int64_t* seeds, Ctl* ctl, unsigned long long* tr,
                                          const unsigned long long* ssq_in, const int32_t* x32) {
    const uint32_t Kw = Kp / 4;
    __shared__ int64_t s_r;
    if (ssq_in && gamma_unit && x32) {
        // The producer (a residual stage) already summed the squares of the
        // clamped vector and wrote it as int32 too (|x| <= 2^24): thread 0
        // computes r while the 4-byte copy is in flight; r <= 2^24, so the
        // products are 32 x 32 bits throughout.
        if (threadIdx.x == 0) {
            const uint64_t ss = uint64_t(ld_cg64(reinterpret_cast<const int64_t*>(ssq_in)));
            const int64_t ms = int64_t(((K & (K - 1)) ? ss / K : ss >> (__ffs(K) - 1)) >> 16);
            s_r = inv_sqrt_q16(ms + 1, seeds);  // ms >= 0: ms + 1 > 0
        }
        int32_t* xs32 = reinterpret_cast<int32_t*>(xb);
        copy_g2s(xs32, x32, Kp * 4);
        __syncthreads();
        if (tr) tr[4] = tr[5] = clock64();
        const int64_t r_inv = s_r;
        if (tr) tr[6] = clock64();
        int fits = 1;
#pragma unroll 1
        for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
            const int4 e4 = *reinterpret_cast<const int4*>(xs32 + 4 * w);
            const int32_t xs[4] = {e4.x, e4.y, e4.z, e4.w};
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) lo[e] = norm_lo32(4 * w + e < K ? xs[e] : 0, int32_t(r_inv), fits);
            put_planes3(planes, Kw, w, lo);
        }
        fits = __syncthreads_and(fits);
        if (tr) tr[7] = clock64();
        if (fits) return 3;
        // wide (needs > 3 limbs): 8 planes of the normalised vector into the
        // global scratch, recomputed from the global int32 copy (rare)
#pragma unroll 1
        for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x)
#pragma unroll 1
            for (int k = 0; k < 8; ++k) {
                uint32_t word = 0;
                for (int e = 0; e < 4; ++e) {
                    const uint32_t j = 4 * w + e;
                    const int64_t v = j < K ? (int64_t(__ldcg(x32 + j)) * int32_t(r_inv)) >> 16 : 0;
                    word |= uint32_t((uint64_t(v) >> (8 * k)) & 0xFF) << (8 * e);
                }
                wplanes[k * Kw + w] = word;
            }
        if (threadIdx.x == 0) atomicAdd(&ctl->stats[0], 1ull);
        __syncthreads();
        return 8;
    }
    if (erow) {
        for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
            const int64_t v = int64_t(uint64_t(int64_t(erow[j])) * uint64_t(es));
            xb[j] = v;
            if (x_resid) x_resid[j] = v;
        }
    } else {
        copy_g2s(xb, x, K * 8);
    }
    __syncthreads();
    if (tr) tr[4] = clock64();
    // ms = ((sum x^2) / n) >> 16 in int128, r = inv_sqrt(ms + 1) (kernels.cpp:56-68).
    // Squares of |x| < 2^31 are < 2^62: split into 21-bit chunks whose per-
    // warp sums fit 32 bits, so three REDUX.SUM give the exact warp totals;
    // any larger element goes through the 128-bit path.
    __shared__ uint32_t s_part[PK_WARPS][3];
    __shared__ int s_big;
    if (threadIdx.x == 0) s_big = 0;
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    u128 big = 0;
    int small = 1;
#pragma unroll 4
    for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
        const int64_t v = xb[j];
        if (fits_i32(v)) {
            const uint64_t q = uint64_t(int64_t(int32_t(v)) * int32_t(v));
            c0 += uint32_t(q) & 0x1FFFFFu;
            c1 += uint32_t(q >> 21) & 0x1FFFFFu;
            c2 += uint32_t(q >> 42);
        } else {
            big += mul_full(v, v);
            small = 0;
        }
    }
    c0 = __reduce_add_sync(0xffffffffu, c0);
    c1 = __reduce_add_sync(0xffffffffu, c1);
    c2 = __reduce_add_sync(0xffffffffu, c2);
    if ((threadIdx.x & 31) == 0) {
        s_part[threadIdx.x >> 5][0] = c0;
        s_part[threadIdx.x >> 5][1] = c1;
        s_part[threadIdx.x >> 5][2] = c2;
    }
    if (!small) s_big = 1;
    __syncthreads();
    uint64_t t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
    for (int w = 0; w < PK_WARPS; ++w) {
        t0 += s_part[w][0];
        t1 += s_part[w][1];
        t2 += s_part[w][2];
    }
    u128 ss = u128(t0) + (u128(t1) << 21) + (u128(t2) << 42);
    const bool any_big = s_big;
    if (any_big) ss += block_sum_u128(big, red);  // uniform branch
    if (tr) tr[5] = clock64();
    // one thread computes r; the others wait instead of contending for the
    // multiplier with 255 redundant copies of the 128-bit Newton iteration
    if (threadIdx.x == 0) {
        int64_t ms;
        if ((ss >> 63) == 0) ms = int64_t((uint64_t(ss) / K) >> 16);  // usual case: one u64 divide
        else ms = int64_t((i128(ss) / i128(K)) >> 16);
        if (ms + 1 <= 0) {
            atomicOr(&ctl->err, 1u);
            s_r = 0;
        } else {
            s_r = inv_sqrt_q16(ms + 1, seeds);
        }
    }
    __syncthreads();
    const int64_t r_inv = s_r;
    if (tr) tr[6] = clock64();
    const bool fast = !any_big && fits_i32(r_inv) && gamma_unit;
    int fits = 1;
#pragma unroll 2
    for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
        uint32_t lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t j = 4 * w + e;
            int64_t v = 0;
            if (j < K) {
                if (fast) {
                    v = mul16_small(xb[j], r_inv);
                } else {
                    v = mul16(xb[j], r_inv);
                    if (!gamma_unit) v = mul16(v, ld_cg64(gamma + j));  // mul16(v, ONE) == v
                }
            }
            xb[j] = v;
            fits &= uint64_t(v + (int64_t(1) << 23)) < (uint64_t(1) << 24);  // -2^23 <= v < 2^23
            lo[e] = uint32_t(v);
        }
        // bytes 0, 1, 2 of the four elements -> one word per plane
        planes[w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0040), __byte_perm(lo[2], lo[3], 0x0040), 0x5410);
        planes[Kw + w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0051), __byte_perm(lo[2], lo[3], 0x0051), 0x5410);
        planes[2 * Kw + w] = __byte_perm(__byte_perm(lo[0], lo[1], 0x0062), __byte_perm(lo[2], lo[3], 0x0062), 0x5410);
    }
    fits = __syncthreads_and(fits);
    if (tr) tr[7] = clock64();
    if (fits) return 3;
#pragma unroll 1
    for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x)
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            uint32_t word = 0;
            for (int e = 0; e < 4; ++e) word |= uint32_t((uint64_t(xb[4 * w + e]) >> (8 * k)) & 0xFF) << (8 * e);
            wplanes[k * Kw + w] = word;
        }
    if (threadIdx.x == 0) atomicAdd(&ctl->stats[0], 1ull);
    __syncthreads();
    return 8;
}


// rmsnorm of the residual stream published as tagged words by the previous
// residual stage (no grid barrier in between): poll every word (16-byte
// loads, 8 in flight per thread), keep x (|x| <= 2^24) as int32 in shared
// memory and sum x^2 exactly (x^2 < 2^48, K < 2^12 -> u64) while doing so;
// then r = inv_sqrt(ms + 1) and the normalised limb planes. Returns 3, 8
// (planes in the global scratch) or -1 (a producer never published).
__device__ __noinline__ int prologue_norm_words(uint32_t K, uint32_t Kp, bool gamma_unit, const int64_t* gamma,
                                                const uint32_t* words, uint32_t tag6, int32_t* xs32, uint32_t* planes,
                                                uint32_t* wplanes, const int64_t* seeds, Ctl* ctl,
                                                unsigned long long* tr) {
    __shared__ uint64_t s_ss[PK_WARPS];
    __shared__ int64_t s_r2;
    const uint32_t Kw = Kp / 4;
    constexpr int B = 4;
    uint64_t ss = 0;
    int ok = 1;
#pragma unroll 1
    for (uint32_t w0 = threadIdx.x; w0 < Kw && ok; w0 += B * PK_THREADS) {
        // the whole batch is reloaded until every word carries this layer's
        // tag: one round trip per retry, not one per late word
        uint4 q[B];
        uint64_t g0 = 0;
        for (uint32_t spins = 1;; ++spins) {
            bool ready = true;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t w = w0 + b * PK_THREADS;
                q[b] = w < Kw && 4 * w < K ? ld_words4(words + 4 * w) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t j = 4 * (w0 + b * PK_THREADS);
                ready &= (j >= K || (q[b].x >> 26) == tag6) && (j + 1 >= K || (q[b].y >> 26) == tag6) &&
                         (j + 2 >= K || (q[b].z >> 26) == tag6) && (j + 3 >= K || (q[b].w >> 26) == tag6);
            }
            if (ready) break;
            if ((spins & 255) == 0) {
                const uint64_t now = globaltimer();
                if (!g0) g0 = now;
                if ((*((volatile uint32_t*)&ctl->err) & 4u) || now - g0 > 4000000000ull) {
                    atomicOr(&ctl->err, 4u);
                    ok = 0;
                    break;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const uint32_t w = w0 + b * PK_THREADS;
            if (w >= Kw) continue;
            const uint32_t e4[4] = {q[b].x, q[b].y, q[b].z, q[b].w};
            int32_t xv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                xv[e] = 4 * w + e < K ? x_of_word(e4[e]) : 0;
                ss += uint64_t(int64_t(xv[e]) * xv[e]);
            }
            *reinterpret_cast<int4*>(xs32 + 4 * w) = make_int4(xv[0], xv[1], xv[2], xv[3]);
        }
    }
    if (*((volatile uint32_t*)&ctl->err) & 4u) ok = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) s_ss[threadIdx.x >> 5] = ss;
    if (!__syncthreads_and(ok)) return -1;  // also publishes the warp sums
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < PK_WARPS; ++w) t += s_ss[w];
        const int64_t ms = int64_t(((K & (K - 1)) ? t / K : t >> (__ffs(K) - 1)) >> 16);  // d_model 2^k: a shift
        s_r2 = inv_sqrt_q16(ms + 1, seeds);  // ms >= 0: ms + 1 > 0
    }
    __syncthreads();
    if (tr) tr[4] = tr[5] = tr[6] = clock64();
    const int64_t r_inv = s_r2;  // <= 2^24: 32 x 32-bit products
    int fits = 1;
    const int64_t* gk = gamma_unit ? nullptr : gamma;  // mul16(v, ONE) == v: unit gains skipped
    if (!gk) {  // unit gains: 32-bit limbs straight from the product (block-uniform branch)
#pragma unroll 1
        for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
            const int4 e4 = *reinterpret_cast<const int4*>(xs32 + 4 * w);
            const int32_t xs[4] = {e4.x, e4.y, e4.z, e4.w};  // padding slots hold 0
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) lo[e] = norm_lo32(xs[e], int32_t(r_inv), fits);
            put_planes3(planes, Kw, w, lo);
        }
    } else {
#pragma unroll 1
        for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x) {
            const int4 e4 = *reinterpret_cast<const int4*>(xs32 + 4 * w);
            const int32_t xs[4] = {e4.x, e4.y, e4.z, e4.w};  // padding slots hold 0
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t j = 4 * w + e;
                int64_t v = (int64_t(xs[e]) * int32_t(r_inv)) >> 16;
                if (j < K) v = mul16(v, ld_cg64(gk + j));
                fits &= uint64_t(v + (int64_t(1) << 23)) < (uint64_t(1) << 24);
                lo[e] = uint32_t(v);
            }
            put_planes3(planes, Kw, w, lo);
        }
    }
    fits = __syncthreads_and(fits);
    if (tr) tr[7] = clock64();
    if (fits) return 3;
#pragma unroll 1
    for (uint32_t w = threadIdx.x; w < Kw; w += blockDim.x)
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            uint32_t word = 0;
            for (int e = 0; e < 4; ++e) {
                const uint32_t j = 4 * w + e;
                int64_t v = j < K ? (int64_t(xs32[j]) * int32_t(r_inv)) >> 16 : 0;
                if (!gamma_unit && j < K) v = mul16(v, ld_cg64(gamma + j));
                word |= uint32_t((uint64_t(v) >> (8 * k)) & 0xFF) << (8 * e);
            }
            wplanes[k * Kw + w] = word;
        }
    if (threadIdx.x == 0) atomicAdd(&ctl->stats[0], 1ull);
    __syncthreads();
    return 8;
}

// ---- one row group: 4 rows x K against the limb planes ------------------------

// Sums of 4 rows spread over the warp -> every lane gets all 4 (wrapping).
__device__ __forceinline__ void reduce4(uint64_t (&v)[PK_ROWS]) {
    const int lane = threadIdx.x & 31;
    const bool up = lane & 16;
    uint64_t k0 = (up ? v[2] : v[0]) + __shfl_xor_sync(0xffffffffu, up ? v[0] : v[2], 16);
    uint64_t k1 = (up ? v[3] : v[1]) + __shfl_xor_sync(0xffffffffu, up ? v[1] : v[3], 16);
    const bool b8 = lane & 8;
    uint64_t k = (b8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, b8 ? k0 : k1, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    // lane l now holds row ((l >> 4) & 1) * 2 + ((l >> 3) & 1)
#pragma unroll
    for (int r = 0; r < PK_ROWS; ++r) v[r] = __shfl_sync(0xffffffffu, k, ((r >> 1) << 4) | ((r & 1) << 3));
}

template <int L>
__device__ __forceinline__ void group_dot(const Sched& sc, Pipe& p, uint32_t Kp, uint32_t n_segs,
                                          const uint32_t* planes, uint64_t (&out)[PK_ROWS],
                                          int64_t& scale) {
    const int lane = threadIdx.x & 31;
    const uint32_t Kw = Kp / 4;
    const uint32_t planes_s = L == 3 ? smem_u32(planes) : 0u;  // the 3-limb planes are in shared memory
    int32_t acc[PK_ROWS][L];
#pragma unroll
    for (int r = 0; r < PK_ROWS; ++r)
#pragma unroll
        for (int k = 0; k < L; ++k) acc[r][k] = 0;
    for (uint32_t s = 0; s < n_segs; ++s) {
        const uint8_t* slot = pipe_wait(p);
        const uint32_t w = s + 1 < n_segs ? PK_SEG : Kp - (n_segs - 1) * PK_SEG;
        const uint32_t k0 = s * PK_SEG;
        auto pass = [&](uint32_t c) {
            uint4 xl[L];
#pragma unroll
            for (int k = 0; k < L; ++k) {
                if constexpr (L == 3) xl[k] = lds128(planes_s + 4 * (k * Kw + (k0 + c) / 4));  // shared memory
                else xl[k] = *reinterpret_cast<const uint4*>(planes + k * Kw + (k0 + c) / 4);  // wide: global scratch
            }
#pragma unroll
            for (int r = 0; r < PK_ROWS; ++r) {
                const int4 wv = *reinterpret_cast<const int4*>(slot + r * w + c);
#pragma unroll
                for (int k = 0; k < L - 1; ++k) {
                    acc[r][k] = dp4a_su(wv.x, xl[k].x, acc[r][k]);
                    acc[r][k] = dp4a_su(wv.y, xl[k].y, acc[r][k]);
                    acc[r][k] = dp4a_su(wv.z, xl[k].z, acc[r][k]);
                    acc[r][k] = dp4a_su(wv.w, xl[k].w, acc[r][k]);
                }
                acc[r][L - 1] = dp4a_ss(wv.x, xl[L - 1].x, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(wv.y, xl[L - 1].y, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(wv.z, xl[L - 1].z, acc[r][L - 1]);
                acc[r][L - 1] = dp4a_ss(wv.w, xl[L - 1].w, acc[r][L - 1]);
            }
        };
        if (L == 3 && w == PK_SEG) {  // full segment: a fixed trip count, no loop branches
#pragma unroll
            for (int i = 0; i < PK_SEG / 512; ++i) pass(lane * 16 + 512 * i);
        } else {
            for (uint32_t c = lane * 16; c < w; c += 512) pass(c);
        }
        if (s + 1 == n_segs)  // lane r < 4 takes row r's scale from the chunk tail
            scale = lane < PK_ROWS ? *reinterpret_cast<const int64_t*>(slot + PK_ROWS * w + 8 * lane) : 0;
        pipe_release(sc, p);
    }
#ifndef DIMG_EXP_SHFL_REDUCE
    // per-limb warp totals with REDUX: exact in int32 (|sum| <= K * 128 * 255
    // < 2^31 for K <= 65536, the same bound the per-limb accumulation has),
    // then every lane recombines the limbs (wrapping, as the reference's int64)
#pragma unroll
    for (int r = 0; r < PK_ROWS; ++r) {
        uint64_t v = 0;
#pragma unroll
        for (int k = 0; k < L; ++k) v += uint64_t(int64_t(__reduce_add_sync(0xffffffffu, acc[r][k]))) << (8 * k);
        out[r] = v;
    }
#else
#pragma unroll
    for (int r = 0; r < PK_ROWS; ++r) {
        uint64_t v = 0;
#pragma unroll
        for (int k = 0; k < L; ++k) v += uint64_t(int64_t(acc[r][k])) << (8 * k);
        out[r] = v;
    }
    reduce4(out);
#endif
}

// Everything the GEMV loop needs, by value (registers).
struct GemvRT {
    uint32_t epi, rows, Kp, n_groups, n_segs, tag7;
    int64_t* y;
    uint32_t* out_words;      // EPI_SILU: tagged limb words of y
    int64_t* lrow;            // EPI_ARGMAX: this step's logits row
    const int64_t* lut;
    unsigned long long* ssq;  // EPI_RESID: sum-of-squares accumulator
    int32_t* x32;             // EPI_RESID: int32 copy of the clamped x
    uint32_t* xw_out;         // EPI_RESID: tagged residual-stream words out
    const uint32_t* xw_in;    // EPI_RESID: tagged residual words in (nullptr: y / embedding)
    uint32_t tag6_out, tag6_in;
    const int8_t* erow;       // EPI_RESID on layer 0: the token's embedding row
    int64_t es;
    Ctl* ctl;
    unsigned long long* ytag; // EPI_STORE: tagged word pairs of y
    uint64_t tg;              // their tag << 32
    uint32_t vb, vg;          // this CTA of the rank's vg
    uint32_t g_lo, g_hi;      // its row groups (cta_range, precomputed per stage at launch)
    uint32_t row_off;         // EPI_ARGMAX: vocab index of row 0 (tensor parallel: the rank's slice)
    uint32_t tp_buf, tp_tag;  // EPI_RESID, tensor parallel: 1 + inbox buffer (0: single GPU), exchange tag
};

// Tensor parallel: row `row`'s pre-scale accumulator summed over the tp_g
// ranks (wrapping u64 adds: order-free, so every rank gets the same bits).
// This rank's partial goes into slot [buf][tp_rank][row] of every peer's
// inbox as two tagged words; the peers' partials of the same row arrive in
// this rank's inbox the same way (they stream the same row groups in the same
// order, so the wait is the ranks' skew). A peer that never publishes trips
// the 4 s timeout: ctl->err bit 2, the launch fails instead of hanging.
__device__ __forceinline__ uint64_t tp_sum_row(const PkArgs& a, uint32_t buf, uint32_t tag, uint32_t row,
                                               uint32_t rows, uint64_t mine, Ctl* ctl) {
    const uint32_t G = a.tp_g, me = a.tp_rank;
    const uint64_t tg = uint64_t(tag) << 32;
    const size_t out = ((size_t(buf) * G + me) * rows + row) * 2;
#pragma unroll
    for (uint32_t q = 0; q < PK_TP_MAX; ++q)
        if (q < G && q != me) st_tagged2_sys(a.tp_in[q] + out, tg | uint32_t(mine), tg | uint32_t(mine >> 32));
    uint64_t sum = mine;
#pragma unroll
    for (uint32_t q = 0; q < PK_TP_MAX; ++q) {
        if (q >= G || q == me) continue;
        const unsigned long long* w = a.tp_in[me] + ((size_t(buf) * G + q) * rows + row) * 2;
        uint64_t lo, hi;
        uint64_t g0 = 0;
        for (uint32_t spins = 1;; ++spins) {
            ld_tagged2_sys(w, lo, hi);
            if (uint32_t(lo >> 32) == tag && uint32_t(hi >> 32) == tag) break;
            if ((spins & 1023) == 0) {
                const uint64_t now = globaltimer();
                if (!g0) g0 = now;
                if ((*((volatile uint32_t*)&ctl->err) & 4u) || now - g0 > 4000000000ull) {
                    atomicOr(&ctl->err, 4u);
                    break;
                }
            }
        }
        sum += (hi << 32) | (lo & 0xFFFFFFFFull);
    }
    return sum;
}

// All of this CTA's row groups of a GEMV stage, epilogues fused.
template <int L>
__device__ __forceinline__ void run_gemv(const PkArgs& a, const Sched& sc, Pipe& p, const GemvRT& g_,
                                         const uint32_t* planes, uint32_t tag, int64_t& best_v,
                                         uint32_t& best_i) {
    const int lane = threadIdx.x & 31;
    const uint32_t g_lo = g_.g_lo, g_hi = g_.g_hi;
    for (uint32_t g = g_lo + (threadIdx.x >> 5); g < g_hi; g += PK_WARPS) {
        const uint32_t r0 = g * PK_ROWS;
        int64_t resid = 0, scale = 0;  // residual issued now, consumed after the dot product
        uint32_t rw = 0;
        if (g_.epi == EPI_RESID && lane < PK_ROWS && r0 + lane < g_.rows) {
            if (g_.erow) resid = int64_t(uint64_t(int64_t(g_.erow[r0 + lane])) * uint64_t(g_.es));
            else if (g_.xw_in) rw = ld_word(g_.xw_in + r0 + lane);
            else resid = ld_cg64(g_.y + r0 + lane);
        }
        uint64_t v[PK_ROWS];
        group_dot<L>(sc, p, g_.Kp, g_.n_segs, planes, v, scale);
        if (g_.tp_buf && lane < PK_ROWS && r0 + lane < g_.rows) {
            // the row-parallel partials -> the full pre-scale sum (kernels.cpp:18-30 on the whole row)
            uint64_t mine = v[0];
#pragma unroll
            for (int r = 1; r < PK_ROWS; ++r) mine = lane == r ? v[r] : mine;
            const uint64_t tot = tp_sum_row(a, g_.tp_buf - 1, g_.tp_tag, r0 + lane, g_.rows, mine, g_.ctl);
#pragma unroll
            for (int r = 0; r < PK_ROWS; ++r)
                if (lane == r) v[r] = tot;
        }
        uint64_t sq = 0;
        if (g_.epi == EPI_SILU) {
            // rows (2i, 2i+1) = (gate_i, up_i): lanes 0,1 finish pairs 0,1
            const int64_t s_g = __shfl_sync(0xffffffffu, scale, 2 * (lane & 1));
            const int64_t s_u = __shfl_sync(0xffffffffu, scale, 2 * (lane & 1) + 1);
            if (lane < 2 && r0 + 2 * lane + 1 < g_.rows) {
                const uint32_t row = r0 + 2 * lane;
                const int64_t gs = scale_row(int64_t(lane ? v[2] : v[0]), s_g);
                const int64_t us = scale_row(int64_t(lane ? v[3] : v[1]), s_u);
                const int64_t h = mul16(silu_q16(gs, g_.lut), us);
                g_.y[row / 2] = h;
                if (g_.out_words) st_word(g_.out_words + row / 2, limb_word(h, g_.tag7));
            }
        } else if (lane < PK_ROWS && r0 + lane < g_.rows) {
            const uint32_t row = r0 + lane;
            uint64_t acc = v[0];
#pragma unroll
            for (int r = 1; r < PK_ROWS; ++r) acc = lane == r ? v[r] : acc;
            const int64_t val = scale_row(int64_t(acc), scale);
            if (g_.epi == EPI_STORE) {
                g_.y[row] = val;
                if (g_.ytag) st_tagged2(g_.ytag + 2 * row, g_.tg | uint32_t(val), g_.tg | uint32_t(uint64_t(val) >> 32));
            } else if (g_.epi == EPI_RESID) {
                if (g_.xw_in && !g_.erow) {
                    if ((rw >> 26) != g_.tag6_in) rw = poll_word(g_.xw_in + row, g_.tag6_in, 26, g_.ctl);
                    resid = x_of_word(rw);  // published by the previous residual stage
                }
                const int64_t x = add_clamp(resid, val);
                g_.y[row] = x;
                if (g_.x32) g_.x32[row] = int32_t(x);
                if (g_.xw_out) st_word(g_.xw_out + row, x_word(x, g_.tag6_out));
                sq = uint64_t(x * x);  // |x| <= 2^24: x^2 < 2^49, 8192 rows < 2^62
            } else {  // EPI_ARGMAX (vocab row = the rank's first row + row)
                g_.lrow[row] = val;
                if (better(val, g_.row_off + row, best_v, best_i)) {
                    best_v = val;
                    best_i = g_.row_off + row;
                }
            }
        }
        if (g_.epi == EPI_RESID && g_.ssq) {  // this group's rows -> the next rmsnorm's sum of squares
            sq += __shfl_xor_sync(0xffffffffu, sq, 1);
            sq += __shfl_xor_sync(0xffffffffu, sq, 2);
            if (lane == 0 && sq) atomicAdd(g_.ssq, (unsigned long long)sq);
        }
    }
}

// The 8-limb instantiation only runs on out-of-range activations: out of line.
__device__ __forceinline__ void run_gemv_wide(const PkArgs& a, const Sched& sc, Pipe& p, const GemvRT& g_,
                                              const uint32_t* planes, uint32_t tag, int64_t& best_v,
                                              uint32_t& best_i) {
    run_gemv<8>(a, sc, p, g_, planes, tag, best_v, best_i);
}

// ---- attention, positions split across the head's CTAs ---------------------------

__device__ __forceinline__ bool below23(int64_t x) {  // |x| < 2^23
    return uint64_t(x + (int64_t(1) << 23)) < (uint64_t(1) << 24);
}

// Exact general-case pieces of the attention step, out of line (rare, or one
// position): int128 scores of positions [t0, t1) from the int64 cache (the
// newest key from krot), one warp per position.
__device__ __noinline__ void attn_scores_slow(const int64_t* K, const int64_t* qrot, const int64_t* krot,
                                              uint32_t dh, uint32_t t0, uint32_t t1, uint32_t pos,
                                              int64_t inv_scale, int64_t* S) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t t = t0 + warp; t < t1; t += ATTN_THREADS / 32) {
        const int64_t* kt = t == pos ? krot : K + size_t(t) * dh;
        u128 d = 0;
        for (uint32_t j = lane; j < dh; j += 32) d += mul_full(qrot[j], kt[j]);
        d = warp_sum_u128(d);
        if (lane == 0) S[t] = mul16(int64_t(i128(d) >> 16), inv_scale);
    }
}

// PV sums of dims [d0, d1) over all positions from the int64 cache.
__device__ __noinline__ void attn_pv_slow(const int64_t* V, const int64_t* v, const int64_t* S, uint32_t dh,
                                          uint32_t d0, uint32_t d1, uint32_t pos, uint64_t* out) {
    for (uint32_t j = d0 + threadIdx.x; j < d1; j += ATTN_THREADS) {
        uint64_t acc = 0;
        for (uint32_t t = 0; t <= pos; ++t) acc += uint64_t(mul16_prob(S[t], t == pos ? v[j] : V[size_t(t) * dh + j]));
        out[j - d0] = acc;
    }
}

// RoPE of q (and, for the owner, k -> krot and the KV append) for dims past
// what one pass of the block covers (dh > 2 * ATTN_THREADS).
__device__ __noinline__ void attn_rope_tail(const int64_t* q, const int64_t* k, const int64_t* v,
                                            const int64_t* cr, const int64_t* sr, uint32_t dh, bool owner,
                                            int64_t* qrot, int64_t* krot, int64_t* K64, int64_t* V64,
                                            int32_t* K32, int32_t* V32, int* kv_big) {
    const uint32_t half = dh / 2;
    for (uint32_t i = threadIdx.x + ATTN_THREADS; i < half; i += ATTN_THREADS) {
        int64_t x0, x1;
        rope_pair(q[i], q[i + half], cr[i], sr[i], x0, x1);
        qrot[i] = x0;
        qrot[i + half] = x1;
        if (owner) {
            rope_pair(k[i], k[i + half], cr[i], sr[i], x0, x1);
            krot[i] = x0;
            krot[i + half] = x1;
            K64[i] = x0;
            K64[i + half] = x1;
            K32[i] = int32_t(x0);
            K32[i + half] = int32_t(x1);
            *kv_big |= !fits_i32(x0) || !fits_i32(x1);
        }
    }
    if (owner)
        for (uint32_t j = threadIdx.x + ATTN_THREADS; j < dh; j += ATTN_THREADS) {
            V64[j] = v[j];
            V32[j] = int32_t(v[j]);
            *kv_big |= !fits_i32(v[j]);
        }
}

// attention_step (proj/src/kernels.cpp:117-177) for head h as part `pi` of
// `np` CTAs. Each part scores its own contiguous block of cached positions
// (the K strip is read once per head, not once per part), publishes them to
// the head's strip in global memory and meets the other parts at a per-head
// counter; then every part runs the exact softmax over the whole strip in
// shared memory and the probability-weighted V sum for its own slice of the
// head's dimensions. Integer sums throughout: no split moves a bit.
//
// The cache is kept twice: int64 (the reference's values) and an int32
// mirror that the reads use while every value of the head fits (kvwide flag
// clear) -- half the bytes on the latency-critical path. The part owning
// position `pos` appends both rows and maintains the flag (rewritten at
// position 0, sticky after). The int32 rows are loaded speculatively at
// entry, before anything else is known. This runs once per layer under a
// saturated memory system, so the common path is kept short (instruction
// fetches are L2 round trips too); everything else is out of line.
// Returns false if the head's peers never arrived (ctl->err |= 4, as a barrier timeout).
__device__ __forceinline__ bool attn_split(const PkArgs& A, uint32_t layer, uint32_t h, uint32_t pi, uint32_t np,
                                           uint32_t pos, uint32_t epoch, int64_t* scratch, u128* red,
                                           uint32_t* out_words, const int64_t* lut, unsigned long long* tr) {
#define ASTAMP(i) \
    if (tr) tr[i] = clock64()
    ASTAMP(9);
    const uint32_t dh = A.attn.dh, half = dh / 2, H = A.attn.H, D = H * dh, T = pos + 1, mc = A.attn.max_ctx;
    int64_t* qrot = scratch;                                               // [dh]
    int64_t* krot = scratch + dh;                                          // [dh]
    int32_t* q32 = reinterpret_cast<int32_t*>(scratch + 2 * dh);           // [dh]
    int32_t* k32 = q32 + dh;                                               // [dh]
    int64_t* qkv_s = scratch + 3 * dh;                                     // [3][dh] this step's q | k | v
    uint64_t* part = reinterpret_cast<uint64_t*>(scratch + 6 * dh + 257);  // [4 * ATTN_THREADS]
    int64_t* S = reinterpret_cast<int64_t*>(part + 4 * ATTN_THREADS);      // [max_ctx] score strip
    // T <= max_ctx, np <= 64: 32-bit exact; shifts when np is a power of two
    const int nps = A.attn_np_shift;
    const uint32_t t0 = nps >= 0 ? (T * pi) >> nps : T * pi / np, t1 = nps >= 0 ? (T * (pi + 1)) >> nps : T * (pi + 1) / np;
    const bool owner = pi + 1 == np;                        // t1 == T: the newest position is the last part's
    // fast path shape: whole 4-dim quads (16-byte int32 rows), q rows within one pass
    const bool shape_ok = (dh & 3) == 0 && dh <= 512;
    const int64_t* q = qkv_s;
    const int64_t* k = qkv_s + dh;
    const int64_t* v = qkv_s + 2 * dh;
    const size_t hoff = size_t(layer) * A.kv_layer_stride + size_t(h) * mc * dh;
    int64_t* K64 = A.attn.kc + hoff;
    int64_t* V64 = A.attn.vc + hoff;
    int32_t* K32 = A.kc32 + hoff;
    int32_t* V32 = A.vc32 + hoff;
    uint32_t* wflag = A.kvwide + size_t(layer) * H + h;
    const int64_t* cr = A.attn.rope_cos + size_t(pos) * half;
    const int64_t* sr = A.attn.rope_sin + size_t(pos) * half;

    // PV mapping: thread = (4-dim quad jq, position slice sl)
    const uint32_t dpp = A.attn_dpp;
    const uint32_t d0 = min(dh, pi * dpp), d1 = min(dh, d0 + dpp), nd = d1 - d0, nquads = nd / 4;
    const bool pv_shape = shape_ok && nquads > 0 && nquads <= ATTN_THREADS;
    const int nqs = nquads == dpp / 4 ? A.attn_nq_shift : -1;  // the last part may be short
    const uint32_t slices = !pv_shape ? 1 : nqs >= 0 ? ATTN_THREADS >> nqs : ATTN_THREADS / nquads;
    const uint32_t jq = !pv_shape ? 0 : nqs >= 0 ? threadIdx.x & (nquads - 1) : threadIdx.x % nquads;
    const uint32_t sl = !pv_shape ? ATTN_THREADS : nqs >= 0 ? threadIdx.x >> nqs : threadIdx.x / nquads;
    const uint32_t jv = d0 + 4 * jq;

    // 1. The head's wide flag and the RoPE rows (L2); then, speculatively as
    //    int32 from HBM, the K rows of the first score pass and the V rows of
    //    the first PV round -- none of which depends on this step's q/k/v.
    const bool rope_thread = threadIdx.x < half;
    int64_t c_ = 0, s_ = 0;
    uint32_t wide_in = 0;
    if (threadIdx.x == 0) wide_in = ld_cg32(wflag);
    if (rope_thread) {
        c_ = cr[threadIdx.x];
        s_ = sr[threadIdx.x];
    }
    ASTAMP(10);

    const uint32_t oc = threadIdx.x >> 3, e = threadIdx.x & 7;  // scores: octet = position, lane = 4 dims
    constexpr uint32_t NOCT = ATTN_THREADS / 8;
    int4 ka[4], kb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint32_t j = 4 * e + 32 * u, ta = t0 + oc, tb = ta + NOCT;
        ka[u] = (shape_ok && j < dh && ta < t1 && ta != pos) ? *reinterpret_cast<const int4*>(K32 + size_t(ta) * dh + j)
                                                           : make_int4(0, 0, 0, 0);
        kb[u] = (shape_ok && j < dh && tb < t1 && tb != pos) ? *reinterpret_cast<const int4*>(K32 + size_t(tb) * dh + j)
                                                           : make_int4(0, 0, 0, 0);
    }
    constexpr int PV_U = 8;
    int4 vv[PV_U];
#pragma unroll
    for (int u = 0; u < PV_U; ++u) {
        const uint32_t tt = sl + u * slices;
        vv[u] = (sl < slices && tt < pos) ? *reinterpret_cast<const int4*>(V32 + size_t(tt) * dh + jv)
                                          : make_int4(0, 0, 0, 0);
    }
    ASTAMP(11);

    // 2. This step's q/k/v rows of the head, published by the QKV stage as
    //    tagged word pairs (no grid barrier in between): poll them into
    //    shared memory.
    {
        const unsigned long long* W = A.qkv_x;
        const uint64_t tagq = uint32_t(A.tag_base + epoch);
        int ok = 1;
        if (3 * dh <= 2 * ATTN_THREADS) {
            // at most two words per thread: both loads in flight per retry
            const uint32_t i0 = threadIdx.x, i1 = threadIdx.x + ATTN_THREADS;
            const bool h0 = i0 < 3 * dh, h1 = i1 < 3 * dh;
            const size_t r0 = size_t(i0 / dh) * D + size_t(h) * dh + (i0 % dh);
            const size_t r1 = size_t(i1 / dh) * D + size_t(h) * dh + (i1 % dh);
            uint64_t lo0 = tagq << 32, hi0 = tagq << 32, lo1 = tagq << 32, hi1 = tagq << 32;
            uint32_t spins = 0;
            uint64_t g0 = 0;
            for (;;) {
                if (h0) ld_tagged2(W + 2 * r0, lo0, hi0);
                if (h1) ld_tagged2(W + 2 * r1, lo1, hi1);
                if ((lo0 >> 32) == tagq && (hi0 >> 32) == tagq && (lo1 >> 32) == tagq && (hi1 >> 32) == tagq) break;
                if ((++spins & 1023) == 0) {
                    const uint64_t now = globaltimer();
                    if (!g0) g0 = now;
                    if ((*((volatile uint32_t*)&A.ctl->err) & 4u) || now - g0 > 4000000000ull) {
                        atomicOr(&A.ctl->err, 4u);
                        ok = 0;
                        break;
                    }
                }
            }
            if (h0) qkv_s[i0] = int64_t((hi0 << 32) | (lo0 & 0xFFFFFFFFull));
            if (h1) qkv_s[i1] = int64_t((hi1 << 32) | (lo1 & 0xFFFFFFFFull));
        } else
#pragma unroll 1
        for (uint32_t i = threadIdx.x; i < 3 * dh && ok; i += ATTN_THREADS) {
            const uint32_t which = i / dh, j = i - which * dh;
            const size_t row = size_t(which) * D + size_t(h) * dh + j;
            uint64_t lo, hi;
            uint32_t spins = 0;
            uint64_t g0 = 0;
            for (;;) {
                ld_tagged2(W + 2 * row, lo, hi);
                if ((lo >> 32) == tagq && (hi >> 32) == tagq) break;
                if ((++spins & 1023) == 0) {
                    const uint64_t now = globaltimer();
                    if (!g0) g0 = now;
                    if ((*((volatile uint32_t*)&A.ctl->err) & 4u) || now - g0 > 4000000000ull) {
                        atomicOr(&A.ctl->err, 4u);
                        ok = 0;
                        break;
                    }
                }
            }
            qkv_s[i] = int64_t((hi << 32) | (lo & 0xFFFFFFFFull));
        }
        if (!__syncthreads_and(ok)) return false;
    }
    ASTAMP(13);

    // 3. RoPE (rope_apply_inplace, kernels.cpp:70-82) and the KV append (:139-142)
    int q_small = 1, kv_big = 0;
    const int64_t vnew = owner && threadIdx.x < dh ? v[threadIdx.x] : 0;
    if (rope_thread) {
        const uint32_t i = threadIdx.x;
        const int64_t q0 = q[i], q1 = q[i + half];
        int64_t x0, x1;
        rope_pair(q0, q1, c_, s_, x0, x1);
        qrot[i] = x0;
        qrot[i + half] = x1;
        if (shape_ok) {
            q32[i] = int32_t(x0);
            q32[i + half] = int32_t(x1);
        }
        q_small = below23(x0) && below23(x1);
        if (owner) {
            rope_pair(k[i], k[i + half], c_, s_, x0, x1);
            krot[i] = x0;
            krot[i + half] = x1;
            K64[size_t(pos) * dh + i] = x0;
            K64[size_t(pos) * dh + i + half] = x1;
            K32[size_t(pos) * dh + i] = int32_t(x0);
            K32[size_t(pos) * dh + i + half] = int32_t(x1);
            if (shape_ok) {
                k32[i] = int32_t(x0);
                k32[i + half] = int32_t(x1);
            }
            kv_big = !fits_i32(x0) || !fits_i32(x1);
        }
    }
    if (owner && threadIdx.x < dh) {
        V64[size_t(pos) * dh + threadIdx.x] = vnew;
        V32[size_t(pos) * dh + threadIdx.x] = int32_t(vnew);
        kv_big |= !fits_i32(vnew);
    }
    if (dh > 2 * ATTN_THREADS)
        attn_rope_tail(q, k, v, cr, sr, dh, owner, qrot, krot, K64 + size_t(pos) * dh, V64 + size_t(pos) * dh,
                       K32 + size_t(pos) * dh, V32 + size_t(pos) * dh, &kv_big);
    ASTAMP(12);
    // Block-uniform decisions. fast: every |q| < 2^23 and every cached |k|
    // < 2^31 (flag clear), dh <= 512: the int64 score sums are exact
    // (2^23 * 2^31 * 2^9 = 2^63). The owner's own row counts for its path.
    q_small = __syncthreads_and(q_small);
    const int big = __syncthreads_or(kv_big);
    const bool wide = __syncthreads_or(wide_in != 0) || big || !shape_ok;
    if (owner && threadIdx.x == 0 && (pos == 0 || big)) *reinterpret_cast<volatile uint32_t*>(wflag) = big ? 1u : 0u;
    if (owner) __threadfence();  // the appended K/V row is read by the other parts in later steps
    if (tr) tr[4] = clock64();

    // 3. scores of this part's positions (kernels.cpp:143-151); the newest
    //    key (owner only) comes from shared memory. Each score is published
    //    at once as two tagged words for the head's other parts.
    unsigned long long* X = A.xg + size_t(h) * mc * 2;
    const uint32_t tagv = A.tag_base + epoch;
    const uint64_t tg = uint64_t(tagv) << 32;
    if (!wide && q_small) {
        if (owner && (t0 + oc == pos || t0 + oc + NOCT == pos)) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = 4 * e + 32 * u;
                const int4 kk = j < dh ? *reinterpret_cast<const int4*>(k32 + j) : make_int4(0, 0, 0, 0);
                if (t0 + oc == pos) ka[u] = kk;
                else kb[u] = kk;
            }
        }
        for (uint32_t b = t0; b < t1; b += 2 * NOCT) {
            const uint32_t ta = b + oc, tb = ta + NOCT;
            int64_t da = 0, db = 0;
#pragma unroll 1
            for (uint32_t c0 = 0; c0 < dh; c0 += 128) {
                if (b != t0 || c0 != 0) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t j = c0 + 4 * e + 32 * u;
                        const int32_t* pa = ta == pos ? k32 : K32 + size_t(ta) * dh;
                        const int32_t* pb = tb == pos ? k32 : K32 + size_t(tb) * dh;
                        ka[u] = (j < dh && ta < t1) ? *reinterpret_cast<const int4*>(pa + j) : make_int4(0, 0, 0, 0);
                        kb[u] = (j < dh && tb < t1) ? *reinterpret_cast<const int4*>(pb + j) : make_int4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = c0 + 4 * e + 32 * u;
                    const int4 qq = j < dh ? *reinterpret_cast<const int4*>(q32 + j) : make_int4(0, 0, 0, 0);
                    da += int64_t(qq.x) * ka[u].x + int64_t(qq.y) * ka[u].y + int64_t(qq.z) * ka[u].z +
                          int64_t(qq.w) * ka[u].w;
                    db += int64_t(qq.x) * kb[u].x + int64_t(qq.y) * kb[u].y + int64_t(qq.z) * kb[u].z +
                          int64_t(qq.w) * kb[u].w;
                }
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                da += __shfl_xor_sync(0xffffffffu, da, o);
                db += __shfl_xor_sync(0xffffffffu, db, o);
            }
            if (e == 0) {
                if (ta < t1) {
                    const int64_t sc = mul16(da >> 16, A.attn.inv_scale);
                    S[ta] = sc;
                    if (np > 1) st_tagged2(X + 2 * ta, tg | uint32_t(sc), tg | uint32_t(uint64_t(sc) >> 32));
                }
                if (tb < t1) {
                    const int64_t sc = mul16(db >> 16, A.attn.inv_scale);
                    S[tb] = sc;
                    if (np > 1) st_tagged2(X + 2 * tb, tg | uint32_t(sc), tg | uint32_t(uint64_t(sc) >> 32));
                }
            }
        }
    } else {
        attn_scores_slow(K64, qrot, krot, dh, t0, t1, pos, A.attn.inv_scale, S);
        if (threadIdx.x == 0 && wide) atomicAdd(&A.ctl->stats[1], 1ull);
        if (np > 1) {
            __syncthreads();
#pragma unroll 1
            for (uint32_t t = t0 + threadIdx.x; t < t1; t += ATTN_THREADS)
                st_tagged2(X + 2 * t, tg | uint32_t(S[t]), tg | uint32_t(uint64_t(S[t]) >> 32));
        }
    }
    ASTAMP(14);
    if (np > 1) {
        // gather the other parts' scores as their tagged words arrive
        int ok = 1;
#pragma unroll 1
        for (uint32_t t = threadIdx.x; t < T && ok; t += ATTN_THREADS) {
            if (t >= t0 && t < t1) continue;
            uint64_t lo, hi;
            uint32_t spins = 0;
            uint64_t g0 = 0;
            for (;;) {
                ld_tagged2(X + 2 * t, lo, hi);
                if (uint32_t(lo >> 32) == tagv && uint32_t(hi >> 32) == tagv) break;
                if ((++spins & 1023) == 0) {
                    const uint64_t now = globaltimer();
                    if (!g0) g0 = now;
                    if ((*((volatile uint32_t*)&A.ctl->err) & 4u) || now - g0 > 4000000000ull) {
                        atomicOr(&A.ctl->err, 4u);
                        ok = 0;
                        break;
                    }
                }
            }
            S[t] = int64_t((hi << 32) | (lo & 0xFFFFFFFFull));
        }
        ASTAMP(17);
        if (!__syncthreads_and(ok)) return false;
    }
    __syncthreads();
    if (tr) tr[5] = clock64();
    softmax_strip_fast(S, T, lut, red);
    if (tr) tr[6] = clock64();

    // 4. out_j = sum_t mul16(p_t, V[t]_j) (kernels.cpp:153-159) over this
    //    part's dims: p < 2^17 and |v| < 2^31, so p*v is one exact 64-bit
    //    product; the newest row (int64) comes from the projection.
    if (!wide && pv_shape) {
        int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        if (sl < slices) {
            for (uint32_t t = sl; t < pos; t += PV_U * slices) {
                if (t != sl) {
#pragma unroll
                    for (int u = 0; u < PV_U; ++u) {
                        const uint32_t tt = t + u * slices;
                        vv[u] = tt < pos ? *reinterpret_cast<const int4*>(V32 + size_t(tt) * dh + jv) : make_int4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < PV_U; ++u) {
                    const uint32_t tt = t + u * slices;
                    const int64_t p = tt < pos ? S[tt] : 0;
                    a0 += (p * vv[u].x) >> 16;
                    a1 += (p * vv[u].y) >> 16;
                    a2 += (p * vv[u].z) >> 16;
                    a3 += (p * vv[u].w) >> 16;
                }
            }
            if (pos % slices == sl) {  // the newest row
                const int64_t p = S[pos];
                a0 += mul16_prob(p, v[jv]);
                a1 += mul16_prob(p, v[jv + 1]);
                a2 += mul16_prob(p, v[jv + 2]);
                a3 += mul16_prob(p, v[jv + 3]);
            }
        }
        part[4 * threadIdx.x + 0] = uint64_t(a0);
        part[4 * threadIdx.x + 1] = uint64_t(a1);
        part[4 * threadIdx.x + 2] = uint64_t(a2);
        part[4 * threadIdx.x + 3] = uint64_t(a3);
    } else {
        attn_pv_slow(V64, v, S, dh, d0, d1, pos, part);
    }
    ASTAMP(19);
    __syncthreads();
    ASTAMP(20);
    if (!wide && pv_shape && nd * 8 == ATTN_THREADS && (slices & 7) == 0) {
        // eight lanes per output dim, each summing every eighth slice, then a
        // 3-step shuffle tree (instead of one lane walking all the slices)
        const uint32_t j = threadIdx.x >> 3, g = threadIdx.x & 7, qd = j >> 2, z = j & 3;
        uint64_t sum = 0;
#pragma unroll 4
        for (uint32_t s2 = g; s2 < slices; s2 += 8) sum += part[4 * (s2 * nquads + qd) + z];
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        if (g == 0) {
            const uint32_t o = h * dh + d0 + j;
            A.attn.out[o] = int64_t(sum);
            st_word(out_words + o, limb_word(int64_t(sum), tag7_of(A.tag_base + epoch)));
        }
    } else if (threadIdx.x < nd) {
        uint64_t sum = 0;
        if (!wide && pv_shape) {
            const uint32_t qd = threadIdx.x >> 2, z = threadIdx.x & 3;
#pragma unroll 4
            for (uint32_t s2 = 0; s2 < slices; ++s2) sum += part[4 * (s2 * nquads + qd) + z];
        } else {
            sum = part[threadIdx.x];
        }
        const uint32_t o = h * dh + d0 + threadIdx.x;
        A.attn.out[o] = int64_t(sum);  // before the word: read after a grid barrier on the wide path
        st_word(out_words + o, limb_word(int64_t(sum), tag7_of(A.tag_base + epoch)));
    }
    ASTAMP(21);
    __syncthreads();  // scratch is reused by the next head / stage
    if (tr) tr[7] = clock64();
    return true;
#undef ASTAMP
}

// ---- the kernel -------------------------------------------------------------------

// The kernel body for CTA vb of the vg CTAs of one rank (a single-GPU
// launch: blockIdx.x of gridDim.x).
__device__ __forceinline__ void pk_run(const PkArgs& a, const uint32_t vb, const uint32_t vg) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t depth = a.ring_depth;
    uint8_t* slots = smem;                                                // [warps][depth][SLOT]
    uint8_t* stage_mem = smem + size_t(PK_WARPS) * depth * PK_SLOT;       // planes_bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(stage_mem + a.planes_bytes);  // [warps][depth]
    uint32_t* wide_planes = a.wide_planes + size_t(vb) * a.wide_stride;  // 8-limb planes (rare)
    FetchInfo* s_fi = reinterpret_cast<FetchInfo*>(bars + PK_WARPS * PK_MAX_DEPTH);   // [n_layer_stages + 1]
    __shared__ u128 red[32];
    __shared__ int64_t s_bv[PK_WARPS];
    __shared__ uint32_t s_bi[PK_WARPS];
    __shared__ __align__(16) PkStage s_st[2];
    // exp LUT and inv-sqrt seeds live in shared memory for the whole launch
    __shared__ int64_t s_lut[257], s_seeds[64];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Sched sc{a.stages, a.n_layer_stages, a.n_steps, a.n_prefill, s_fi};
    const uint32_t n_stage_all = a.n_layer_stages + (a.n_steps > a.n_prefill ? 1u : 0u);  // + the head
    for (uint32_t i = threadIdx.x; i < n_stage_all; i += PK_THREADS) {
        const PkStage* st = a.stages + i;
        FetchInfo fi{};
        if (st->kind == SK_GEMV) {
            cta_range(st->n_groups, fi.g_lo, fi.g_hi, vb, vg);
            fi.W = st->W;
            fi.n_segs = st->n_segs;
            fi.Kp = st->Kp;
        }
        s_fi[i] = fi;
    }
    Ctl* const ctl = a.ctl;
    if (threadIdx.x < PK_WARPS * depth) mbar_init(&bars[threadIdx.x], 1);
    for (int i = threadIdx.x; i < 257; i += PK_THREADS) s_lut[i] = a.exp_lut[i];
    if (threadIdx.x < 64) s_seeds[threadIdx.x] = a.seeds[threadIdx.x];
    constexpr int kStWords = sizeof(PkStage) / 4;
    static_assert(kStWords <= PK_THREADS, "stage descriptor too large");
    if (threadIdx.x < kStWords)
        reinterpret_cast<uint32_t*>(&s_st[0])[threadIdx.x] = reinterpret_cast<const uint32_t*>(sc.stages)[threadIdx.x];
    fence_proxy_async();
    __syncthreads();

    // prime this warp's pipeline
    Pipe p;
    p.slots = slots + size_t(warp) * depth * PK_SLOT;
    p.bars = bars + warp * depth;
    p.slot = 0;
    p.phase = 0;
    p.depth = depth;
#ifdef DIMG_CHUNK_TRACE
    p.ctn = 0;
#endif
    p.f.step = 0;
    p.f.stage = 0;
    p.f.done = sc.n_steps == 0;
    if (!p.f.done) {
        fetch_load(sc, p.f);
        fetch_settle(sc, p.f);
    }
    for (uint32_t d = 0; d < depth && !p.f.done; ++d) {
        if (lane == 0) fetch_issue(p.f, p.slots + d * PK_SLOT, &p.bars[d]);
        fetch_advance(sc, p.f);
    }

    uint32_t pos = ctl->pos;
    const uint32_t logit_base = ctl->logit_base, keep_cap = ctl->keep_cap;
    uint32_t token = a.tokens[pos];
    uint32_t nbar = 0, cur = 0, attn_epoch = 0, nseq = 0;

    for (uint32_t step = 0; step < sc.n_steps; ++step) {
        const uint32_t nst = stages_in_step(sc, step);
        const uint32_t tag = step + 1;
        int64_t best_v = INT64_MIN;
        uint32_t best_i = 0xFFFFFFFFu;
        for (uint32_t si = 0; si < nst; ++si) {
            const PkStage st = s_st[cur];  // by value: registers for the whole stage
            // the next stage's descriptor: loaded now, stored before the barrier
            uint32_t next_word = 0;
            if (threadIdx.x < kStWords)
                next_word = reinterpret_cast<const uint32_t*>(sc.stages + (si + 1 < nst ? si + 1 : 0))[threadIdx.x];
            unsigned long long* tr =
                a.trace && vb == 0 && threadIdx.x == 0 && nseq < a.trace_cap ? a.trace + 32 * nseq : nullptr;
            ++nseq;
            if (tr) {
                tr[8] = clock64();
                tr[0] = globaltimer();
            }
#ifdef DIMG_CHUNK_TRACE
            if (threadIdx.x == 0 && blockIdx.x < 148 && p.ctn < CT_MAX) {
                g_ct[blockIdx.x][p.ctn][0] = clock64();
                g_ct[blockIdx.x][p.ctn][1] = (1ull << 63) | (uint64_t(si) << 8) | 0;
                ++p.ctn;
            }
#endif
            if (st.kind == SK_ATTN) {
                const uint32_t np = a.attn_parts;
                ++attn_epoch;
                for (uint32_t c = vb; c < a.attn.H * np; c += vg)
                    if (!attn_split(a, st.layer, c / np, c % np, np, pos, attn_epoch,
                                    reinterpret_cast<int64_t*>(stage_mem), red, st.out_words, s_lut,
                                    tr && c == 0 ? tr : nullptr))
                        return;
            } else {
                uint32_t* planes;
                int L;
                if (st.mode == MODE_PLAIN) {
                    planes = reinterpret_cast<uint32_t*>(stage_mem);
                    L = prologue_plain(st.K, st.Kp, st.x, st.in_words, tag7_of(a.tag_base + attn_epoch), planes,
                                       wide_planes, ctl);
                    if (L < 0) return;
                    if (L == PLAIN_WIDE) {  // grid-uniform: the int64 vector is visible after the barrier
                        if (!grid_sync(a.bar, ctl, nbar++, vg)) return;
                        L = planes_from_x(st.K, st.Kp, st.x, planes, wide_planes, ctl, true);
                    }
                } else {
                    // Stages are not always separated by grid barriers: a CTA
                    // without rows here must not read x / the sums at all (it
                    // could lag behind their next writers). The embedding is
                    // written by the CTA holding group 0.
                    const uint32_t glo = s_fi[si].g_lo, ghi = s_fi[si].g_hi;  // cta_range at launch
                    int64_t* xb = reinterpret_cast<int64_t*>(stage_mem);
                    planes = reinterpret_cast<uint32_t*>(xb + st.Kp);
                    L = 3;
                    if (glo < ghi && st.xw_in) {
                        L = prologue_norm_words(st.K, st.Kp, st.gamma_unit != 0, st.gamma, st.xw_in,
                                                tag6_of(a.tag_base + attn_epoch - st.xw_lag),
                                                reinterpret_cast<int32_t*>(xb), planes, wide_planes, s_seeds, ctl,
                                                tr);
                        if (L < 0) return;
                    } else if (glo < ghi) {
                        const bool embed = st.mode == MODE_EMBED;
                        L = prologue_norm(st.K, st.Kp, st.gamma_unit != 0, st.x, st.gamma,
                                          embed ? a.embd + size_t(token) * st.K : nullptr,
                                          embed ? a.embd_scales[token] : 0,
                                          embed && glo == 0 ? a.x_resid : nullptr, xb, planes, wide_planes,
                                          red, s_seeds, ctl, tr, st.ssq_in, st.x32_in);
                    }
                }
                if (L == 8) planes = wide_planes;  // out-of-range inputs: 8 planes in the global scratch
                // the sum the previous stages' prologues consumed: every reader
                // is done once this stage's inputs are complete
                if (st.ssq_clear && vb == 0 && threadIdx.x == 0) *st.ssq_clear = 0;
                if (tr) tr[1] = globaltimer();
#ifdef DIMG_CHUNK_TRACE
                if (threadIdx.x == 0 && blockIdx.x < 148 && p.ctn < CT_MAX) {
                    g_ct[blockIdx.x][p.ctn][0] = clock64();
                    g_ct[blockIdx.x][p.ctn][1] = (1ull << 63) | (uint64_t(si) << 8) | 1;
                    ++p.ctn;
                }
#endif
                if (a.trace_all && threadIdx.x == 0 && nseq - 1 < a.trace_cap)
                    a.trace_all[(size_t(nseq - 1) * vg + vb) * 2] = globaltimer();
                GemvRT g_;
                g_.epi = st.epi; g_.rows = st.rows; g_.Kp = st.Kp; g_.n_groups = st.n_groups;
                g_.n_segs = st.n_segs; g_.tag7 = tag7_of(a.tag_base + attn_epoch); g_.y = st.y;
                g_.out_words = st.out_words; g_.lut = s_lut;
                g_.lrow = nullptr;
                g_.ssq = st.ssq_out;
                g_.x32 = st.x32_out;
                g_.xw_out = st.xw_out;
                g_.xw_in = st.xw_in;
                g_.tag6_out = tag6_of(a.tag_base + attn_epoch);
                g_.tag6_in = tag6_of(a.tag_base + attn_epoch - st.xw_lag);
                g_.erow = st.resid_embed ? a.embd + size_t(token) * st.rows : nullptr;
                g_.es = st.resid_embed ? a.embd_scales[token] : 0;
                g_.ctl = ctl;
                g_.ytag = st.ytag;
                g_.vb = vb;
                g_.vg = vg;
                g_.g_lo = s_fi[si].g_lo;
                g_.g_hi = s_fi[si].g_hi;
                g_.row_off = a.vocab_off;
                g_.tp_buf = a.tp_g > 1 ? st.tp_sum : 0u;
                g_.tp_tag = a.tag_base + attn_epoch;
                g_.tg = uint64_t(a.tag_base + attn_epoch + 1) << 32;  // the coming attention stage's tag
                if (st.epi == EPI_ARGMAX) {
                    uint32_t slot = pos - logit_base;
                    slot = slot < keep_cap ? slot : keep_cap;
                    g_.lrow = st.y + size_t(slot) * st.rows;
                }
                if (L == 3) run_gemv<3>(a, sc, p, g_, planes, tag, best_v, best_i);
                else run_gemv_wide(a, sc, p, g_, planes, tag, best_v, best_i);
                if (tr) tr[2] = globaltimer();
#ifdef DIMG_CHUNK_TRACE
                if (threadIdx.x == 0 && blockIdx.x < 148 && p.ctn < CT_MAX) {
                    g_ct[blockIdx.x][p.ctn][0] = clock64();
                    g_ct[blockIdx.x][p.ctn][1] = (1ull << 63) | (uint64_t(si) << 8) | 2;
                    ++p.ctn;
                }
#endif
                if (a.trace_all && threadIdx.x == 0 && nseq - 1 < a.trace_cap)
                    a.trace_all[(size_t(nseq - 1) * vg + vb) * 2 + 1] = globaltimer();
                if (st.epi == EPI_ARGMAX) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        int64_t ov = __shfl_xor_sync(0xffffffffu, best_v, o);
                        uint32_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
                        if (better(ov, oi, best_v, best_i)) { best_v = ov; best_i = oi; }
                    }
                    if (lane == 0) { s_bv[warp] = best_v; s_bi[warp] = best_i; }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        for (int w2 = 1; w2 < PK_WARPS; ++w2)
                            if (better(s_bv[w2], s_bi[w2], best_v, best_i)) { best_v = s_bv[w2]; best_i = s_bi[w2]; }
                        a.parts[vb].v = best_v;
                        a.parts[vb].idx = best_i;
                        const uint64_t tg = uint64_t(a.tag_base + attn_epoch) << 32;
                        if (a.tp_g > 1) {
                            // tensor parallel: this CTA's pair into slot tp_rank * vg + vb of every rank
                            const size_t o = (size_t(step & 1) * a.tp_g * vg + size_t(a.tp_rank) * vg + vb) * 4;
#pragma unroll
                            for (uint32_t q = 0; q < PK_TP_MAX; ++q)
                                if (q < a.tp_g) {
                                    st_tagged2_sys(a.tp_parts[q] + o, tg | uint32_t(uint64_t(best_v)),
                                                   tg | uint32_t(uint64_t(best_v) >> 32));
                                    st_tagged2_sys(a.tp_parts[q] + o + 2, tg | best_i, tg);
                                }
                        } else if (a.parts_w) {  // tagged copy: the next token needs no grid barrier
                            unsigned long long* pw = a.parts_w + (size_t(step & 1) * vg + vb) * 4;
                            st_tagged2(pw, tg | uint32_t(uint64_t(best_v)), tg | uint32_t(uint64_t(best_v) >> 32));
                            st_tagged2(pw + 2, tg | best_i, tg);
                        }
                    }
                }
            }
            if (tr) tr[3] = globaltimer();
            __syncthreads();  // everyone has its register copy of s_st[cur]; safe to overwrite the other
            if (threadIdx.x < kStWords) reinterpret_cast<uint32_t*>(&s_st[cur ^ 1])[threadIdx.x] = next_word;
            cur ^= 1;
            if (st.no_barrier) __syncthreads();  // the next descriptor is complete before anyone reads it
            else if (!grid_sync(a.bar, ctl, nbar++, vg)) return;
        }
        if (step >= sc.n_prefill) {
            // every CTA reduces the lm_head partials itself (no extra barrier)
            int64_t bv = INT64_MIN;
            uint32_t bi = 0xFFFFFFFFu;
            const uint32_t ptag = a.tag_base + attn_epoch;
            const bool tp = a.tp_g > 1;
            const uint32_t n_parts = tp ? a.tp_g * vg : vg;  // every rank's CTAs
            for (uint32_t b = threadIdx.x; b < n_parts; b += blockDim.x) {
                int64_t v;
                uint32_t i;
                if (a.parts_w) {
                    const unsigned long long* pw = a.parts_w + (size_t(step & 1) * n_parts + b) * 4;
                    uint64_t w0, w1, w2, w3;
                    uint32_t spins = 0;
                    for (;;) {
                        if (tp) {
                            ld_tagged2_sys(pw, w0, w1);
                            ld_tagged2_sys(pw + 2, w2, w3);
                        } else {
                            ld_tagged2(pw, w0, w1);
                            ld_tagged2(pw + 2, w2, w3);
                        }
                        if (uint32_t(w0 >> 32) == ptag && uint32_t(w1 >> 32) == ptag && uint32_t(w2 >> 32) == ptag) break;
                        if ((++spins & 1023) == 0 && (*((volatile uint32_t*)&ctl->err) & 4u)) break;
                        if ((spins & 0xFFFFF) == 0) atomicOr(&ctl->err, 4u);  // ~seconds: give up
                    }
                    v = int64_t((w1 << 32) | (w0 & 0xFFFFFFFFull));
                    i = uint32_t(w2);
                } else {
                    v = ld_cg64(&a.parts[b].v);
                    i = ld_cg32(&a.parts[b].idx);
                }
                if (better(v, i, bv, bi)) { bv = v; bi = i; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
                uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            __syncthreads();
            if (lane == 0) { s_bv[warp] = bv; s_bi[warp] = bi; }
            __syncthreads();
            for (int w2 = 0; w2 < PK_WARPS; ++w2)
                if (better(s_bv[w2], s_bi[w2], bv, bi)) { bv = s_bv[w2]; bi = s_bi[w2]; }
            token = bi;
            if (vb == 0 && threadIdx.x == 0) a.tokens[pos + 1] = token;
        } else {
            token = a.tokens[pos + 1];
        }
        ++pos;
    }
    if (vb == 0 && threadIdx.x == 0) ctl->pos = pos;
}

__global__ void __launch_bounds__(PK_THREADS, 1) decode_persistent_kernel(const PkArgs a) {
    pk_run(a, blockIdx.x, gridDim.x);
}

// A tensor-parallel group on ONE device (the in-process backend that tests
// the sharded program without more GPUs): one cooperative launch of
// g x vg CTAs, CTAs [r vg, (r + 1) vg) running rank r with its own arguments
// (copied to shared memory), so ranks that wait on one another are
// co-resident by construction.
__global__ void __launch_bounds__(PK_THREADS, 1) decode_persistent_group_kernel(const PkArgs* __restrict__ ranks,
                                                                               uint32_t vg) {
    __shared__ __align__(16) PkArgs s_a;
    const uint32_t r = blockIdx.x / vg;
    constexpr int kWords = sizeof(PkArgs) / 4;
    for (int i = threadIdx.x; i < kWords; i += PK_THREADS)
        reinterpret_cast<uint32_t*>(&s_a)[i] = reinterpret_cast<const uint32_t*>(ranks + r)[i];
    __syncthreads();
    pk_run(s_a, blockIdx.x - r * vg, vg);
}

}  // namespace dimg::dev
