// Tensor-parallel generation (BASELINE config C4): one model
// sharded Megatron-style over g ranks (dimg_model_upload's tp_rank/tp_size),
// each decode step a chain of per-stage kernels per rank with two exchanges
// per layer (the pre-scale WO / w_down accumulators) and one per token (the
// lm_head's (max, index) pair), see kernels/tp.cuh for the exactness argument.
//
// Two collective backends behind one step program:
//   DIMG_TP_NCCL   one process per GPU (torchrun), this process = rank r:
//                  ncclAllReduce (uint64 sum: wrapping, order-free) of the
//                  4096 accumulators in place, ncclAllGather of the 16-byte
//                  argmax pairs. NCCL is loaded with dlopen (the copy torch
//                  already mapped, else the system libnccl.so.2), so
//                  libdimg has no link-time NCCL dependency.
//   DIMG_TP_LOCAL  all g shards on one device in this process, one stream:
//                  each rank's raw GEMV writes its own slot of a [g][D]
//                  buffer and every rank's residual kernel sums the g slots
//                  -- the same arithmetic as the all-reduce, with no kernel
//                  ever waiting on another, so the sharded kernels are
//                  testable on one GPU (tests/test_gpu_tp.py: C4 and C2
//                  hashes at g = 2, 4, 8).
// Each step (all ranks on this process) is captured once as a CUDA graph
// (with and without the lm_head) and replayed; positions and tokens live in
// device memory, as for the single-GPU engine.
//
// The fused backends run the single-GPU persistent decode kernel on each
// rank's shard instead (one launch per generation), with the two
// all-reduces per layer and the argmax gather done inside it over peer
// memory (kernels/persistent.cuh tp_sum_row; no collective library):
//   DIMG_TP_FUSED_IPC    one process per GPU; each rank allocates one
//                  exchange block (inbox [2][g][D][2] + lm_head slots
//                  [2][g * grid][4], tagged 8-byte words) and maps its
//                  peers' with CUDA IPC handles the caller distributes.
//   DIMG_TP_FUSED_LOCAL  every shard on one device; one cooperative launch
//                  of g x (SMs / g) CTAs, each CTA running its rank's
//                  arguments (decode_persistent_group_kernel), so ranks that
//                  wait on each other are resident together by construction.
#include <dlfcn.h>
#include <nccl.h>

#include "kernels/tp.cuh"

namespace {

// ---- NCCL through dlopen ------------------------------------------------------
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string why;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.all_reduce, "ncclAllReduce");
        sym(a.all_gather, "ncclAllGather");
        sym(a.error_string, "ncclGetErrorString");
        if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.all_gather ||
            !a.error_string)
            a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    if (!api.why.empty()) fail(DIMG_ENCCL, api.why);
    return api;
}

#define NK(expr)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (expr);                                                                  \
        if (r_ != ncclSuccess) fail(DIMG_ENCCL, std::string(#expr) + ": " + nccl_api().error_string(r_)); \
    } while (0)

// ---- one rank's device state ---------------------------------------------------
struct TpRank {
    std::unique_ptr<dimg_model, dimg_status (*)(dimg_model*)> m{nullptr, dimg_model_free};
    DevBuf mem;
    int64_t *x = nullptr, *qkv = nullptr, *att = nullptr, *h = nullptr, *acc = nullptr;
    int64_t *kc = nullptr, *vc = nullptr, *scores = nullptr, *row = nullptr, *keep = nullptr;
    unsigned long long* best = nullptr;  // [2] this rank's (max, index) pair
    uint32_t* tokens = nullptr;
    Ctl* ctl = nullptr;
    std::vector<GemvArgs> qkv_a, wo_a, gu_a, dn_a;
    std::vector<AttnArgs> at_a;
    GemvArgs head_a{};
    // fused backends: the shard's persistent-kernel session and its
    // exchange block (released before the model: declared after it)
    dimg_session* s = nullptr;
    unsigned long long* xch = nullptr;
    ~TpRank() { delete s; }
};

}  // namespace

struct dimg_tp {
    int backend = DIMG_TP_LOCAL;
    int device = 0;
    uint32_t g = 1;             // tensor-parallel degree
    int rank = 0;               // NCCL: this process's rank
    DevCtx* ctx = nullptr;
    cudaStream_t st = nullptr;
    std::vector<std::unique_ptr<TpRank>> ranks;  // LOCAL: g shards; NCCL: this rank's
    DevBuf mem;
    int64_t* parts = nullptr;              // LOCAL: [g][D] raw partials of the row-parallel GEMVs
    unsigned long long* pairs = nullptr;   // [g][2] gathered argmax pairs
    ncclComm_t comm = nullptr;
    uint32_t D = 0, V = 0, L = 0, vmax = 0, keep_cap = 0, ctx_len = 0;
    uint32_t n_prompt = 0, max_new = 0, len = 0;
    cudaGraphExec_t graph_head = nullptr, graph_prompt = nullptr;
    uint64_t launches_per_step = 0;
    // fused backends
    bool fused = false, connected = false;
    uint32_t vg = 0;                          // CTAs per rank
    size_t inbox_elems = 0, slot_elems = 0;   // u64 words of the exchange block's two parts
    std::vector<unsigned long long*> xch;     // every rank's exchange block (own or peer-mapped)
    std::vector<void*> ipc_open;              // mapped peer blocks
    PkArgs* d_args = nullptr;                 // FUSED_LOCAL: the ranks' kernel arguments
    ~dimg_tp() {
        for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
        if (graph_head) cudaGraphExecDestroy(graph_head);
        if (graph_prompt) cudaGraphExecDestroy(graph_prompt);
        if (comm) nccl_api().comm_destroy(comm);
        if (st) cudaStreamDestroy(st);
    }
};

namespace {

bool tp_graphs_enabled() {
    const char* e = std::getenv("DIMG_TP_GRAPH");
    return !e || std::atoi(e) != 0;
}

void tp_build_rank(dimg_tp& t, TpRank& r) {
    const dimg_model& m = *r.m;
    const uint32_t D = m.D, L = m.L, ctx = m.cfg.max_ctx;
    r.x = r.mem.alloc<int64_t>(D);
    r.qkv = r.mem.alloc<int64_t>(3 * size_t(m.Dl));
    r.att = r.mem.alloc<int64_t>(m.Dl);
    r.h = r.mem.alloc<int64_t>(m.Fl);
    r.acc = r.mem.alloc<int64_t>(D);
    const size_t kv_layer = size_t(m.Hl) * ctx * m.dh;
    r.kc = r.mem.alloc<int64_t>(kv_layer * L);
    r.vc = r.mem.alloc<int64_t>(kv_layer * L);
    r.scores = r.mem.alloc<int64_t>(size_t(m.Hl) * ctx);
    r.row = r.mem.alloc<int64_t>(t.vmax);
    r.keep = t.keep_cap ? r.mem.alloc<int64_t>(size_t(t.keep_cap) * t.vmax) : nullptr;
    if (r.keep) CK(cudaMemset(r.keep, 0, size_t(t.keep_cap) * t.vmax * 8));  // gathered padding stays 0
    r.best = r.mem.alloc<unsigned long long>(2);
    r.tokens = r.mem.alloc<uint32_t>(size_t(ctx) + 1);
    r.ctl = r.mem.alloc<Ctl>(1);
    CK(cudaMemset(r.ctl, 0, sizeof(Ctl)));
    CK(cudaMemset(r.tokens, 0, (size_t(ctx) + 1) * 4));
    const uint32_t ri = uint32_t(m.tp_rank);
    auto base = [&](const DevMat& W, uint32_t mode) {
        GemvArgs a{};
        a.W = W.rm;
        a.scales = W.s;
        a.rows = W.rows;
        a.K = W.K;
        a.Kp = W.Kp;
        a.ctl = r.ctl;
        a.exp_lut = m.ctx->exp_lut;
        a.seeds = m.ctx->seeds;
        if (mode == MODE_EMBED) {
            a.embd = m.embd;
            a.embd_scales = m.embd_s;
            a.tokens = r.tokens;
            a.x_out = r.x;
        }
        return a;
    };
    // the row-parallel GEMVs' raw partials: this rank's own acc (NCCL) or its
    // slot of the shared [g][D] buffer (LOCAL)
    int64_t* raw_out = t.backend == DIMG_TP_LOCAL ? t.parts + size_t(ri) * D : r.acc;
    for (uint32_t l = 0; l < L; ++l) {
        const auto& lw = m.layers[l];
        GemvArgs q = base(lw.qkv, l == 0 ? MODE_EMBED : MODE_NORM);
        q.x = r.x;
        q.gamma = lw.attn_norm;
        q.y = r.qkv;
        r.qkv_a.push_back(q);
        AttnArgs at{};
        at.qkv = r.qkv;
        at.kc = r.kc + l * kv_layer;
        at.vc = r.vc + l * kv_layer;
        at.rope_cos = m.rope_cos;
        at.rope_sin = m.rope_sin;
        at.scores = r.scores;
        at.out = r.att;
        at.ctl = r.ctl;
        at.H = m.Hl;
        at.dh = m.dh;
        at.max_ctx = ctx;
        at.inv_scale = m.inv_scale;
        at.exp_lut = m.ctx->exp_lut;
        r.at_a.push_back(at);
        GemvArgs wo = base(lw.wo, MODE_PLAIN);
        wo.x = r.att;
        wo.y = raw_out;
        r.wo_a.push_back(wo);
        GemvArgs gu = base(lw.gu, MODE_NORM);
        gu.x = r.x;
        gu.gamma = lw.ffn_norm;
        gu.y = r.h;
        r.gu_a.push_back(gu);
        GemvArgs dn = base(lw.down, MODE_PLAIN);
        dn.x = r.h;
        dn.y = raw_out;
        r.dn_a.push_back(dn);
    }
    r.head_a = base(m.head, MODE_NORM);
    r.head_a.x = r.x;
    r.head_a.gamma = m.final_norm;
    r.head_a.y = r.row;
}

// Enqueues one forward step of every local rank on t.st (with the lm_head and
// the greedy pick, or a prompt step that only advances the position).
uint64_t tp_enqueue_step(dimg_tp& t, bool head) {
    const cudaStream_t st = t.st;
    const DevCtx& c = *t.ctx;
    const bool local = t.backend == DIMG_TP_LOCAL;
    const uint32_t D = t.D;
    uint64_t n = 0;
    auto exchange = [&]() {  // the all-reduce of the row-parallel partials
        if (local || t.g == 1) return;
        TpRank& r = *t.ranks[0];
        NK(nccl_api().all_reduce(r.acc, r.acc, D, ncclUint64, ncclSum, t.comm, st));
        ++n;
    };
    auto resid = [&](TpRank& r, const int64_t* s) {
        const int64_t* src = local ? t.parts : r.acc;
        const uint32_t np = local ? t.g : 1;
        tp_resid_kernel<<<(D + 255) / 256, 256, 0, st>>>(r.x, src, np, D, s, D);
        ++n;
    };
    for (uint32_t l = 0; l < t.L; ++l) {
        for (auto& rp : t.ranks) {
            TpRank& r = *rp;
            if (l == 0) launch_gemv<EPI_STORE, MODE_EMBED>(r.qkv_a[l], c, st);
            else launch_gemv<EPI_STORE, MODE_NORM>(r.qkv_a[l], c, st);
            attn_decode_kernel<<<r.at_a[l].H, ATTN_THREADS, attn_op_scratch_bytes(r.at_a[l].dh), st>>>(r.at_a[l]);
            launch_gemv<EPI_RAW, MODE_PLAIN>(r.wo_a[l], c, st);
            n += 3;
        }
        exchange();
        for (auto& rp : t.ranks) resid(*rp, rp->m->layers[l].wo.s);
        for (auto& rp : t.ranks) {
            TpRank& r = *rp;
            launch_gemv<EPI_SILU, MODE_NORM>(r.gu_a[l], c, st);
            launch_gemv<EPI_RAW, MODE_PLAIN>(r.dn_a[l], c, st);
            n += 2;
        }
        exchange();
        for (auto& rp : t.ranks) resid(*rp, rp->m->layers[l].down.s);
    }
    if (head) {
        for (auto& rp : t.ranks) {
            TpRank& r = *rp;
            launch_gemv<EPI_STORE, MODE_NORM>(r.head_a, c, st);
            unsigned long long* best = local ? t.pairs + 2 * size_t(r.m->tp_rank) : r.best;
            tp_argmax_kernel<<<1, TP_ARG_THREADS, 0, st>>>(r.row, r.m->Vl, r.m->v0, r.ctl, r.keep, t.vmax, best);
            n += 2;
        }
        if (!local) {
            TpRank& r = *t.ranks[0];
            if (t.g > 1) NK(nccl_api().all_gather(r.best, t.pairs, 2, ncclUint64, t.comm, st));
            else CK(cudaMemcpyAsync(t.pairs, r.best, 16, cudaMemcpyDeviceToDevice, st));
            ++n;
        }
        for (auto& rp : t.ranks) {
            tp_pick_kernel<<<1, 1, 0, st>>>(t.pairs, t.g, rp->tokens, rp->ctl);
            ++n;
        }
    } else {
        for (auto& rp : t.ranks) {
            advance_pos_kernel<<<1, 1, 0, st>>>(rp->ctl);
            ++n;
        }
    }
    CK(cudaGetLastError());
    return n;
}

// Instantiates the step graph (with or without the lm_head) once.
void tp_ensure_graph(dimg_tp& t, bool head) {
    cudaGraphExec_t& ge = head ? t.graph_head : t.graph_prompt;
    if (ge || !tp_graphs_enabled()) return;
    cudaGraph_t gr = nullptr;
    CK(cudaStreamBeginCapture(t.st, cudaStreamCaptureModeThreadLocal));
    uint64_t n = 0;
    try {
        n = tp_enqueue_step(t, head);
    } catch (...) {
        cudaStreamEndCapture(t.st, &gr);
        if (gr) cudaGraphDestroy(gr);
        throw;
    }
    CK(cudaStreamEndCapture(t.st, &gr));
    CK(cudaGraphInstantiate(&ge, gr, 0));
    cudaGraphDestroy(gr);
    if (head) t.launches_per_step = n;
}

void tp_run_steps(dimg_tp& t, bool head, uint32_t steps) {
    if (steps == 0) return;
    if (!tp_graphs_enabled()) {
        for (uint32_t i = 0; i < steps; ++i) {
            const uint64_t n = tp_enqueue_step(t, head);
            if (head) t.launches_per_step = n;
        }
        return;
    }
    tp_ensure_graph(t, head);
    cudaGraphExec_t ge = head ? t.graph_head : t.graph_prompt;
    for (uint32_t i = 0; i < steps; ++i) CK(cudaGraphLaunch(ge, t.st));
}

void tp_begin(dimg_tp& t, const uint32_t* prompt, uint32_t p, uint32_t n, bool keep) {
    const dimg_model& m = *t.ranks[0]->m;
    check_prompt(m, prompt, p, n);
    if (keep && n > t.keep_cap) fail(DIMG_EINVAL, "tp generate: keep_logits beyond the group's keep_logits_cap");
    CK(cudaSetDevice(t.device));
    const uint32_t hdr[5] = {0, p - 1, keep ? n : 0, 0, 0};
    for (auto& rp : t.ranks) {
        CK(cudaMemcpyAsync(rp->tokens, prompt, size_t(p) * 4, cudaMemcpyHostToDevice, t.st));
        CK(cudaMemcpyAsync(rp->ctl, hdr, sizeof hdr, cudaMemcpyHostToDevice, t.st));
    }
    t.n_prompt = p;
    t.max_new = n;
    t.len = 0;
}

void tp_check_err(dimg_tp& t) {
    CK(cudaStreamSynchronize(t.st));
    for (auto& rp : t.ranks) {
        uint32_t err = 0;
        CK(cudaMemcpy(&err, &rp->ctl->err, 4, cudaMemcpyDeviceToHost));
        if (err & 1u) fail(DIMG_EDOMAIN, "inv_sqrt_q16: input must be positive");
    }
}

// Prompt steps (positions 0 .. P-2) then max_new lm_head steps.
void tp_generate(dimg_tp& t) {
    tp_run_steps(t, false, t.n_prompt - 1);
    tp_run_steps(t, true, t.max_new);
    t.len = t.n_prompt - 1 + t.max_new;
}

// The kept logits [max_new][V] in host memory: every rank's slice.
void tp_gather_logits(dimg_tp& t, int64_t* out) {
    const uint32_t n = t.max_new;
    if (t.backend == DIMG_TP_LOCAL) {
        for (auto& rp : t.ranks)
            CK(cudaMemcpy2DAsync(out + rp->m->v0, size_t(t.V) * 8, rp->keep, size_t(t.vmax) * 8, size_t(rp->m->Vl) * 8,
                                 n, cudaMemcpyDeviceToHost, t.st));
        CK(cudaStreamSynchronize(t.st));
        return;
    }
    int64_t* all = t.mem.alloc<int64_t>(size_t(t.g) * t.keep_cap * t.vmax);
    TpRank& r = *t.ranks[0];
    NK(nccl_api().all_gather(r.keep, all, size_t(t.keep_cap) * t.vmax, ncclInt64, t.comm, t.st));
    const uint32_t V = t.V, g = t.g;
    for (uint32_t q = 0; q < g; ++q) {
        const uint32_t v0 = uint32_t(uint64_t(V) * q / g), vl = uint32_t(uint64_t(V) * (q + 1) / g) - v0;
        CK(cudaMemcpy2DAsync(out + v0, size_t(V) * 8, all + size_t(q) * t.keep_cap * t.vmax, size_t(t.vmax) * 8,
                             size_t(vl) * 8, n, cudaMemcpyDeviceToHost, t.st));
    }
    CK(cudaStreamSynchronize(t.st));
}

// ---- fused backends --------------------------------------------------------------

// Experiment knob (tools/tp_fused_probe.py --solo): DIMG_TP_SOLO=1 runs a
// DIMG_TP_FUSED_IPC rank alone, WITHOUT the exchange (tp_g forced to 1): the
// per-GPU cost of a g-way shard on a whole GPU, minus the peer latency. Its
// tokens are wrong by construction (partial sums); never a product path.
bool tp_solo() {
    const char* e = std::getenv("DIMG_TP_SOLO");
    return e && std::atoi(e) != 0;
}

void tpf_require_connected(const dimg_tp& t) {
    if (t.fused && !t.connected) fail(DIMG_ELOGIC, "tp: dimg_tp_connect the group before generating");
}

// One persistent launch of n_steps forward steps (the first n_prefill
// without the lm_head) on every rank of this process.
void tpf_launch(dimg_tp& t, uint32_t n_steps, uint32_t n_prefill) {
    if (n_steps == 0) return;
    tpf_require_connected(t);
    const uint64_t n_attn = uint64_t(n_steps) * t.L;
    std::vector<PkArgs> args;
    for (auto& rp : t.ranks) {
        dimg_session& s = *rp->s;
        const dimg_model& m = *rp->m;
        if (uint64_t(s.attn_tag) + n_attn + 2 > 0xFFFFFFFFull) {
            // tags restart at 0: every buffer that holds tagged words is
            // cleared. Across processes a peer may already be writing this
            // rank's inbox for the next launch, so only the one-device group
            // can do that safely.
            if (t.backend == DIMG_TP_FUSED_IPC)
                fail(DIMG_ELOGIC, "tp: exchange tag space exhausted (2^32 attention stages); recreate the group");
            CK(cudaMemsetAsync(s.xg, 0, size_t(m.Hl) * m.cfg.max_ctx * 16, t.st));
            CK(cudaMemsetAsync(rp->xch, 0, (t.inbox_elems + t.slot_elems) * 8, t.st));
            s.attn_tag = 0;
        }
        PkArgs a = pk_args(s, s.stages, n_layer_stages(s), n_steps, n_prefill);
        a.tag_base = s.attn_tag;
        s.attn_tag += uint32_t(n_attn);
        a.tp_g = t.g;
        a.tp_rank = uint32_t(m.tp_rank);
        a.vocab_off = m.v0;
        for (uint32_t q = 0; q < t.g; ++q) {
            a.tp_in[q] = t.xch[q];
            a.tp_parts[q] = t.xch[q] + t.inbox_elems;
        }
        a.parts_w = a.tp_parts[a.tp_rank];
        if (t.backend == DIMG_TP_FUSED_IPC && tp_solo()) {  // timing experiment only (see tp_solo)
            a.tp_g = 1;
            a.parts_w = t.xch[t.rank] + t.inbox_elems;
        }
        CK(cudaMemsetAsync(s.bar, 0, 64 * sizeof(unsigned int), t.st));
        CK(cudaMemsetAsync(s.ssq, 0, size_t(2) * m.L * sizeof(unsigned long long), t.st));
        args.push_back(a);
    }
    const dimg_session& s0 = *t.ranks[0]->s;
    if (t.backend == DIMG_TP_FUSED_LOCAL) {
        CK(cudaMemcpyAsync(t.d_args, args.data(), args.size() * sizeof(PkArgs), cudaMemcpyHostToDevice, t.st));
        const PkArgs* d = t.d_args;
        uint32_t vg = t.vg;
        void* params[] = {&d, &vg};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(decode_persistent_group_kernel), dim3(t.g * t.vg),
                                       dim3(PK_THREADS), params, s0.smem, t.st));
    } else {
        void* params[] = {&args[0]};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(decode_persistent_kernel), dim3(t.vg),
                                       dim3(PK_THREADS), params, s0.smem, t.st));
    }
}

void tpf_begin(dimg_tp& t, const uint32_t* prompt, uint32_t p, uint32_t n, bool keep) {
    tpf_require_connected(t);
    if (keep && t.backend == DIMG_TP_FUSED_IPC)
        fail(DIMG_EINVAL, "tp: keep_logits is not available with DIMG_TP_FUSED_IPC (each process holds its vocab slice)");
    for (auto& rp : t.ranks) begin(*rp->s, prompt, p, n, keep);
    t.n_prompt = p;
    t.max_new = n;
    t.len = 0;
}

void tpf_check_err(dimg_tp& t) {
    for (auto& rp : t.ranks) check_ctl_err(*rp->s);
}

// The kept logits [max_new][V]: every rank's vocab slice (one device).
void tpf_gather_logits(dimg_tp& t, int64_t* out) {
    for (auto& rp : t.ranks)
        CK(cudaMemcpy2DAsync(out + rp->m->v0, size_t(t.V) * 8, rp->s->logits, size_t(rp->m->Vl) * 8,
                             size_t(rp->m->Vl) * 8, t.max_new, cudaMemcpyDeviceToHost, t.st));
    CK(cudaStreamSynchronize(t.st));
}

const uint32_t* tp_tokens_dev(const dimg_tp& t) { return t.fused ? t.ranks[0]->s->tokens : t.ranks[0]->tokens; }

}  // namespace

extern "C" {

dimg_status dimg_nccl_unique_id(uint8_t id[128]) {
    DIMG_API_GUARD({
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId u;
        NK(nccl_api().get_unique_id(&u));
        std::memcpy(id, &u, 128);
    })
}

dimg_status dimg_tp_create(int device, const dimg_model_desc* desc, int backend, int tp_rank, int tp_size,
                           const uint8_t nccl_id[128], uint32_t keep_logits_cap, dimg_tp** out) {
    DIMG_API_GUARD({
        if (backend < DIMG_TP_LOCAL || backend > DIMG_TP_FUSED_IPC) fail(DIMG_EINVAL, "tp: unknown backend");
        const bool fused = backend == DIMG_TP_FUSED_LOCAL || backend == DIMG_TP_FUSED_IPC;
        const bool multi = backend == DIMG_TP_NCCL || backend == DIMG_TP_FUSED_IPC;  // one rank per process
        if (tp_size < 1 || tp_size > 64) fail(DIMG_EINVAL, "tp: tp_size in 1..64");
        if (fused && tp_size > PK_TP_MAX) fail(DIMG_EINVAL, "tp: the fused backends take tp_size <= 8");
        if (multi && (tp_rank < 0 || tp_rank >= tp_size))
            fail(DIMG_EINVAL, "tp: rank outside 0..tp_size-1");
        if (backend == DIMG_TP_NCCL && !nccl_id) fail(DIMG_EINVAL, "tp: the NCCL backend needs the unique id");
        auto t = std::make_unique<dimg_tp>();
        t->backend = backend;
        t->device = device;
        t->g = uint32_t(tp_size);
        t->rank = multi ? tp_rank : 0;
        t->fused = fused;
        t->ctx = &dev_ctx(device);
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
        t->D = desc->cfg.d_model;
        t->V = desc->cfg.vocab;
        t->L = desc->cfg.n_layers;
        t->ctx_len = desc->cfg.max_ctx;
        t->vmax = (t->V + t->g - 1) / t->g;
        t->keep_cap = keep_logits_cap;
        if (backend == DIMG_TP_LOCAL) {
            t->parts = t->mem.alloc<int64_t>(size_t(t->g) * t->D);
        }
        t->pairs = t->mem.alloc<unsigned long long>(2 * size_t(t->g));
        const int lo = multi ? tp_rank : 0, hi = multi ? tp_rank + 1 : tp_size;
        if (fused) {
            t->vg = backend == DIMG_TP_FUSED_LOCAL ? uint32_t(t->ctx->sm_count) / t->g : uint32_t(t->ctx->sm_count);
            if (t->vg == 0) fail(DIMG_EINVAL, "tp: more ranks than SMs");
            t->inbox_elems = size_t(2) * t->g * t->D * 2;
            t->slot_elems = size_t(2) * t->g * t->vg * 4;
            t->xch.assign(t->g, nullptr);
            if (backend == DIMG_TP_FUSED_LOCAL) t->d_args = t->mem.alloc<PkArgs>(t->g);
        }
        for (int r = lo; r < hi; ++r) {
            auto rk = std::make_unique<TpRank>();
            // fused: the persistent kernel's blocked layout and a session per
            // shard (sharing the group's stream); else the row-major GEMV layout
            rk->m.reset(model_upload(device, desc, r, tp_size, !fused));
            if (fused) {
                rk->s = session_new(rk->m.get(), keep_logits_cap, t->vg);
                CK(cudaStreamDestroy(rk->s->stream));
                rk->s->stream = t->st;
                rk->s->own_stream = false;
                rk->xch = t->mem.alloc<unsigned long long>(t->inbox_elems + t->slot_elems);
                CK(cudaMemset(rk->xch, 0, (t->inbox_elems + t->slot_elems) * 8));
                t->xch[r] = rk->xch;
            } else {
                tp_build_rank(*t, *rk);
            }
            t->ranks.push_back(std::move(rk));
        }
        t->connected = backend != DIMG_TP_FUSED_IPC || tp_size == 1 || tp_solo();
        if (fused) t->launches_per_step = 1;  // at most: one launch runs all the steps of a call
        if (backend == DIMG_TP_NCCL) {
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, 128);
            NK(nccl_api().comm_init_rank(&t->comm, tp_size, u, tp_rank));
        }
        CK(cudaDeviceSynchronize());
        *out = t.release();
    })
}

dimg_status dimg_tp_free(dimg_tp* t) {
    DIMG_API_GUARD({
        if (t) {
            cudaSetDevice(t->device);
            cudaStreamSynchronize(t->st);
            delete t;
        }
    })
}

dimg_status dimg_tp_generate_greedy(dimg_tp* t, const uint32_t* prompt, uint32_t n_prompt, uint32_t max_new,
                                    uint32_t* tokens_out, uint8_t hash_out[32], int64_t* logits_out) {
    // run_generation (proj/src/engine.cpp:31-54) on the sharded model; every
    // rank ends with the same tokens
    DIMG_API_GUARD({
        if (t->fused) tpf_begin(*t, prompt, n_prompt, max_new, logits_out != nullptr);
        else tp_begin(*t, prompt, n_prompt, max_new, logits_out != nullptr);
        g_generations.fetch_add(1, std::memory_order_relaxed);
        if (max_new > 0) {
            if (t->fused) {
                tpf_launch(*t, n_prompt - 1 + max_new, n_prompt - 1);
                t->len = n_prompt - 1 + max_new;
            } else {
                tp_generate(*t);
            }
            CK(cudaMemcpyAsync(tokens_out, tp_tokens_dev(*t) + n_prompt, size_t(max_new) * 4,
                               cudaMemcpyDeviceToHost, t->st));
        }
        if (t->fused) tpf_check_err(*t);
        else tp_check_err(*t);
        if (logits_out && max_new > 0) {
            if (t->fused) tpf_gather_logits(*t, logits_out);
            else tp_gather_logits(*t, logits_out);
        }
        if (hash_out) {
            auto d = b3::hash(tokens_out, size_t(max_new) * 4, 1);
            std::memcpy(hash_out, d.data(), 32);
        }
    })
}

dimg_status dimg_tp_time_decode(dimg_tp* t, const uint32_t* prompt, uint32_t n_prompt, uint32_t n_steps,
                                float* ms) {
    // the prompt steps untimed, then n_steps lm_head steps between CUDA
    // events on the group's stream (tokens: dimg_tp_tokens)
    DIMG_API_GUARD({
        if (t->fused) {
            tpf_begin(*t, prompt, n_prompt, n_steps, false);
            tpf_launch(*t, n_prompt - 1, n_prompt - 1);  // the prompt positions, untimed
        } else {
            tp_begin(*t, prompt, n_prompt, n_steps, false);
            tp_run_steps(*t, false, n_prompt - 1);
            tp_ensure_graph(*t, true);  // instantiated outside the timed region
        }
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaStreamSynchronize(t->st));
        CK(cudaEventRecord(e0, t->st));
        if (t->fused) tpf_launch(*t, n_steps, 0);
        else tp_run_steps(*t, true, n_steps);
        CK(cudaEventRecord(e1, t->st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        t->len = n_prompt - 1 + n_steps;
        if (t->fused) tpf_check_err(*t);
        else tp_check_err(*t);
    })
}

dimg_status dimg_tp_tokens(dimg_tp* t, uint32_t* out, uint32_t n_generated) {
    DIMG_API_GUARD({
        CK(cudaMemcpyAsync(out, tp_tokens_dev(*t) + t->n_prompt, size_t(n_generated) * 4, cudaMemcpyDeviceToHost,
                           t->st));
        CK(cudaStreamSynchronize(t->st));
    })
}

dimg_status dimg_tp_stream(dimg_tp* t, void** stream) { DIMG_API_GUARD(*stream = t->st) }

dimg_status dimg_tp_info(dimg_tp* t, uint64_t* weight_bytes, uint64_t* launches_per_step) {
    // device bytes of this process's shards; kernels (+ collectives) per step
    DIMG_API_GUARD({
        uint64_t b = 0;
        for (auto& rp : t->ranks) b += rp->m->mem.bytes;
        if (weight_bytes) *weight_bytes = b;
        if (launches_per_step) *launches_per_step = t->launches_per_step;
    })
}

dimg_status dimg_tp_exchange_handle(dimg_tp* t, uint8_t handle[64]) {
    DIMG_API_GUARD({
        if (t->backend != DIMG_TP_FUSED_IPC) fail(DIMG_EINVAL, "tp: exchange handles belong to DIMG_TP_FUSED_IPC");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
        CK(cudaSetDevice(t->device));
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, t->ranks[0]->xch));
        std::memcpy(handle, &h, 64);
    })
}

dimg_status dimg_tp_connect(dimg_tp* t, const uint8_t* handles) {
    // maps every peer's exchange block (NVLink peer access enabled lazily)
    DIMG_API_GUARD({
        if (t->backend != DIMG_TP_FUSED_IPC) fail(DIMG_EINVAL, "tp: dimg_tp_connect belongs to DIMG_TP_FUSED_IPC");
        if (t->connected) fail(DIMG_ELOGIC, "tp: already connected");
        CK(cudaSetDevice(t->device));
        for (uint32_t q = 0; q < t->g; ++q) {
            if (int(q) == t->rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + size_t(q) * 64, 64);
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            t->ipc_open.push_back(p);
            t->xch[q] = static_cast<unsigned long long*>(p);
        }
        t->connected = true;
    })
}

}  // extern "C"
