"""GPU parity: the sm_100a engine against the reference's own outputs.

Goldens come from the reference engine itself (tests/golden/make_golden.py
drives oracle/_ref, the unmodified reference compiled from its sources);
live comparisons use the C oracle (oracle/dim_oracle.c) on the same seeded
inputs. Integer/byte work: the bar is bit-exact, no tolerance anywhere.
"""
import numpy as np
import pytest

from conftest import ops_cases, wild_arrays

pytestmark = pytest.mark.gpu

ONE = 1 << 16


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def _digest(P, arrs):
    return P.weight_hash(np.ascontiguousarray(np.stack(arrs), np.int64).tobytes())


# ---- operators -------------------------------------------------------------

def test_dense_matches_reference(P, ops_fixture):
    for w, s, x, want in ops_cases(ops_fixture, "dense"):
        got = P.dense_forward(w, s, x)
        assert np.array_equal(got, want), (w.shape, int(np.abs(x).max()))


def test_rmsnorm_matches_reference(P, ops_fixture):
    for x, g, want in ops_cases(ops_fixture, "rmsnorm"):
        assert np.array_equal(P.rmsnorm(x, g), want)


def test_softmax_matches_reference(P, ops_fixture):
    for s, want in ops_cases(ops_fixture, "softmax"):
        assert np.array_equal(P.softmax_q16(s), want)
    p = P.softmax_q16(np.array([0, -20 * ONE], np.int64))
    assert list(p) == [65514, 21]  # proj/tests/test_kernels.cpp:197-203


def test_attention_matches_reference(P, ops_fixture):
    for (dims, q, k, v, want) in ops_cases(ops_fixture, "attention"):
        H, dh, ctx = (int(t) for t in dims)
        got = P.attention_steps(H, dh, ctx, 10000.0, q, k, v)
        assert np.array_equal(got, want), (H, dh)


def test_ffn_matches_reference(P, ops_fixture):
    for wg, sg, wu, su, wd, sd, x, want in ops_cases(ops_fixture, "ffn"):
        assert np.array_equal(P.ffn_silu(x, wg, sg, wu, su, wd, sd), want)


def test_dense_against_oracle_wide_values(P, oracle):
    """Activations past 2^23 take the 8-limb path; values near 2^62 make the
    reference's int64 accumulator wrap -- the wrap must be reproduced."""
    rng = np.random.default_rng(3)
    for mag in (1 << 22, 1 << 23, (1 << 23) + 1, 1 << 40, 1 << 62):
        for rows, cols in ((5, 4096), (33, 11008), (7, 17), (130, 100)):
            w = rng.integers(-127, 128, (rows, cols)).astype(np.int8)
            s = rng.integers(1, 1 << 20, rows, dtype=np.int64)
            x = rng.integers(-mag, mag, cols, dtype=np.int64)
            assert np.array_equal(P.dense_forward(w, s, x), oracle.dense(w, s, x)), (mag, rows, cols)


def test_dense_edge_values(P, oracle):
    w = np.full((4, 64), 127, np.int8)
    w[1] = -127
    s = np.array([1, 65536, 1 << 40, 8], np.int64)
    for x in (np.full(64, (1 << 23) - 1, np.int64), np.full(64, -(1 << 23), np.int64),
              np.full(64, np.iinfo(np.int64).max, np.int64), np.full(64, np.iinfo(np.int64).min, np.int64),
              np.zeros(64, np.int64)):
        assert np.array_equal(P.dense_forward(w, s, x), oracle.dense(w, s, x))


# ---- whole generations -------------------------------------------------------

SMALL = ["micro_s1", "micro_s9", "micro_s123456789", "small_s6", "small_s7", "small_s8",
         "small_s9", "small_s10", "small_s11", "odd_d12", "odd_dh2", "odd_k688", "accept_101",
         "accept_102", "accept_105", "medium", "wide_heads", "long_ctx", "wild_a", "wild_b"]


def _model_for(P, g):
    cfg = P.ModelConfig(*g["config"], rope_theta=g["rope_theta"])
    m = P.gen_toy_model(g["seed"], cfg)
    if g["kind"] == "toy":
        assert m.weight_hash == g["weight_hash"]
        return m
    names = ["tok_embd"] + [f"layers.{l}.{t}" for l in range(cfg.n_layers)
                            for t in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")] + ["output"]
    tens = [m.tensor(n) for n in names]
    all_s = np.concatenate([s for _, s in tens])
    s, n = wild_arrays(g["config"], g["seed"], all_s, m.norms())
    out, o = [], 0
    for w, s0 in tens:
        out.append((w.copy(), s[o:o + len(s0)]))
        o += len(s0)
    return P.ModelFile.from_arrays(cfg, out, n)


@pytest.mark.parametrize("name", SMALL)
def test_generation_matches_reference(P, golden_models, name):
    g = golden_models[name]
    m = _model_for(P, g)
    res = P.generate_greedy(m, g["prompt"], g["max_new"], P.EngineOptions(keep_logits=True))
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]
    assert _digest(P, res.logits) == g["logits_digest"]


def test_wild_models_take_the_wide_path(P, golden_models):
    g = golden_models["wild_b"]
    m = _model_for(P, g)
    s = P.InferenceSession(m)
    s.generate_greedy(g["prompt"], g["max_new"])
    assert s.stats()["wide_limb_ctas"] > 0


def test_kv_beyond_int32_takes_the_int64_cache(P, oracle):
    """K/V values past int32 (scaled-up wk/wv) must switch the head to the
    int64 cache mid-sequence and still match the oracle bit for bit."""
    from oracle.pyoracle import Config
    cfgt = (2, 64, 2, 64, 64, 40)
    cfg = P.ModelConfig(*cfgt)
    base = oracle.gen_toy(21, Config(*cfgt))
    shapes = Config(*cfgt).tensor_shapes()
    scales = base.scales.copy()
    boost = {1 + 7 * 0 + 2: 1 << 14, 1 + 7 * 1 + 1: 1 << 16, 1 + 7 * 1 + 2: 1 << 16}  # l0.wv, l1.wk, l1.wv
    tens, so = [], 0
    w_off = 0
    for i, (r, c) in enumerate(shapes):
        if i in boost:
            scales[so:so + r] *= boost[i]
        tens.append((base.weights[w_off:w_off + r * c].reshape(r, c), scales[so:so + r]))
        so += r
        w_off += r * c
    om = oracle.model(Config(*cfgt), base.weights, scales, base.norms)
    m = P.ModelFile.from_arrays(cfg, tens, base.norms)
    prompt = [3, 9, 27, 17, 51, 25]
    toks, h, lg = oracle.generate_greedy(om, prompt, 20, keep_logits=True)
    s = P.InferenceSession(m, keep_logits_cap=20)
    res = s.generate_greedy(prompt, 20, keep_logits=True)
    assert res.token_ids == [int(t) for t in toks]
    assert res.output_hash.hex() == h
    assert np.array_equal(np.stack(res.logits), lg)
    assert s.stats()["wide_kv_ctas"] > 0
    res2 = s.generate_greedy(prompt, 20)  # a fresh sequence re-derives the flags
    assert res2.output_hash.hex() == h


def test_tinyllama_c1(P, golden_models):
    g = golden_models["tinyllama_c1"]
    m = _model_for(P, g)
    res = P.generate_greedy(m, g["prompt"], g["max_new"], P.EngineOptions(keep_logits=True))
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]
    assert _digest(P, res.logits) == g["logits_digest"]


# ---- session contract (proj/tests/test_engine.cpp) ---------------------------

def test_forward_matches_oracle_and_validates(P, oracle):
    from oracle.pyoracle import Config
    cfg = P.ModelConfig(1, 4, 2, 8, 8, 16)
    for seed in (1, 9, 123456789):
        m = P.gen_toy_model(seed, cfg)
        om = oracle.gen_toy(seed, Config(1, 4, 2, 8, 8, 16))
        s = P.InferenceSession(m)
        os_ = oracle.session(om)
        for pos, tok in enumerate([1, 5, 2, 7]):
            assert np.array_equal(s.forward(tok, pos), os_.forward(tok, pos))
    m = P.gen_toy_model(5, cfg)
    s = P.InferenceSession(m)
    with pytest.raises(P.OutOfRange):
        s.forward(99, 0)
    with pytest.raises(P.LogicError):
        s.forward(1, 5)
    for p in range(cfg.max_ctx):
        s.forward(1, p)
    with pytest.raises(P.ContextOverflow):
        s.forward(1, cfg.max_ctx)


def test_generation_preconditions(P):
    m = P.gen_toy_model(6, P.ModelConfig(2, 16, 2, 32, 32, 64))
    with pytest.raises(P.InvalidArgument):
        P.generate_greedy(m, [], 4)
    with pytest.raises(P.ContextOverflow):
        P.generate_greedy(m, [1, 2], 1000)
    with pytest.raises(P.OutOfRange):
        P.generate_greedy(m, [1, 64], 4)
    assert P.generate_greedy(m, [1, 2], 0).token_ids == []


def test_repeat_and_cached_vs_recompute(P, oracle):
    from oracle.pyoracle import Config
    cfg = P.ModelConfig(2, 16, 2, 32, 32, 64)
    m = P.gen_toy_model(7, cfg)
    hashes = {P.generate_greedy(m, [3, 1, 4], 12).output_hash for _ in range(100)}
    assert len(hashes) == 1
    # KV-cached decode equals full recomputation (test_engine.cpp:113-126)
    m9 = P.gen_toy_model(9, cfg)
    fast = P.generate_greedy(m9, [2, 4, 8], 6).token_ids
    om = oracle.gen_toy(9, Config(2, 16, 2, 32, 32, 64))
    for i in range(6):
        full = np.array([2, 4, 8] + fast[:i], np.uint32)
        toks, _, _ = oracle.generate_greedy(om, full, 1)
        assert int(toks[0]) == fast[i]


def test_imported_rope_tables(P):
    cfg = P.ModelConfig(2, 16, 2, 32, 32, 64)
    m = P.gen_toy_model(11, cfg)
    base = P.generate_greedy(m, [6, 2], 8)
    tabs = P.build_rope_tables(cfg.rope_theta, cfg.d_head, cfg.max_ctx)
    imp = P.generate_greedy(m, [6, 2], 8, imported_tables=tabs)
    assert imp.output_hash == base.output_hash


def test_device_resident_stepping_matches_generate(P, golden_models):
    g = golden_models["medium"]
    m = _model_for(P, g)
    s = P.InferenceSession(m)
    s.begin(g["prompt"], g["max_new"])
    s.prefill()
    s.decode(5)
    s.decode(g["max_new"] - 5)
    s.sync()
    assert s.tokens(g["max_new"]) == g["tokens"]
    d, p = s.launches()
    assert d == 1 and p == 1  # one persistent launch per call


# ---- tensor-core prefill GEMM (tcgen05 kind::i8 over byte limbs) ---------------

@pytest.mark.parametrize("N,K,T", [(128, 128, 128), (256, 4096, 130), (100, 300, 7), (4096, 4096, 256),
                                   (384, 11008, 64), (33, 17, 1)])
def test_dense_tokens_matches_oracle(P, oracle, N, K, T):
    rng = np.random.default_rng(N * 7 + K + T)
    w = rng.integers(-127, 128, (N, K), dtype=np.int8)
    s = rng.integers(1, 1 << 12, N, dtype=np.int64)
    # the whole signed-digit range (put_sdigits: -0x808080 .. 0x7F7F7F) with its ends
    x = rng.integers(-0x808080, 0x7F7F80, (T, K), dtype=np.int64)
    x[0, :7] = [-0x808080, 0x7F7F7F, 0, -1, 255, -128, 0x7F7F80 - 0x10000]
    got = P.dense_tokens(w, s, x)
    for t in range(T):
        assert np.array_equal(got[t], oracle.dense(w, s, x[t])), t


def test_dense_tokens_wide_rows_fall_back_exactly(P, oracle):
    rng = np.random.default_rng(5)
    w = rng.integers(-127, 128, (64, 96), dtype=np.int8)
    s = rng.integers(1, 1 << 12, 64, dtype=np.int64)
    x = rng.integers(-(1 << 20), 1 << 20, (5, 96), dtype=np.int64)
    x[3, 7] = 1 << 40
    got = P.dense_tokens(w, s, x)
    for t in range(5):
        assert np.array_equal(got[t], oracle.dense(w, s, x[t]))
    # one past either end of the three-digit range
    for v in (0x7F7F80, -0x808081):
        x2 = x.copy()
        x2[3, 7] = v
        got = P.dense_tokens(w, s, x2)
        for t in range(5):
            assert np.array_equal(got[t], oracle.dense(w, s, x2[t]))


# ---- tensor-core prefill (whole prompt per layer) ------------------------------

@pytest.mark.parametrize("cfg6,plen,seed,kd4,pv", [((2, 64, 2, 64, 64, 256), 200, 3, 0, 1),
                                                    ((2, 256, 2, 512, 300, 400), 300, 4, 0, 1),
                                                    ((2, 256, 2, 512, 300, 400), 300, 4, 1, 1),
                                                    ((2, 256, 2, 512, 300, 400), 300, 4, 0, 0),
                                                    ((1, 512, 4, 256, 300, 1024), 700, 6, 0, 1),
                                                    ((1, 512, 4, 256, 300, 1024), 700, 6, 0, 0),
                                                    ((2, 128, 1, 256, 64, 256), 130, 8, 0, 1),
                                                    ((3, 96, 3, 160, 77, 200), 40, 5, 0, 1)])
def test_tensor_core_prefill_matches_oracle(P, oracle, monkeypatch, cfg6, plen, seed, kd4, pv):
    """kd4=1 forces the tensor-core scores' 4th key digit plane; pv=0 keeps
    all of PV on the CUDA cores (dh = 128 shapes: pv=1 puts its linear half on
    the tensor cores, pf_pv.cuh)."""
    from oracle.pyoracle import Config
    monkeypatch.setenv("DIMG_PREFILL", "1")
    monkeypatch.setenv("DIMG_PF_KD4", str(kd4))
    monkeypatch.setenv("DIMG_PF_PV", str(pv))
    m = P.gen_toy_model(seed, P.ModelConfig(*cfg6))
    om = oracle.gen_toy(seed, Config(*cfg6))
    prompt = P.prompt_from_seed(seed + 100, cfg6[4], plen)
    toks, h, lg = oracle.generate_greedy(om, prompt, 6, keep_logits=True)
    s = P.InferenceSession(m, keep_logits_cap=6)
    res = s.generate_greedy(prompt, 6, keep_logits=True)
    assert s.stats()["tc_prefills"] == 1 and s.stats()["tc_fallbacks"] == 0
    assert res.token_ids == [int(t) for t in toks]
    assert res.output_hash.hex() == h
    assert np.array_equal(np.stack(res.logits), lg)


def test_tensor_core_prefill_falls_back_exactly(P, oracle, golden_models, monkeypatch):
    """A model whose activations exceed 3 byte limbs: the tensor-core prefill
    detects it and the exact decode path redoes the prompt."""
    monkeypatch.setenv("DIMG_PREFILL", "1")
    g = golden_models["wild_b"]
    m = _model_for(P, g)
    s = P.InferenceSession(m)
    prompt = (g["prompt"] * 40)[:60]
    res = s.generate_greedy(prompt, 5)
    assert s.stats()["tc_fallbacks"] == 1
    monkeypatch.setenv("DIMG_PREFILL", "2")
    ref = P.InferenceSession(m).generate_greedy(prompt, 5)
    assert res.token_ids == ref.token_ids and res.output_hash == ref.output_hash


# ---- batched generation (C5) ----------------------------------------------------

@pytest.mark.parametrize("cfg6,n_seqs,plen,new", [((2, 64, 2, 64, 64, 256), 5, 12, 9),
                                                  ((2, 256, 2, 512, 300, 200), 8, 30, 6),
                                                  ((3, 96, 3, 160, 77, 100), 3, 1, 7),
                                                  ((2, 64, 2, 64, 64, 256), 1, 8, 5),      # one sequence
                                                  ((2, 128, 2, 256, 100, 128), 20, 5, 6),  # 64-token tiles, cluster norm
                                                  ((2, 64, 2, 64, 64, 128), 70, 3, 4)])    # two token tiles
def test_batch_generation_matches_single(P, oracle, cfg6, n_seqs, plen, new):
    from oracle.pyoracle import Config
    m = P.gen_toy_model(11, P.ModelConfig(*cfg6))
    om = oracle.gen_toy(11, Config(*cfg6))
    prompts = [P.prompt_from_seed(500 + i, cfg6[4], plen + (i % 3)) for i in range(n_seqs)]
    res, path = P.generate_greedy_batch(m, prompts, new)
    assert path == "tensor_cores"
    for p, r in zip(prompts, res):
        toks, h, _ = oracle.generate_greedy(om, p, new)
        assert r.token_ids == [int(t) for t in toks]
        assert r.output_hash.hex() == h


def test_batch_generation_wild_falls_back(P, golden_models):
    g = golden_models["wild_b"]
    m = _model_for(P, g)
    prompts = [g["prompt"], g["prompt"][:1] * 3]
    res, path = P.generate_greedy_batch(m, prompts, 4)
    single = [P.generate_greedy(m, p, 4) for p in prompts]
    assert [r.token_ids for r in res] == [s.token_ids for s in single]
    assert [r.output_hash for r in res] == [s.output_hash for s in single]


# ---- repeat determinism of the tensor-core paths (proj/tests/test_engine.cpp:87-111) ----

def test_dense_tokens_ragged_repeat_stress(P, oracle):
    """Ragged shapes through the tensor-core GEMM export, 200 calls per shape
    group with fresh device buffers each call, against the oracle: the upload
    of the weights is stream-ordered before the K-block-major relayout and the
    GEMM (a pageable legacy-stream copy was not)."""
    import itertools
    shapes = list(itertools.product((33, 100, 130), (17, 300, 4095), (1, 7, 65)))
    rng = np.random.default_rng(2024)
    cases = []
    for N, K, T in shapes:
        w = rng.integers(-127, 128, (N, K), dtype=np.int8)
        s = rng.integers(1, 1 << 12, N, dtype=np.int64)
        x = rng.integers(-0x808080, 0x7F7F80, (T, K), dtype=np.int64)
        want = np.stack([oracle.dense(w, s, x[t]) for t in range(T)])
        cases.append((w, s, x, want))
    for rep in range(200 // 8):
        for i, (w, s, x, want) in enumerate(cases):
            if (rep + i) % 3 and rep > 0:
                continue  # every shape at least ~8x, 200+ calls in all
            got = P.dense_tokens(w, s, x)
            assert np.array_equal(got, want), (rep, w.shape, x.shape)


def test_tensor_core_prefill_and_batch_repeat(P, oracle, monkeypatch):
    """The same small tensor-core prefill and batch generations 20 times:
    identical tokens every time (split-K scratch and PDL chains included)."""
    from oracle.pyoracle import Config
    cfg6 = (2, 128, 2, 256, 100, 160)
    m = P.gen_toy_model(21, P.ModelConfig(*cfg6))
    om = oracle.gen_toy(21, Config(*cfg6))
    prompts = [P.prompt_from_seed(900 + i, cfg6[4], 5 + (i % 4)) for i in range(9)]
    want = [oracle.generate_greedy(om, p, 6)[0] for p in prompts]
    want = [[int(t) for t in w] for w in want]
    monkeypatch.setenv("DIMG_PREFILL", "1")
    s = P.InferenceSession(m)
    for rep in range(20):
        for p, wt in zip(prompts[:3], want[:3]):
            assert s.generate_greedy(p, 6).token_ids == wt, rep
        res, path = P.generate_greedy_batch(m, prompts, 6)
        assert path == "tensor_cores"
        assert [r.token_ids for r in res] == want, rep


def test_partition_invariance(P, golden_models, monkeypatch):
    """The reference's thread/chunk invariance (proj/tests/test_engine.cpp:87-111,
    test_kernels.cpp:79-97) on the GPU's own partitions: the attention split
    into 1, 2 or 4 CTAs per head, the decode kernel vs the tensor-core prefill
    vs the tensor-parallel shards -- identical tokens and logits every time,
    100 repeats of the default path."""
    g = golden_models["medium"]
    m = _model_for(P, g)
    want = g["tokens"]
    for parts in ("1", "2", "4"):
        monkeypatch.setenv("DIMG_ATTN_PARTS", parts)
        for pf in ("1", "2"):
            monkeypatch.setenv("DIMG_PREFILL", pf)
            res = P.InferenceSession(m, keep_logits_cap=g["max_new"]).generate_greedy(g["prompt"], g["max_new"],
                                                                                     keep_logits=True)
            assert res.token_ids == want, (parts, pf)
            assert _digest(P, res.logits) == g["logits_digest"], (parts, pf)
    monkeypatch.delenv("DIMG_ATTN_PARTS")
    monkeypatch.delenv("DIMG_PREFILL")
    s = P.InferenceSession(m)
    hashes = {s.generate_greedy(g["prompt"], g["max_new"]).output_hash.hex() for _ in range(100)}
    assert hashes == {g["output_hash"]}
