"""The CPU oracle (oracle/dim_oracle.c) pinned against the reference.

Two independent anchors:
  * the reference's own known-answer tests (proj/tests/test_*.cpp), restated;
  * golden vectors produced by running the reference engine itself
    (tests/golden/make_golden.py -> kat.json, models.json, ops.npz).
Where oracle/_ref (the reference compiled from its sources) is present, the
oracle is also compared with it live.
"""
import numpy as np
import pytest

from conftest import ops_cases, wild_arrays

ONE = 1 << 16


def _pattern(n):
    return bytes(i % 251 for i in range(n))


def test_blake3_official_vectors(oracle, kat):
    # proj/tests/test_hash.cpp:158-168
    assert oracle.blake3(b"") == "af1349b9f5f9a1a6a0404dea36dcc9499bcb25c9adc112b7cc9a93cae41f3262"
    assert oracle.blake3(_pattern(1)) == "2d3adedff11b61f14c886e35afa036736dcd87a74d27b5c1510225d0f592e213"
    assert oracle.blake3(_pattern(1024)) == "42214739f095a406f3fc83deb889744ac00df831c10daa55189b5d121c855af7"
    assert oracle.blake3(_pattern(1025)) == "d00278ae47eb27b34faecf67b4fe263f82d5412916c1ffd97c8cb7fb814b8444"
    for n, h in kat["blake3_pattern"].items():
        assert oracle.blake3(_pattern(int(n))) == h, n


def test_chacha20_rfc8439(oracle):
    # proj/tests/test_hash.cpp:207-223
    import ctypes as C
    key = (C.c_uint32 * 8)(*[(4 * i) | (4 * i + 1) << 8 | (4 * i + 2) << 16 | (4 * i + 3) << 24
                             for i in range(8)])
    nonce = (C.c_uint32 * 3)(0x09000000, 0x4a000000, 0)
    out = (C.c_uint8 * 64)()
    oracle.lib.orc_chacha20_block(key, nonce, C.c_uint32(1), out)
    assert bytes(out).hex() == (
        "10f1e7e4d13b5915500fdd1fa32071c4c7d1f4c733c068030422aa9ac3d46c4e"
        "d2826446079faa0914c2d705d98b02a2b5129cd1de164eb9cbd083e8a2503c4e")


def test_q16_known_answers(oracle):
    L = oracle.lib
    # q16_from_ratio (proj/tests/test_q16.cpp:15-29)
    for (n, d), want in {(1, 1): 65536, (0, 7): 0, (1, 127): 516, (1, 131072): 1, (-1, 131072): -1,
                         (3, 131072): 2, (1, 3): 21845, (2, 3): 43691, (-2, 3): -43691,
                         (2, -3): -43691}.items():
        assert L.orc_q16_from_ratio(n, d) == want
    # q16_mul (:31-37)
    assert L.orc_q16_mul(ONE, ONE) == ONE
    assert L.orc_q16_mul(32768, 32768) == 16384
    assert L.orc_q16_mul(-65536, 65536) == -65536
    assert L.orc_q16_mul(1 << 40, 1 << 30) == 1 << 54
    # inv_sqrt (:39-47)
    assert L.orc_inv_sqrt(65536) == 65536
    assert L.orc_inv_sqrt(262144) == 32768
    assert abs(L.orc_inv_sqrt(131072) - 46340.95) <= 0.0001 * 46341
    # exp table ends (:71-76), sigmoid (:94-111), softmax (test_kernels.cpp:197-203)
    lut = oracle.exp_lut()
    assert lut[0] == 22 and lut[256] == ONE and np.all(np.diff(lut) >= 0)
    assert L.orc_sigmoid(0) == 32768
    assert oracle.softmax(np.array([0, -20 * ONE])).tolist() == [65514, 21]
    assert oracle.softmax(np.array([42])).tolist() == [ONE]


def test_tables_match_reference_goldens(oracle, kat):
    assert oracle.exp_lut().tolist() == kat["exp_lut"]
    xs, ys = kat["inv_sqrt"]["x"], kat["inv_sqrt"]["y"]
    assert [oracle.lib.orc_inv_sqrt(x) for x in xs] == ys
    sx = kat["sigmoid"]["x"]
    assert [oracle.lib.orc_sigmoid(x) for x in sx] == kat["sigmoid"]["y"]
    assert [oracle.lib.orc_silu(x) for x in sx] == kat["sigmoid"]["silu"]
    for key, want in kat["rope"].items():
        theta, dh, ctx = key.split("_")
        c, s = oracle.rope_tables(float(theta), int(dh), int(ctx))
        assert oracle.blake3(c.tobytes()) == want["cos_digest"], key
        assert oracle.blake3(s.tobytes()) == want["sin_digest"], key


def test_prompts_match_reference(oracle, kat):
    for key, want in kat["prompts"].items():
        seed, vocab, n = (int(v) for v in key.split("_"))
        assert oracle.prompt(seed, vocab, n).tolist() == want


def test_sigmoid_symmetry(oracle):
    rng = np.random.default_rng(12)
    for x in rng.integers(-300 * ONE, 300 * ONE, 2000):
        x = int(x)
        assert oracle.lib.orc_sigmoid(x) + oracle.lib.orc_sigmoid(-x) == ONE


def test_operators_match_reference_goldens(oracle, ops_fixture):
    for w, s, x, want in ops_cases(ops_fixture, "dense"):
        assert np.array_equal(oracle.dense(w, s, x), want)
    for x, g, want in ops_cases(ops_fixture, "rmsnorm"):
        assert np.array_equal(oracle.rmsnorm(x, g), want)
    for s, want in ops_cases(ops_fixture, "softmax"):
        assert np.array_equal(oracle.softmax(s), want)
    for dims, q, k, v, want in ops_cases(ops_fixture, "attention"):
        H, dh, ctx = (int(t) for t in dims)
        assert np.array_equal(oracle.attention(H, dh, ctx, 10000.0, q, k, v), want)
    for wg, sg, wu, su, wd, sd, x, want in ops_cases(ops_fixture, "ffn"):
        assert np.array_equal(oracle.ffn(wg, sg, wu, su, wd, sd, x), want)


FAST = ["micro_s1", "micro_s9", "micro_s123456789", "small_s6", "small_s7", "small_s8", "small_s9",
        "small_s10", "small_s11", "odd_d12", "odd_dh2", "odd_k688", "accept_101", "medium",
        "wild_a", "wild_b"]


def _oracle_model(oracle, g):
    from oracle.pyoracle import Config
    cfg = Config(*g["config"], rope_theta=g["rope_theta"])
    m = oracle.gen_toy(g["seed"], cfg)
    if g["kind"] == "wild":
        s, n = wild_arrays(g["config"], g["seed"], m.scales, m.norms)
        m = oracle.model(cfg, m.weights, s, n)
    return m


@pytest.mark.parametrize("name", FAST)
def test_generation_matches_reference_goldens(oracle, golden_models, name):
    g = golden_models[name]
    m = _oracle_model(oracle, g)
    if g["weight_hash"]:
        assert m.weight_hash() == g["weight_hash"]
    toks, h, logits = oracle.generate_greedy(m, np.array(g["prompt"], np.uint32), g["max_new"],
                                             keep_logits=True)
    assert toks.tolist() == g["tokens"]
    assert h == g["output_hash"]
    assert oracle.blake3_array(logits) == g["logits_digest"]


def test_oracle_matches_live_reference():
    from oracle.pyoracle import Config, Oracle, Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    ref, orc = Reference(), Oracle()
    cfg = Config(2, 32, 4, 48, 64, 96)
    for seed in (3, 4):
        mr, mo = ref.gen_toy(seed, cfg), orc.gen_toy(seed, cfg)
        w, s, n = mr.export()
        assert np.array_equal(w, mo.weights) and np.array_equal(s, mo.scales)
        assert mr.weight_hash() == mo.weight_hash()
        a = ref.generate_greedy(mr, [5, 9, 1], 20, keep_logits=True)
        b = orc.generate_greedy(mo, np.array([5, 9, 1], np.uint32), 20, keep_logits=True)
        assert a[0].tolist() == b[0].tolist() and a[1] == b[1] and np.array_equal(a[2], b[2])


def test_generation_errors(oracle):
    from oracle.pyoracle import Config
    m = oracle.gen_toy(6, Config(2, 16, 2, 32, 32, 64))
    with pytest.raises(RuntimeError):
        oracle.generate_greedy(m, np.array([], np.uint32), 4)
    with pytest.raises(RuntimeError):
        oracle.generate_greedy(m, np.array([1, 2], np.uint32), 1000)
    with pytest.raises(RuntimeError):
        oracle.generate_greedy(m, np.array([1, 64], np.uint32), 4)


def test_sample_restatement_matches_reference_fixtures(oracle):
    """sample_from_logits (proj/src/engine.cpp:122-139) restated on the oracle's
    softmax: every per-step selection of the reference's generate_sampled
    (tests/golden/make_sample_golden.py) and the extreme rows."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "sample_ops.npz"))
    for row, n, t, d, tok in zip(z["logits"], z["lens"], z["temperature"], z["draw"], z["token"]):
        assert oracle.sample_from_logits(row[:n], int(t), int(d)) == int(tok)


def test_chacha20_restatement_matches_reference_prompts(oracle, kat):
    """The restated ChaCha20Rng (draws of generate_sampled) against the
    reference's seeded prompts: prompt[i] = ChaCha20Rng(seed).next_u32() % V,
    the key BLAKE3(seed as u64 LE) (proj/src/chacha20.cpp:57-78)."""
    from oracle.pyoracle import chacha20_u32s
    for name, ids in kat["prompts"].items():
        seed, vocab, n = (int(x) for x in name.split("_"))
        key = bytes.fromhex(oracle.blake3(seed.to_bytes(8, "little")))
        assert [w % vocab for w in chacha20_u32s(key, n)] == ids, name


def test_sample_restatement_matches_reference_edges(oracle):
    """The reference's answers at its edges (tests/golden/sample_edge.npz):
    scaled logits spanning more than 2^63 raise exp_neg_lut's domain_error
    (proj/src/q16.cpp:82) and an all-zero probability mass falls through to
    V - 1 (proj/src/engine.cpp:138); the draws are ChaCha20Rng(key)'s first u32."""
    import os
    from oracle.pyoracle import chacha20_u32s
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "sample_edge.npz"))
    for i, (row, n, t, key, d, st, tok) in enumerate(zip(z["logits"], z["lens"], z["temperature"], z["key"],
                                                          z["draw"], z["status"], z["token"])):
        assert chacha20_u32s(bytes(key), 1)[0] == int(d)
        if st == 6:
            with pytest.raises(ArithmeticError):
                oracle.sample_from_logits(row[:n], int(t), int(d))
        else:
            assert oracle.sample_from_logits(row[:n], int(t), int(d)) == int(tok), i
