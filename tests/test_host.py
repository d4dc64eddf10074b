"""Host half of the product (libdimg.so without a GPU): C-ABI exports, the
DIM1 container, BLAKE3, ChaCha20 model generation, prompt parsing, tables --
each checked against the oracle and the reference's known answers."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ONE = 1 << 16
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def test_library_exports_every_header_symbol(P):
    """Every function declared in include/dimg.h is exported by libdimg.so and
    bound by the Python layer."""
    hdr = open(os.path.join(ROOT, "include", "dimg.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(dimg_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) > 40
    lib = C.CDLL(P.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    from paper_2603_24904_b200._lib import EXPORTED
    assert declared <= set(EXPORTED) | {"dimg_version"}, declared - set(EXPORTED)


def test_blake3_matches_oracle(P, oracle):
    def pat(n):
        return bytes(i % 251 for i in range(n))
    # single-thread chunk path and the parallel 1 MiB-subtree path
    for n in (0, 1, 63, 64, 65, 1023, 1024, 1025, 2048, 2049, 3072, 8192, 100000, 1 << 20,
              (1 << 20) + 1, 3 * (1 << 20) + 7, 5 * (1 << 20)):
        assert P.weight_hash(pat(n)) == oracle.blake3(pat(n)), n
    ids = [5, 1 << 31, 0, 65535]
    assert P.hash_token_ids(ids).hex() == oracle.blake3(np.array(ids, np.uint32).tobytes())
    assert P.hash_token_ids([]).hex() == "af1349b9f5f9a1a6a0404dea36dcc9499bcb25c9adc112b7cc9a93cae41f3262"


@pytest.mark.parametrize("c6,seed", [((1, 4, 2, 8, 8, 16), 1), ((2, 16, 2, 32, 32, 64), 7),
                                      ((3, 12, 3, 20, 37, 40), 21), ((2, 256, 4, 688, 1000, 256), 23)])
def test_toy_model_bytes_match_oracle(P, oracle, c6, seed):
    from oracle.pyoracle import Config
    m = P.gen_toy_model(seed, P.ModelConfig(*c6))
    mo = oracle.gen_toy(seed, Config(*c6))
    assert bytes(m.bytes) == mo.serialize()
    assert m.weight_hash == mo.weight_hash()


def test_weight_hash_goldens(P, golden_models):
    for name in ("small_s7", "odd_k688", "accept_101", "medium"):
        g = golden_models[name]
        m = P.gen_toy_model(g["seed"], P.ModelConfig(*g["config"]))
        assert m.weight_hash == g["weight_hash"], name


def test_toy_scales_rule(P):
    # proj/tests/test_model.cpp:200-208: 1 / (127 * floor(sqrt(d_in)))
    m = P.gen_toy_model(46, P.ModelConfig(1, 64, 4, 8, 8, 16))
    from paper_2603_24904_b200.model import ONE as one
    w, s = m.tensor("layers.0.wq")
    assert s[0] == round(65536 / (127 * 8))
    w, s = m.tensor("layers.0.w_down")
    assert s[0] == round(65536 / (127 * 2))
    assert m.norms()[0] == one
    assert w.min() >= -127 and w.max() <= 127


def test_dim1_roundtrip_and_parse_errors(P):
    m = P.gen_toy_model(45, P.ModelConfig(1, 4, 2, 8, 8, 16))
    b = bytes(m.bytes)
    m2 = P.deserialize(b)
    assert bytes(m2.bytes) == b and m2.weight_hash == m.weight_hash
    # proj/tests/test_model.cpp:131-178
    with pytest.raises(P.ParseError) as e:
        P.deserialize(b"XIM1" + b[4:])
    assert e.value.kind == "bad_magic"
    with pytest.raises(P.ParseError) as e:
        P.deserialize(b[:4] + b"\x02\x00\x00\x00" + b[8:])
    assert e.value.kind == "bad_version"
    for cut in (3, 10, 60, len(b) - 1):
        with pytest.raises(P.ParseError) as e:
            P.deserialize(b[:cut])
        assert e.value.kind == "truncated", cut
    with pytest.raises(P.ParseError) as e:
        P.deserialize(b + b"\x00")
    assert e.value.kind == "invariant"
    # a -128 weight (the last byte is the output tensor's last weight)
    w = np.frombuffer(b, np.uint8).copy()
    w[-1] = 0x80
    with pytest.raises(P.ParseError) as e:
        P.deserialize(w.tobytes())
    assert e.value.kind == "invariant"


def test_save_load(P, tmp_path):
    m = P.gen_toy_model(3, P.ModelConfig(2, 16, 2, 32, 32, 64))
    p = str(tmp_path / "m.dim")
    m.save(p)
    assert P.load_model(p).weight_hash == m.weight_hash
    with pytest.raises(P.errors.IOFailure):
        P.load_model(str(tmp_path / "missing.dim"))


def test_config_validation(P):
    # proj/src/model.cpp:95-109
    for bad in [(0, 4, 2, 8, 8, 16), (1, 4, 0, 8, 8, 16), (1, 6, 4, 8, 8, 16), (1, 8200, 2, 8, 8, 16),
                (1, 6, 2, 8, 8, 16), (1, 4, 2, 0, 8, 16), (1, 4, 2, 8, 1, 16), (1, 4, 2, 8, 8, 0)]:
        with pytest.raises(P.InvalidArgument):
            P.ModelConfig(*bad).validate()
    with pytest.raises(P.InvalidArgument):
        P.ModelConfig(1, 4, 2, 8, 8, 16, rope_theta=-1.0).validate()
    P.ModelConfig(1, 4, 2, 8, 8, 16).validate()


def test_tables_match_reference_goldens(P, kat):
    lut = np.empty(257, np.int64)
    from paper_2603_24904_b200._lib import i64p, lib, ptr
    lib.dimg_exp_lut(ptr(lut, i64p))
    assert lut.tolist() == kat["exp_lut"]
    for key, want in kat["rope"].items():
        theta, dh, ctx = key.split("_")
        c, s = P.build_rope_tables(float(theta), int(dh), int(ctx))
        assert P.weight_hash(c.tobytes()) == want["cos_digest"], key
        assert P.weight_hash(s.tobytes()) == want["sin_digest"], key


def test_prompts_and_parse_prompt(P, kat):
    for key, want in kat["prompts"].items():
        seed, vocab, n = (int(v) for v in key.split("_"))
        assert P.prompt_from_seed(seed, vocab, n) == want
    # proj/tools/dim_cli.cpp:56-70
    assert P.parse_prompt("1,2,,3") == [1, 2, 3]
    assert P.parse_prompt("", "hi") == [104, 105]
    assert P.parse_prompt("7") == [7]
    with pytest.raises(P.InvalidArgument):
        P.parse_prompt("")
    with pytest.raises(P.InvalidArgument):
        P.parse_prompt("x")
    with pytest.raises(P.OutOfRange):
        P.parse_prompt("99999999999999999999999")
    assert P.parse_prompt("4294967297") == [1]  # uint32_t(std::stoul(...)) truncation


def test_select_greedy_ties(P):
    # proj/tests/test_engine.cpp:67-76
    assert P.select_greedy([3, 7, 7, 1]) == 1
    for off in (-100000, -1, 1, 65536, 999999):
        assert P.select_greedy([3 + off, 7 + off, 7 + off, 1 + off]) == 1
    with pytest.raises(P.InvalidArgument):
        P.select_greedy([])


def test_device_entry_points_fail_loudly_without_gpu(P):
    """No CPU fallback: without a CUDA device the engine raises instead of
    computing anything on the host."""
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        if cu.cuInit(0) == 0 and cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0:
            pytest.skip("a GPU is present")
    except OSError:
        pass
    m = P.gen_toy_model(1, P.ModelConfig(1, 4, 2, 8, 8, 16))
    with pytest.raises(P.errors.CudaError):
        P.generate_greedy(m, [1, 2], 3)
    with pytest.raises(P.errors.CudaError):
        P.dense_forward(np.ones((2, 4), np.int8), np.ones(2, np.int64), np.ones(4, np.int64))


# ---- RTAB codec (proj/src/rope.cpp:41-93) against the reference's own bytes ----

def _rtab_golden():
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rtab.json")))


def test_rtab_serialize_is_byte_exact_with_reference():
    import paper_2603_24904_b200 as P
    g = _rtab_golden()
    for t in g["tables"]:
        tab = P.RopeTables.build(t["theta"], t["d_head"], t["max_ctx"])
        assert P.serialize_rope_tables(tab).hex() == t["hex"]
        back = P.deserialize_rope_tables(bytes.fromhex(t["hex"]))  # import the reference's artifact
        assert back == tab
    b = g["big"]
    big = P.serialize_rope_tables(P.RopeTables.build(b["theta"], b["d_head"], b["max_ctx"]))
    assert len(big) == b["size"] and P.weight_hash(big) == b["blake3"]


def test_rtab_parse_errors_match_reference():
    import paper_2603_24904_b200 as P
    for c in _rtab_golden()["parse"]:
        data = bytes.fromhex(c["hex"])
        if c["outcome"] == 0:
            P.deserialize_rope_tables(data)
            continue
        with pytest.raises(P.ParseError) as e:
            P.deserialize_rope_tables(data)
        assert e.value.kind == P.ParseError.KINDS[c["outcome"] - 100], c


def test_rtab_save_load_roundtrip(tmp_path):
    import paper_2603_24904_b200 as P
    t = P.RopeTables.build(10000.0, 16, 33)
    p = str(tmp_path / "t.rtab")
    P.save_rope_tables(t, p)
    assert P.load_rope_tables(p) == t
    with pytest.raises(P.errors.IOFailure):
        P.load_rope_tables(str(tmp_path / "missing.rtab"))
    with pytest.raises(P.errors.IOFailure):
        P.save_rope_tables(t, str(tmp_path / "no" / "dir.rtab"))


def test_inv_sqrt_fast_path_matches_oracle(P, oracle):
    """The kernels' inv_sqrt_q16 (64-bit Newton steps where every product
    provably fits, the int128 steps otherwise; kernels/q16.cuh) against the
    oracle's int128 restatement of q16.cpp:56-68: every octave's ends, a
    spread inside each octave, and all x < 2^14."""
    from paper_2603_24904_b200._lib import lib
    rng = np.random.default_rng(5)
    xs = set(range(1, 1 << 14))
    for b in range(63):
        lo, hi = 1 << b, (1 << (b + 1)) - 1
        xs.update({lo, lo + 1, hi, hi - 1, (lo + hi) // 2})
        xs.update(int(v) for v in rng.integers(lo, hi, size=64, endpoint=True, dtype=np.uint64))
    out = C.c_int64()
    for x in sorted(v for v in xs if v > 0):
        assert lib.dimg_inv_sqrt_q16(x, C.byref(out)) == 0
        assert out.value == oracle.lib.orc_inv_sqrt(x), x


def test_pv_remainder_mod_2_16_identity():
    """The tensor-core prefill PV (pf_attn_kernel<_, true> + pf_pv_kernel)
    recovers sum_p floor(P_p v_p / 2^16) (proj/src/kernels.cpp:153-159 after
    the mul16 of each product) from T = sum_p P_p vh_p (tensor cores) and
    U = sum_p ((P_p v_p mod 2^32) >> 16) (CUDA cores, no vl mask) as
    T + ((U - T) mod 2^16): exact because F = sum_p floor(P_p vl_p / 2^16)
    lies in [0, sum_p P_p) and sum_p P_p <= 2^16. Checked here on random and
    extreme rows, including |v| up to 2^23 and one-hot probabilities."""
    rng = np.random.default_rng(5)
    cases = []
    for n in (1, 2, 7, 64, 300, 2048):
        w = rng.integers(1, 1 << 16, n, dtype=np.int64)
        P = (w << 16) // w.sum()  # floor(w 2^16 / total): sums to <= 2^16
        for lim in (1 << 8, 1 << 16, 1 << 23):
            cases.append((P, rng.integers(-lim, lim, n, dtype=np.int64)))
    onehot = np.zeros(5, np.int64)
    onehot[2] = (1 << 16) - 1
    cases.append((onehot, np.array([-(1 << 23)] * 5, np.int64)))
    cases.append((np.full(4, 1 << 14, np.int64), np.array([(1 << 23) - 1, -(1 << 23), 65535, -1], np.int64)))
    for P, v in cases:
        assert P.sum() <= 1 << 16
        want = int(((P * v) >> 16).sum())  # floor per product
        vh = v >> 16
        T = int((P * vh).sum())
        U = int((((P * v) & 0xFFFFFFFF) >> 16).sum())
        assert T + ((U - T) & 0xFFFF) == want
