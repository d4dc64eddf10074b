"""Writes tests/golden/sample.json and sample_ops.npz from the REFERENCE's
generate_sampled (proj/src/engine.cpp:122-163, compiled into
oracle/_ref/libdimref.so, shim ref_generate_sampled):

  sample.json      end-to-end cases: model seed/config, prompt, Q16
                   temperature, tokens, output hash, RNG key
  sample_ops.npz   per-step selection fixtures: logits row, temperature, the
                   step's ChaCha20 draw, the reference's token; plus extreme
                   rows answered by the oracle restatement, which this script
                   first checks against every reference step

    python tests/golden/make_sample_golden.py      (needs /root/reference)
    python tests/golden/make_sample_golden.py edge (sample_edge.npz only)

  sample_edge.npz  rows at the reference's edges, answered by the reference's
                   own sample_from_logits (shim ref_sample_from_logits):
                   scaled logits spanning more than 2^63 (exp_neg_lut throws
                   std::domain_error: status 6) and vocabularies above 65536
                   whose probabilities all truncate to 0 (the walk falls
                   through to V - 1)
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Config, Oracle, Reference, chacha20_u32s  # noqa: E402

ONE = 1 << 16
CASES = [((2, 16, 2, 32, 32, 64), 1001, [4, 8, 15], ONE, 12),
         ((2, 16, 2, 32, 32, 64), 1001, [4, 8, 15], ONE // 4, 12),
         ((2, 16, 2, 32, 32, 64), 1001, [4, 8, 15], 3 * ONE, 12),
         ((2, 64, 2, 160, 100, 64), 3, None, ONE // 2, 20),
         ((2, 64, 4, 128, 300, 96), 5, None, 2 * ONE, 16),
         ((2, 16, 2, 32, 32, 64), 1001, [4, 8, 15], 1, 10),         # T = 1 raw: logit << 16 wraps
         ((2, 16, 2, 32, 32, 64), 1001, [4, 8, 15], 1 << 40, 10),   # T = 2^24 ONE: near-flat
         ((2, 64, 2, 160, 1000, 64), 7, None, ONE, 12)]             # larger vocabulary


def main():
    ref, orc = Reference(), Oracle()
    lib = ref.lib
    u32p, u8p, i64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), C.POINTER(C.c_int64)
    lib.ref_generate_sampled.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_uint32, C.c_int64, u32p, u8p, i64p]
    cases, rows, temps, draws, toks = [], [], [], [], []
    for cfg6, seed, prompt, T, n in CASES:
        cfg = Config(*cfg6)
        m = ref.gen_toy(seed, cfg)
        if prompt is None:
            prompt = [int(t) for t in ref.prompt(seed + 100, cfg.vocab, 7)]
        p = np.array(prompt, np.uint32)
        out = np.zeros(n, np.uint32)
        h = (C.c_uint8 * 32)()
        logits = np.zeros((n, cfg.vocab), np.int64)
        assert lib.ref_generate_sampled(m.h, p.ctypes.data_as(u32p), len(p), n, T, out.ctypes.data_as(u32p), h,
                                        logits.ctypes.data_as(i64p)) == 0
        nb = lib.ref_model_bytes(m.h, None)
        mb = (C.c_uint8 * nb)()
        lib.ref_model_bytes(m.h, mb)
        key = bytes.fromhex(ref.blake3(bytes(mb) + p.astype("<u4").tobytes()))
        dr = chacha20_u32s(key, n)
        for i in range(n):  # the restatement reproduces every reference selection
            assert orc.sample_from_logits(logits[i], T, dr[i]) == int(out[i]), (cfg6, T, i)
            rows.append(logits[i]); temps.append(T); draws.append(dr[i]); toks.append(int(out[i]))
        cases.append({"config": list(cfg6), "seed": seed, "prompt": prompt, "temperature": T, "max_new": n,
                      "tokens": [int(t) for t in out], "output_hash": bytes(h).hex(), "key": key.hex()})
    # extreme rows: wrap of the int64 cast, ties, flat and one-hot masses, V = 1
    rng = np.random.default_rng(11)
    V = max(len(r) for r in rows)
    extra = [np.full(V, 5 * ONE, np.int64), np.array([(1 << 62) - 1, -(1 << 62)] * (V // 2), np.int64),
             rng.integers(-(1 << 40), 1 << 40, V, dtype=np.int64), rng.integers(-ONE, ONE, V, dtype=np.int64),
             np.array([7 * ONE], np.int64)]
    for r in extra:
        for T in (1, ONE, 1 << 40):
            for d in (0, 1, 0x7FFFFFFF, 0xFFFFFFFF, int(rng.integers(0, 1 << 32))):
                rows.append(r); temps.append(T); draws.append(d); toks.append(orc.sample_from_logits(r, T, d))
    width = max(len(r) for r in rows)
    L = np.zeros((len(rows), width), np.int64)
    lens = np.array([len(r) for r in rows], np.uint32)
    for i, r in enumerate(rows):
        L[i, :len(r)] = r
    np.savez_compressed(os.path.join(HERE, "sample_ops.npz"), logits=L, lens=lens,
                        temperature=np.array(temps, np.int64), draw=np.array(draws, np.uint32),
                        token=np.array(toks, np.uint32))
    with open(os.path.join(HERE, "sample.json"), "w") as f:
        json.dump({"cases": cases}, f, indent=1)
    print(len(cases), "cases,", len(rows), "selection fixtures")


def edge():
    ref, orc = Reference(), Oracle()
    rng = np.random.default_rng(23)
    rows, temps = [], []
    # spans beyond 2^63 after the temperature division: domain_error
    rows.append(np.array([1 << 62, -(1 << 62)], np.int64)); temps.append(ONE)
    rows.append(np.array([5, 1 << 46, 7, -(1 << 46)], np.int64)); temps.append(1)
    rows.append(np.concatenate([rng.integers(-ONE, ONE, 300), [(1 << 62) + 5, -(1 << 62)]]).astype(np.int64))
    temps.append(ONE)
    # span exactly 2^63 - 1: allowed
    rows.append(np.array([(1 << 62) - 1, -(1 << 62)], np.int64)); temps.append(ONE)
    # vocab > 65536, near-flat: every p truncates to 0 -> V - 1
    rows.append(rng.integers(-ONE, ONE, 70000).astype(np.int64)); temps.append(1 << 40)
    rows.append(np.full(131072, 3 * ONE, np.int64)); temps.append(ONE)
    # vocab > 65536 with a peak: ordinary walk
    r = rng.integers(-4 * ONE, 4 * ONE, 70000).astype(np.int64)
    r[12345] = 40 * ONE
    rows.append(r); temps.append(ONE)
    # exactly 65536 flat: p = 1 each
    rows.append(np.zeros(65536, np.int64)); temps.append(ONE)
    keys, status, toks = [], [], []
    for i, (row, T) in enumerate(zip(rows, temps)):
        key = bytes((7 * i + j) & 0xFF for j in range(32))
        rc, tok = ref.sample_from_logits(row, T, key)
        assert rc in (0, 6), rc
        d = chacha20_u32s(key, 1)[0]
        try:  # the restatement agrees, error included
            got = orc.sample_from_logits(row, T, d)
        except ArithmeticError:
            got = None
        assert (rc == 6 and got is None) or (rc == 0 and got == tok), (i, rc, tok, got)
        keys.append(np.frombuffer(key, np.uint8)); status.append(rc); toks.append(tok if rc == 0 else 0xFFFFFFFF)
        print(i, len(row), T, rc, tok)
    width = max(len(r) for r in rows)
    L = np.zeros((len(rows), width), np.int64)
    for i, r in enumerate(rows):
        L[i, :len(r)] = r
    np.savez_compressed(os.path.join(HERE, "sample_edge.npz"), logits=L,
                        lens=np.array([len(r) for r in rows], np.uint32), temperature=np.array(temps, np.int64),
                        key=np.array(keys), draw=np.array([chacha20_u32s(bytes(k), 1)[0] for k in keys], np.uint32),
                        status=np.array(status, np.int32), token=np.array(toks, np.uint32))


if __name__ == "__main__":
    edge() if sys.argv[1:] == ["edge"] else main()
