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


if __name__ == "__main__":
    main()
