"""Regenerates tests/golden/* by running the REFERENCE engine itself.

The reference (/root/reference/proj/src) is compiled from its own sources by
oracle/Makefile into oracle/_ref/libdimref.so; this script drives it through
oracle/pyoracle.Reference and writes:

  kat.json      tables and primitive known answers (exp LUT, inv-sqrt,
                sigmoid/silu sweeps, RoPE rows, BLAKE3 vectors, prompts)
  models.json   per-config weight_hash / tokens / output_hash / logits digest
  ops.npz       operator-level cases (dense, rmsnorm, softmax, attention, ffn)

Run (in the container that has /root/reference):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box only reads them.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Config, Reference  # noqa: E402

ONE = 65536


def digest_logits(ref: Reference, logits) -> str:
    return ref.blake3(np.ascontiguousarray(logits, np.int64).tobytes())


# (name, cfg, seed, prompt spec, max_new, kind)
#   prompt spec: list of ids, or ("chacha", prompt_seed, n)
#   kind: "toy" = gen_toy_model(seed); "wild" = toy weights with large random
#         scales/gains (drives activations past 2^23 and the dense sums
#         towards the 64-bit wrap, exercising exact wide-limb paths)
MODEL_CASES = [
    ("micro_s1", (1, 4, 2, 8, 8, 16), 1, [1, 5, 2, 7], 6, "toy"),
    ("micro_s9", (1, 4, 2, 8, 8, 16), 9, [1, 5, 2, 7], 6, "toy"),
    ("micro_s123456789", (1, 4, 2, 8, 8, 16), 123456789, [1, 5, 2, 7], 6, "toy"),
    ("small_s6", (2, 16, 2, 32, 32, 64), 6, [1, 2], 12, "toy"),
    ("small_s7", (2, 16, 2, 32, 32, 64), 7, [3, 1, 4], 12, "toy"),
    ("small_s8", (2, 16, 2, 32, 32, 64), 8, [5, 9], 16, "toy"),
    ("small_s9", (2, 16, 2, 32, 32, 64), 9, [2, 4, 8], 6, "toy"),
    ("small_s10", (2, 16, 2, 32, 32, 64), 10, [1], 5, "toy"),
    ("small_s11", (2, 16, 2, 32, 32, 64), 11, [6, 2], 8, "toy"),
    ("odd_d12", (3, 12, 3, 20, 37, 40), 21, [36, 0, 5, 17], 20, "toy"),
    ("odd_dh2", (2, 6, 3, 10, 11, 24), 22, [3, 10], 12, "toy"),
    ("odd_k688", (2, 256, 4, 688, 1000, 256), 23, ("chacha", 24, 9), 24, "toy"),
    ("accept_101", (16, 64, 4, 128, 256, 512), 101, ("chacha", 3000, 4), 64, "toy"),
    ("accept_102", (16, 64, 4, 128, 256, 512), 102, ("chacha", 3010, 4), 64, "toy"),
    ("accept_105", (16, 64, 4, 128, 256, 512), 105, ("chacha", 3040, 4), 64, "toy"),
    ("medium", (4, 512, 8, 1376, 4096, 1024), 31, ("chacha", 32, 16), 32, "toy"),
    ("wide_heads", (2, 1024, 4, 2816, 2048, 300), 33, ("chacha", 34, 40), 40, "toy"),
    ("long_ctx", (2, 128, 2, 344, 512, 1100), 35, ("chacha", 36, 8), 1080, "toy"),
    ("wild_a", (2, 64, 4, 160, 96, 64), 41, ("chacha", 42, 5), 16, "wild"),
    ("wild_b", (3, 128, 8, 352, 300, 96), 43, ("chacha", 44, 7), 24, "wild"),
    ("tinyllama_c1", (22, 2048, 32, 5632, 32000, 2048), 1, ("chacha", 2, 16), 8, "toy"),
]


def wild_model(ref: Reference, cfg: Config, seed: int):
    toy = ref.gen_toy(seed, cfg)
    w, s, n = toy.export()
    rng = np.random.default_rng(seed)
    s = rng.integers(1, 1 << 22, size=s.shape, dtype=np.int64)          # huge row scales
    n = rng.integers(-(1 << 21), 1 << 21, size=n.shape, dtype=np.int64)  # signed, large gains
    return ref.model_from_arrays(cfg, w, s, n), (s, n)


def make_models(ref: Reference):
    out = {}
    for name, c6, seed, pspec, max_new, kind in MODEL_CASES:
        cfg = Config(*c6)
        if isinstance(pspec, tuple):
            prompt = ref.prompt(pspec[1], cfg.vocab, pspec[2])
        else:
            prompt = np.array(pspec, np.uint32)
        extra = {}
        if kind == "toy":
            m = ref.gen_toy(seed, cfg)
            wh = m.weight_hash()
        else:
            m, (s, n) = wild_model(ref, cfg, seed)
            wh = None
            extra = {"wild_rng": "numpy.default_rng(seed): scales in [1,2^22), norms in [-2^21,2^21)"}
        toks, h, logits = ref.generate_greedy(m, prompt, max_new, keep_logits=True)
        out[name] = {
            "config": list(c6), "rope_theta": cfg.rope_theta, "seed": seed, "kind": kind,
            "prompt": [int(t) for t in prompt], "max_new": max_new,
            "weight_hash": wh, "tokens": [int(t) for t in toks], "output_hash": h,
            "logits_digest": digest_logits(ref, logits),
            "last_logits_head": [int(v) for v in logits[-1][:8]], **extra,
        }
        print(name, h, flush=True)
    return out


def make_kat(ref: Reference):
    pat = lambda n: bytes(i % 251 for i in range(n))  # noqa: E731
    b3 = {str(n): ref.blake3(pat(n)) for n in (0, 1, 63, 64, 65, 1023, 1024, 1025, 2048, 2049,
                                               3072, 4096, 5000, 8192, 31744, 100000)}
    rng = np.random.default_rng(5)
    inv_x = [1, 2, 3, 65535, 65536, 65537, 131072, 262144, (1 << 24) + 1, 1 << 40, (1 << 62) + 12345,
             (1 << 63) - 1] + [int(v) for v in rng.integers(1, 1 << 62, 200)] + \
            [int(v) for v in rng.integers(1, 1 << 30, 200)]
    inv = [ref.inv_sqrt(x) for x in inv_x]
    sig_x = sorted(set([0, 1, -1, 8 * ONE, -8 * ONE, 8 * ONE + 1, -(8 * ONE) - 1, ONE, -ONE,
                        (1 << 62), -(1 << 62)] +
                       [int(v) for v in rng.integers(-12 * ONE, 12 * ONE, 3000)]))
    sig = [ref.lib.ref_sigmoid(x) for x in sig_x]
    silu = [ref.lib.ref_silu(x) for x in sig_x]
    rope = {}
    for theta, dh, ctx in ((10000.0, 128, 4096), (10000.0, 64, 2048), (10000.0, 4, 16),
                           (500000.0, 16, 64)):
        c, s = ref.rope_tables(theta, dh, ctx)
        rope[f"{theta}_{dh}_{ctx}"] = {"cos_digest": ref.blake3(c.tobytes()),
                                       "sin_digest": ref.blake3(s.tobytes()),
                                       "cos_last": [int(v) for v in c[-(dh // 2):]],
                                       "sin_last": [int(v) for v in s[-(dh // 2):]]}
    prompts = {f"{seed}_{v}_{n}": [int(t) for t in ref.prompt(seed, v, n)]
               for seed, v, n in ((2, 32000, 16), (8, 32000, 16), (9, 32000, 2048),
                                  (10, 32000, 16), (1001, 32000, 16))}
    return {"blake3_pattern": b3, "exp_lut": [int(v) for v in ref.exp_lut()],
            "inv_sqrt": {"x": inv_x, "y": inv}, "sigmoid": {"x": sig_x, "y": sig, "silu": silu},
            "rope": rope, "prompts": prompts}


def make_ops(ref: Reference):
    from oracle.pyoracle import _ptr, i8p, i64p  # noqa
    rng = np.random.default_rng(17)
    ops = {}
    # dense: random shapes incl. odd K, activations from small to near-wrap
    cases = []
    for i in range(60):
        rows = int(rng.integers(1, 70))
        cols = int(rng.choice([1, 3, 4, 7, 15, 16, 17, 31, 64, 100, 513, 1000, 2048]))
        mag = int(rng.choice([4 * ONE, 1 << 23, 1 << 31, 1 << 40, 1 << 56, 1 << 62]))
        w = rng.integers(-127, 128, (rows, cols), dtype=np.int64).astype(np.int8)
        s = rng.integers(1, 1 << int(rng.choice([4, 17, 40])), rows, dtype=np.int64)
        x = rng.integers(-mag, mag, cols, dtype=np.int64)
        out = np.empty(rows, np.int64)
        assert ref.lib.ref_dense(rows, cols, _ptr(w, i8p), _ptr(s, i64p), _ptr(x, i64p), 0,
                                 _ptr(out, i64p)) == 0
        cases.append((w, s, x, out))
    ops["dense"] = cases
    # rmsnorm
    cases = []
    for i in range(40):
        n = int(rng.choice([1, 4, 16, 64, 100, 4096]))
        mag = int(rng.choice([1, ONE, 256 * ONE, 1 << 40]))
        x = rng.integers(-mag, mag + 1, n, dtype=np.int64)
        g = rng.integers(ONE // 2, 3 * ONE // 2, n, dtype=np.int64)
        out = np.empty(n, np.int64)
        assert ref.lib.ref_rmsnorm(_ptr(x, i64p), _ptr(g, i64p), n, _ptr(out, i64p)) == 0
        cases.append((x, g, out))
    ops["rmsnorm"] = cases
    # softmax
    cases = [np.array([0, -20 * ONE], np.int64), np.array([42], np.int64),
             np.array([123, 123], np.int64)]
    for i in range(40):
        n = int(rng.integers(1, 600))
        cases.append(rng.integers(-20 * ONE, 20 * ONE, n, dtype=np.int64))
    outs = []
    for s in cases:
        out = np.empty(len(s), np.int64)
        assert ref.lib.ref_softmax(_ptr(s, i64p), len(s), _ptr(out, i64p)) == 0
        outs.append(out)
    ops["softmax"] = list(zip(cases, outs))
    # attention: T consecutive steps
    cases = []
    for H, dh, T, mag in ((2, 4, 4, 4 * ONE), (4, 8, 20, 8 * ONE), (32, 128, 6, 4 * ONE),
                          (3, 64, 33, 1 << 20), (2, 16, 10, 1 << 40)):
        D = H * dh
        q = rng.integers(-mag, mag, (T, D), dtype=np.int64)
        k = rng.integers(-mag, mag, (T, D), dtype=np.int64)
        v = rng.integers(-mag, mag, (T, D), dtype=np.int64)
        out = np.empty((T, D), np.int64)
        assert ref.lib.ref_attention(H, dh, max(T, 16), 10000.0, T, _ptr(q, i64p), _ptr(k, i64p),
                                     _ptr(v, i64p), 1, _ptr(out, i64p)) == 0
        cases.append(((H, dh, max(T, 16)), q, k, v, out))
    ops["attention"] = cases
    # ffn
    cases = []
    for d, f in ((4, 6), (16, 40), (64, 172), (100, 300)):
        wg = rng.integers(-127, 128, (f, d)).astype(np.int8)
        wu = rng.integers(-127, 128, (f, d)).astype(np.int8)
        wd = rng.integers(-127, 128, (d, f)).astype(np.int8)
        sg, su = (rng.integers(1, 65536, f, dtype=np.int64) for _ in range(2))
        sd = rng.integers(1, 65536, d, dtype=np.int64)
        x = rng.integers(-4 * ONE, 4 * ONE, d, dtype=np.int64)
        out = np.empty(d, np.int64)
        assert ref.lib.ref_ffn(d, f, _ptr(wg, i8p), _ptr(sg, i64p), _ptr(wu, i8p), _ptr(su, i64p),
                               _ptr(wd, i8p), _ptr(sd, i64p), _ptr(x, i64p), _ptr(out, i64p)) == 0
        cases.append((wg, sg, wu, su, wd, sd, x, out))
    ops["ffn"] = cases
    flat = {}
    for kind, cs in ops.items():
        flat[f"{kind}_n"] = np.array(len(cs))
        for i, c in enumerate(cs):
            for j, a in enumerate(c):
                flat[f"{kind}_{i}_{j}"] = np.asarray(a)
    return flat


def main():
    ref = Reference()
    kat = make_kat(ref)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **make_ops(ref))
    models = make_models(ref)
    with open(os.path.join(HERE, "models.json"), "w") as f:
        json.dump(models, f, indent=1)


if __name__ == "__main__":
    main()
