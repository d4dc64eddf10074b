"""7B-shaped goldens, written to models_7b.json.

    python tests/golden/make_golden_7b.py ref    C2 + smoke-7B with the REFERENCE
                                                 engine (oracle/_ref; ~10 min)
    python tests/golden/make_golden_7b.py c4     C4 (P=16, N=1024) with the C oracle
    python tests/golden/make_golden_7b.py c5 I J C5 sequences I..J-1 with the C oracle
    python tests/golden/make_golden_7b.py c3     C3 (P=2048, N=8) with the C oracle

The C-oracle goldens are pinned by the oracle's bit-agreement with the
reference on C1 and C2 (tests/test_oracle.py); the reference itself would
need hours per config (3.2 s/forward, single-threaded dense).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
from oracle.pyoracle import Config, Oracle, Reference  # noqa: E402

OUT = os.path.join(HERE, "models_7b.json")
C7B = (32, 4096, 32, 11008, 32000, 4096)


def load():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return {}


def save(d):
    with open(OUT + ".tmp", "w") as f:
        json.dump(d, f, indent=1)
    os.replace(OUT + ".tmp", OUT)


def record(name, engine, cfg6, seed, prompt_seed, P, N, toks, h, logits_digest, wh, secs):
    d = load()
    d[name] = {"config": list(cfg6), "seed": seed, "prompt_seed": prompt_seed, "P": P,
               "max_new": N, "engine": engine, "weight_hash": wh,
               "tokens": [int(t) for t in toks], "output_hash": h,
               "logits_digest": logits_digest, "seconds": round(secs, 1)}
    save(d)
    print(name, h, flush=True)


def main():
    what = sys.argv[1]
    cfg = Config(*C7B)
    if what == "ref":
        ref = Reference()
        t = time.time()
        m = ref.gen_toy(7, cfg)
        wh = m.weight_hash()
        print("gen", time.time() - t, wh, flush=True)
        p = ref.prompt(8, cfg.vocab, 16)
        t = time.time()
        toks, h, lg = ref.generate_greedy(m, p[:4], 2, keep_logits=True)
        record("smoke7b", "reference", C7B, 7, 8, 4, 2, toks, h, ref.blake3(lg.tobytes()), wh,
               time.time() - t)
        t = time.time()
        toks, h, lg = ref.generate_greedy(m, p, 128, keep_logits=True)
        record("c2", "reference", C7B, 7, 8, 16, 128, toks, h, ref.blake3(lg.tobytes()), wh,
               time.time() - t)
        return
    orc = Oracle()
    t = time.time()
    m = orc.gen_toy(7, cfg)
    print("gen", time.time() - t, flush=True)
    if what == "c4":
        p = orc.prompt(10, cfg.vocab, 16)
        t = time.time()
        toks, h, _ = orc.generate_greedy(m, p, 1024)
        record("c4", "oracle", C7B, 7, 10, 16, 1024, toks, h, None, None, time.time() - t)
    elif what == "c3":
        p = orc.prompt(9, cfg.vocab, 2048)
        t = time.time()
        toks, h, lg = orc.generate_greedy(m, p, 8, keep_logits=True)
        record("c3", "oracle", C7B, 7, 9, 2048, 8, toks, h, orc.blake3_array(lg), None,
               time.time() - t)
    elif what == "c5":
        lo, hi = int(sys.argv[2]), int(sys.argv[3])
        for i in range(lo, hi):
            ps = 8 if i == 0 else 1000 + i
            p = orc.prompt(ps, cfg.vocab, 16)
            t = time.time()
            toks, h, _ = orc.generate_greedy(m, p, 128)
            record(f"c5_{i}", "oracle", C7B, 7, ps, 16, 128, toks, h, None, None, time.time() - t)


if __name__ == "__main__":
    main()
