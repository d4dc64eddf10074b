"""Decode ms/token at 7B (C2 prompt, positions 24..151) for settings of one
environment knob, each checked against the C2 golden tokens.

    python tools/decode_sweep.py DIMG_L2PF 0 2 4 8
"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402

knob, vals = sys.argv[1], sys.argv[2:]
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "models_7b.json")))["c2"]
prompt = P.prompt_from_seed(8, cfg.vocab, 16)
s = P.InferenceSession(m)
B = 6.620346376e9
for rep in range(2):
    for v in vals:
        os.environ[knob] = v
        s.begin(prompt, 136)
        s.prefill()
        s.decode(8)
        s.sync()
        ms = s.time_decode(128)
        ok = s.tokens(136)[:128] == gold["tokens"]
        st = ms / 128
        print(f"{knob}={v:>5s}  {st * 1e3:7.1f} us/token  {1e3 / st:6.1f} tok/s  {B / (st * 1e-3) / 6546.6e9:.3f} of HBM  tokens_ok={ok}",
              flush=True)
