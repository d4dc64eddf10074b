import os, sys, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2603_24904_b200 as P
from conftest import wild_arrays
g = json.load(open("tests/golden/models.json"))[sys.argv[1] if len(sys.argv) > 1 else "wild_a"]
cfg = P.ModelConfig(*g["config"], rope_theta=g["rope_theta"])
m = P.gen_toy_model(g["seed"], cfg)
names = ["tok_embd"] + [f"layers.{l}.{t}" for l in range(cfg.n_layers) for t in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")] + ["output"]
tens = [m.tensor(n) for n in names]
s, n = wild_arrays(g["config"], g["seed"], np.concatenate([s for _, s in tens]), m.norms())
out, o = [], 0
for w, s0 in tens:
    out.append((w.copy(), s[o:o + len(s0)])); o += len(s0)
mw = P.ModelFile.from_arrays(cfg, out, n)
print("config", g["config"], "prompt", len(g["prompt"]))
r = P.generate_greedy(mw, g["prompt"], g["max_new"])
print("ok", r.token_ids == g["tokens"])
