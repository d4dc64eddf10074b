"""C3 workload: 7B-shaped model, 2048-token synthetic prompt, prefill time on
the tensor cores vs the decode kernel, and the continuation compared."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
prompt = P.prompt_from_seed(9, cfg.vocab, 2048)
out = {}
for mode in ("1", "2"):
    os.environ["DIMG_PREFILL"] = mode
    s = P.InferenceSession(m)
    times = []
    for rep in range(2 if mode == "1" else 1):
        s.begin(prompt, 8)
        t = time.time()
        s.prefill()
        s.sync()
        times.append(time.time() - t)
    s.decode(8)
    s.sync()
    out[mode] = s.tokens(8)
    print("mode", mode, "prefill s", ["%.4f" % x for x in times], "stats", s.stats(), "tokens", out[mode], flush=True)
print("same continuation:", out["1"] == out["2"])
