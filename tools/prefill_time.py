"""C3 prefill time at 7B (2048-token prompt, seed 9): tensor-core prefill +
the last position's decode step, CUDA events, 2 warm + 3 timed; the first
token checked against the golden."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402

cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "models_7b.json")))["c3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
prompt = P.prompt_from_seed(9, cfg.vocab, n)
s = P.InferenceSession(m)
ts = []
for i in range(5):
    s.begin(prompt, 1)
    ms, tc = s.time_prefill()
    ms += s.time_decode(1)
    if i >= 2:
        ts.append(ms)
print(f"n={n} prefill+first token {sorted(ts)[1]:.2f} ms (tc={tc}) first token {s.tokens(1)} golden {gold['tokens'][:1]}",
      flush=True)
