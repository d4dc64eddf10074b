"""Workload for ncu: 7B model, prompt prefill (launch 1), a warm-up decode of
`skip` steps (launch 2), then a 2-step decode (launch 3) of the persistent
kernel -- profile launch 3 (position 16 + skip)."""
import sys
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
skip = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
s = P.InferenceSession(m)
s.begin(P.prompt_from_seed(8, cfg.vocab, 16), skip + 8)
s.prefill()
s.decode(max(1, skip))
s.decode(2)
s.sync()
print("ok", s.tokens(2))
