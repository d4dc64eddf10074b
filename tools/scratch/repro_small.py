"""Small-model generate for debugging (compute-sanitizer friendly)."""
import sys
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(*(int(x) for x in (sys.argv[1:7] if len(sys.argv) > 6 else (2, 16, 2, 32, 32, 64))))
m = P.gen_toy_model(7, cfg)
r = P.generate_greedy(m, [1, 2, 3], 4)
print("ok", r.token_ids)
