"""One C5-style batched generation at 7B (B sequences, P=16, N new) -- profiling workload."""
import sys
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in range(B)]
res, path = P.generate_greedy_batch(m, prompts, N)
print("ok", path, res[0].token_ids)
