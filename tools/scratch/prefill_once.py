"""One 7B tensor-core prefill of a 2048-token prompt (profiling workload)."""
import os, sys
sys.path.insert(0, ".")
os.environ["DIMG_PREFILL"] = "1"
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
s = P.InferenceSession(m)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s.begin(P.prompt_from_seed(9, cfg.vocab, n), 1)
s.prefill()
s.sync()
print("ok", s.stats())
