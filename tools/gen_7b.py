"""gen_toy_model at 7B: host generator (all cores) vs the weight stream on
the GPU (keystream + compaction on the device, then the container copy)."""
import sys, time
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
P.gen_toy_model(1, P.ModelConfig(1, 8, 1, 8, 8, 8), device=0)  # CUDA context
t = time.perf_counter(); g = P.gen_toy_model(7, cfg, device=0); tg = time.perf_counter() - t
t = time.perf_counter(); h = P.gen_toy_model(7, cfg); th = time.perf_counter() - t
print(f"7B gen_toy_model: gpu {tg:.2f} s   host {th:.2f} s   same weight hash {g.weight_hash == h.weight_hash}")
