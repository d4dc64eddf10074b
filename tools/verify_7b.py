"""verify_by_reexecution of a 7B attestation (16-token prompt, 128 new
tokens): wall time of the whole call (model id by the GPU BLAKE3 of the
6.75 GB container, prompt hash, deserialize, model upload, one greedy
re-execution on the GPU) and of make_attestation."""
import sys, time
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
prompt = P.prompt_from_seed(8, cfg.vocab, 16)
res = P.generate_greedy(m, prompt, 128)
t = time.perf_counter()
att = P.make_attestation(m.bytes, prompt, res, 1000, 100)
t_make = time.perf_counter() - t
for _ in range(2):
    t = time.perf_counter()
    out = P.verify_by_reexecution(att, m.bytes, prompt, 128)
    t_ver = time.perf_counter() - t
print(f"make_attestation {t_make:.2f} s   verify_by_reexecution {t_ver:.2f} s   {out.to_text()}   "
      f"output {res.output_hash.hex()[:16]}")
