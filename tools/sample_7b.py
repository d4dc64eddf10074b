"""generate_sampled at 7B (16-token prompt, 128 tokens, T = 0.8 in Q16):
wall time of the call (key = GPU BLAKE3 of the 6.75 GB container + prompt,
prefill, 128 one-step launches each followed by the device sampler) vs
generate_greedy on the same session."""
import sys, time
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
prompt = P.prompt_from_seed(8, cfg.vocab, 16)
T = int(0.8 * 65536)
P.generate_greedy(m, prompt, 8)
key = P.sample_key(m.bytes, prompt)
sess = P.engine._cached_session(m, P.EngineOptions(), 0, None)
for _ in range(2):
    t = time.perf_counter(); r = sess.generate_sampled(prompt, 128, T, key); ts = time.perf_counter() - t
t = time.perf_counter(); key2 = P.sample_key(m.bytes, prompt); tk = time.perf_counter() - t
t = time.perf_counter(); g = P.generate_greedy(m, prompt, 128); tg = time.perf_counter() - t
print(f"sampled 128: {ts:.3f} s = {128 / ts:.0f} tok/s (key {tk:.2f} s)   greedy 128: {tg:.3f} s = {128 / tg:.0f} tok/s"
      f"   distinct sampled tokens {len(set(r.token_ids))}")
