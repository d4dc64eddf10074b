"""C5 workload: 7B-shaped model, B independent sequences (prompt seeds 8,
1001, 1002, ...; P=16, N=128) generated together; wall time of the call and
the per-sequence hashes against the committed C5 goldens."""
import json, os, sys, time
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
gold = json.load(open("tests/golden/models_7b.json"))
for B in [int(x) for x in (sys.argv[1:] or ["8", "64"])]:
    prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in range(B)]
    P.generate_greedy_batch(m, prompts, 128)  # warm: buffers + the captured step graph
    t = time.perf_counter()
    res, path = P.generate_greedy_batch(m, prompts, 128)
    dt = time.perf_counter() - t
    ok = [res[i].output_hash.hex() == gold[f"c5_{i}"]["output_hash"] for i in range(B) if f"c5_{i}" in gold]
    print(f"B={B} path={path} {dt:.3f} s  {B * 128 / dt:.0f} tok/s  golden {sum(ok)}/{len(ok)}", flush=True)
