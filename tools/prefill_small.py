"""Prefill time of short and long prompts at 7B, tensor cores (DIMG_PREFILL=1)
vs one decode step per position (DIMG_PREFILL=2): where the auto threshold
belongs. CUDA events around dimg_session_time_prefill."""
import os, sys
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
s = P.InferenceSession(m)
for n in [int(x) for x in (sys.argv[1:] or "2 4 8 12 16 17 24 32 64".split())]:
    row = []
    for mode in ("1", "2"):
        os.environ["DIMG_PREFILL"] = mode
        best = None
        for _ in range(3):
            s.begin(P.prompt_from_seed(9, cfg.vocab, n), 1)
            ms, tc = s.time_prefill()
            best = ms if best is None else min(best, ms)
        row.append((best, tc))
    print(f"n={n:5d}  tensor cores {row[0][0]:8.2f} ms ({row[0][1]})   decode steps {row[1][0]:8.2f} ms", flush=True)
