"""C5 B=8 step time with launch chains removed (DIMG_BD_SKIP experiment
knob; outputs are wrong by construction): what the norms, RoPE/KV and
attention launches cost inside the graph-replayed step.

    python tools/batch_skip.py
"""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in range(8)]
P.generate_greedy_batch(m, prompts, 128)
best = 1e9
for _ in range(3):
    t = time.perf_counter()
    res, path = P.generate_greedy_batch(m, prompts, 128)
    best = min(best, time.perf_counter() - t)
print(f"{best:.4f} {path}")
'''
for sk in ("0", "1", "2", "4", "7"):
    o = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, DIMG_BD_SKIP=sk), capture_output=True, text=True)
    print(f"DIMG_BD_SKIP={sk}: {o.stdout.strip() or o.stderr[-500:]}", flush=True)
