"""C5 B=8 and B=64 timing for settings of one environment knob (each in
its own process), hashes checked against the goldens.

    python tools/batch_ab.py DIMG_STREAMK 0 1
"""
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
gold = json.load(open("tests/golden/models_7b.json"))
for B in (8, 64):
    prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in range(B)]
    P.generate_greedy_batch(m, prompts, 128)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        res, path = P.generate_greedy_batch(m, prompts, 128)
        best = min(best, time.perf_counter() - t)
    ok = sum(res[i].output_hash.hex() == gold[f"c5_{i}"]["output_hash"] for i in range(B) if f"c5_{i}" in gold)
    print(f"B={B} {best:.4f} s {B * 128 / best:.0f} tok/s golden {ok} {path}")
'''
def main():
    knob, vals = sys.argv[1], sys.argv[2:]
    for rnd in range(2):
        for v in vals:
            o = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **{knob: v}), capture_output=True,
                               text=True)
            print(f"{knob}={v}: " + (" | ".join(o.stdout.strip().splitlines()) or o.stderr[-800:]), flush=True)


if __name__ == "__main__":
    main()
