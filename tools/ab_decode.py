"""A/B decode timing of library builds on one GPU: each build in its own
subprocess (DIMG_LIB=...), alternated over rounds so clock / thermal drift
hits both; prints per-build median us/token (7B, C2 prompt, 128 steps after 8).

    python tools/ab_decode.py LIB_A LIB_B [rounds]
"""
import json
import os
import statistics
import subprocess
import sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
gold = json.load(open("tests/golden/models_7b.json"))["c2"]
s = P.InferenceSession(m)
out = []
for _ in range(5):
    s.begin(P.prompt_from_seed(8, cfg.vocab, 16), 136)
    s.prefill(); s.decode(8); s.sync()
    out.append(s.time_decode(128) / 128 * 1e3)
    assert s.tokens(136)[:128] == gold["tokens"]
print(json.dumps(out))
'''

if __name__ == "__main__":
    libs = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    res = {lib: [] for lib in libs}
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, DIMG_LIB=os.path.abspath(lib))
            o = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            if o.returncode:
                print(lib, o.stderr[-2000:])
                sys.exit(1)
            res[lib] += json.loads(o.stdout.strip().splitlines()[-1])
    for lib, v in res.items():
        print(f"{lib}: median {statistics.median(v):.1f} us/token  min {min(v):.1f}  max {max(v):.1f}  (n={len(v)})")
