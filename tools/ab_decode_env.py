"""A/B decode timing of one library under settings of an environment knob:
each setting in its own subprocess, alternated over rounds (same child as
tools/ab_decode.py: 7B, C2 prompt, 128 steps after 8, tokens checked).

    python tools/ab_decode_env.py DIMG_ATTN_PARTS 2 4 8 [--rounds 4]
"""
import json
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ab_decode import CHILD  # noqa: E402  (module body runs only under __main__ guard below)

args = sys.argv[1:]
rounds = 4
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    del args[i:i + 2]
knob, values = args[0], args[1:]
res = {v: [] for v in values}
for r in range(rounds):
    for v in values:
        o = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **{knob: v}), capture_output=True,
                           text=True)
        if o.returncode:
            print(v, o.stderr[-2000:])
            sys.exit(1)
        res[v] += json.loads(o.stdout.strip().splitlines()[-1])
for v, t in res.items():
    print(f"{knob}={v}: median {statistics.median(t):.1f} us/token  min {min(t):.1f}  max {max(t):.1f}  (n={len(t)})")
