"""Per-stage hand-off skew of the persistent decode kernel at 7B: every
CTA's prologue-end and chunk-loop-end time per GEMV stage (position 16+n0).

    python tools/skew_trace.py [n0]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402
from paper_2603_24904_b200._lib import lib, u64p  # noqa: E402

cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
s = P.InferenceSession(m)
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 130
s.begin(P.prompt_from_seed(8, cfg.vocab, 16), n0 + 4)
s.prefill()
s.decode(n0)
s.sync()
ns = 5 * cfg.n_layers + 1
grid = 148
out = np.zeros(2 * ns * grid * 2, np.uint64)
rc = lib.dimg_session_trace_all(s._h, 2, out.ctypes.data_as(u64p), 2 * ns)
assert rc == 0, lib.dimg_last_error()
t = out.reshape(2 * ns, grid, 2).astype(np.int64)
names = ["qkv", "attn", "wo", "gu", "down"]
agg = {}
for i in range(ns, 2 * ns):
    k = i - ns
    name = "head" if k == ns - 1 else names[k % 5]
    if name == "attn":
        continue
    pe, ce = t[i, :, 0], t[i, :, 1]
    ok = (pe > 0) & (ce > 0)
    pe, ce = pe[ok], ce[ok]
    if len(ce) == 0:
        continue
    base = pe.min()
    agg.setdefault(name, []).append(((pe.max() - pe.min()) / 1e3, (ce.max() - ce.min()) / 1e3,
                                     np.median(ce - pe) / 1e3, (ce - pe).max() / 1e3, (ce - pe).min() / 1e3,
                                     (np.percentile(ce, 90) - np.percentile(ce, 10)) / 1e3))
print(f"position {16 + n0}: us, mean over layers")
print("stage  prologue-end spread  chunk-end spread  chunk-loop median/max/min   chunk-end p90-p10")
for k, v in agg.items():
    a = np.array(v).mean(0)
    print(f"{k:5s}  {a[0]:8.2f}            {a[1]:8.2f}          {a[2]:6.2f} {a[3]:6.2f} {a[4]:6.2f}        {a[5]:6.2f}")
# next-stage start vs previous chunk end: which CTA finishes last
last = {}
for i in range(ns, 2 * ns - 1):
    ce = t[i, :, 1]
    if ce.max() > 0:
        j = int(np.argmax(ce))
        last[j] = last.get(j, 0) + 1
print("CTAs most often last:", sorted(last.items(), key=lambda x: -x[1])[:12])
