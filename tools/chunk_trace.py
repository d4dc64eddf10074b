"""Ring-wait timeline of the persistent decode kernel (experiment build).

    tools/build_variant.sh ct -DDIMG_CHUNK_TRACE
    DIMG_LIB=tools/_libs/libdimg_ct.so python tools/chunk_trace.py [n0] [layer]

Warp 0 of every CTA logs clock64 before/after each weight-ring wait plus
stage markers (start, prologue end, chunk-loop end) for one decode step at
position 16 + n0. Prints, per stage of one layer, the median over CTAs of:
prologue, chunk loop, the time warp 0 spent blocked on the ring inside the
chunk loop, and the number of its chunks.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402
from paper_2603_24904_b200._lib import lib  # noqa: E402

CT_MAX = 4096
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
s = P.InferenceSession(m)
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 130
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s.begin(P.prompt_from_seed(8, cfg.vocab, 16), n0 + 4)
s.prefill()
s.decode(n0)
s.decode(1)
s.sync()
buf = np.zeros(148 * CT_MAX * 2, np.uint64)
assert lib.dimg_debug_chunk_trace(buf.ctypes.data_as(C.c_void_p)) == 0
t = buf.reshape(148, CT_MAX, 2)
names = ["qkv", "attn", "wo", "gu", "down"]
ghz = 1.965
res = {}
for cta in range(148):
    ev = t[cta]
    n = int(np.argmax(ev[:, 0] == 0)) if (ev[:, 0] == 0).any() else CT_MAX
    ev = ev[:n]
    cur = None
    for c0, c1 in ev:
        c0 = int(c0); c1 = int(c1)
        if c1 >> 63:
            si, kind = (c1 >> 8) & 0xFFFF, c1 & 0xFF
            if kind == 0:
                cur = {"si": si, "start": c0, "wait": 0, "n": 0, "first_wait": None}
            elif kind == 1 and cur:
                cur["pro"] = c0
            elif kind == 2 and cur:
                cur["end"] = c0
                res.setdefault(si, []).append(cur)
        elif cur is not None and "pro" in cur and "end" not in cur:
            cur["wait"] += c1 - c0
            cur["n"] += 1
            if cur["first_wait"] is None:
                cur["first_wait"] = c1 - c0
print(f"position {16 + n0 + 1}, layer {layer}: medians over CTAs (us)")
print("stage  from-start-to-prologue-end  chunk-loop  ring-wait  first-wait  chunks(w0)")
step_si = sorted(res)
for si in step_si:
    if si // 5 != layer and not (si == 5 * cfg.n_layers):
        continue
    nm = "head" if si == 5 * cfg.n_layers else names[si % 5]
    r = res[si]
    pro = np.median([x["pro"] - x["start"] for x in r]) / ghz / 1e3
    loop = np.median([x["end"] - x["pro"] for x in r]) / ghz / 1e3
    wait = np.median([x["wait"] for x in r]) / ghz / 1e3
    fw = np.median([x["first_wait"] or 0 for x in r]) / ghz / 1e3
    nc = np.median([x["n"] for x in r])
    print(f"{nm:6s} {pro:10.2f} {loop:12.2f} {wait:10.2f} {fw:10.2f} {nc:8.0f}")
# whole-step totals over all layers
tot = {k: [] for k in names}
for si in step_si:
    if si == 5 * cfg.n_layers:
        continue
    r = res[si]
    tot[names[si % 5]].append((np.median([x["pro"] - x["start"] for x in r]),
                               np.median([x["end"] - x["pro"] for x in r]),
                               np.median([x["wait"] for x in r])))
print("mean over layers: stage  prologue  loop  wait (us)")
for k, v in tot.items():
    if v:
        a = np.array(v).mean(0) / ghz / 1e3
        print(f"  {k:6s} {a[0]:7.2f} {a[1]:7.2f} {a[2]:7.2f}")

# per-chunk timeline of warp 0 in a few CTAs for the chosen layer: the gap
# between one wait's end and the next wait's start is the chunk's compute
# (+ release / epilogue at group ends)
np.save("gpurun_out/ct_raw.npy", t)
for cta in (0, 37, 74, 111):
    ev = t[cta]
    lines = []
    inside = False
    prev_end = None
    for c0, c1 in ev:
        c0 = int(c0); c1 = int(c1)
        if c0 == 0:
            break
        if c1 >> 63:
            si, kind = (c1 >> 8) & 0xFFFF, c1 & 0xFF
            inside = si // 5 == layer
            if inside:
                lines.append(f"  [{names[si % 5]} marker {kind} @ {c0}]")
            prev_end = c0 if kind == 1 else None
            continue
        if inside:
            comp = (c0 - prev_end) if prev_end else -1
            lines.append(f"    compute-before {comp:6d} clk  wait {c1 - c0:6d} clk")
        prev_end = c1
    print(f"CTA {cta}:")
    print("\n".join(lines))
