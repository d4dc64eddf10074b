"""CTA 0's timeline through one decode step of the persistent kernel at 7B
(dimg_session_trace: %globaltimer at stage start / prologue done / chunk loop
done / stage end, clock64 sub-stamps). Prints the mean over layers of each
stage's phases and the gap to the next stage, and the attention sub-steps.

    python tools/stage_trace.py [n0]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402

cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg, device=0)
s = P.InferenceSession(m)
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 130
s.begin(P.prompt_from_seed(8, cfg.vocab, 16), n0 + 8)
s.prefill()
s.decode(n0)
s.sync()
ns = 5 * cfg.n_layers + 1
tr = s.trace(2, 2 * ns).astype(np.int64)
t = tr[ns:2 * ns]  # the second step
names = ["qkv", "attn", "wo", "gu", "down"]
ghz = 1.965
print(f"position {16 + n0 + 1}: CTA 0, mean over layers 1..31 (us)")
print("stage   prologue   chunks   epilogue->end   gap-to-next-start")
for k, nm in enumerate(names):
    rows = [t[5 * l + k] for l in range(1, cfg.n_layers)]
    nxt = [t[5 * l + k + 1] for l in range(1, cfg.n_layers)]
    pro = np.mean([r[1] - r[0] for r in rows]) / 1e3
    ch = np.mean([r[2] - r[1] for r in rows]) / 1e3
    ep = np.mean([r[3] - r[2] for r in rows]) / 1e3
    gap = np.mean([n[0] - r[3] for r, n in zip(rows, nxt)]) / 1e3
    print(f"{nm:6s} {pro:9.2f} {ch:9.2f} {ep:12.2f} {gap:14.2f}")
lay = np.mean([t[5 * l + 5][0] - t[5 * l][0] for l in range(1, cfg.n_layers - 1)]) / 1e3
print(f"layer total {lay:.2f} us")
# norm prologue sub-steps (clock64): 8 start, 4 copy/poll done, 6 r computed, 7 planes done
for k, nm in ((0, "qkv"), (3, "gu")):
    rows = [t[5 * l + k] for l in range(1, cfg.n_layers)]
    a = np.mean([r[4] - r[8] for r in rows]) / ghz / 1e3
    b = np.mean([r[6] - r[4] for r in rows]) / ghz / 1e3
    c = np.mean([r[7] - r[6] for r in rows]) / ghz / 1e3
    print(f"{nm} norm prologue: poll+sumsq {a:.2f}  r {b:.2f}  planes {c:.2f} us")
# attention sub-steps of CTA 0 (head 0 part 0), clock64
rows = [t[5 * l + 1] for l in range(1, cfg.n_layers)]
steps = [(9, 10, "rope rows"), (10, 11, "spec K/V loads"), (11, 13, "poll q/k/v"), (13, 12, "rope+append"),
         (12, 4, "decisions"), (4, 14, "scores"), (14, 17, "gather peers' scores"), (17, 5, "sync"),
         (5, 6, "softmax"), (6, 19, "PV"), (19, 20, "sync"), (20, 21, "sum+publish")]
for a_, b_, nm in steps:
    v = np.mean([r[b_] - r[a_] for r in rows]) / ghz / 1e3
    print(f"  attn {nm:24s} {v:6.2f} us")
