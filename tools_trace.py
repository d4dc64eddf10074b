"""Per-stage phase breakdown of the persistent decode kernel (CTA 0 stamps).

    python tools_trace.py [decode_steps_before]   (position = 16 + that)
"""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
s = P.InferenceSession(m)
prompt = P.prompt_from_seed(8, cfg.vocab, 16)
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s.begin(prompt, n0 + 8)
s.prefill()
s.decode(n0)
ns = 5 * cfg.n_layers + 1
tr = s.trace(2, 2 * ns).astype(np.int64)
names = ["qkv", "attn", "wo", "gu", "down"]
ghz = 1.965e-3  # clock64 cycles per ns at the max SM clock (approximate)
rows, sub, att = {}, {}, []
for i in range(ns, 2 * ns):
    k = i - ns
    name = "head" if k == ns - 1 else names[k % 5]
    t = tr[i]
    nxt = tr[i + 1][0] if i + 1 < 2 * ns else t[3]
    rows.setdefault(name, []).append((t[1] - t[0] if t[1] else 0, t[2] - t[1] if t[2] else 0,
                                      t[3] - (t[2] if t[2] else t[0]), nxt - t[3]))
    if t[4]:
        c = t[8]
        sub.setdefault(name, []).append(((t[4] - c) / ghz, (t[5] - t[4]) / ghz, (t[6] - t[5]) / ghz,
                                         (t[7] - t[6]) / ghz))
    if name == "attn" and t[9]:
        att.append(t)
print("position", 16 + n0)
print("stage   prologue  chunks  epilogue  barrier (us) | sub-steps (us)")
for k, v in rows.items():
    a = np.array(v).mean(0) / 1e3
    extra = ""
    if k in sub:
        b = np.array(sub[k]).mean(0) / 1e3
        extra = "  | " + " ".join(f"{x:5.2f}" for x in b)
    print(f"{k:6s} {a[0]:9.2f} {a[1]:7.2f} {a[2]:9.2f} {a[3]:8.2f}{extra}")
if att:
    # attention stamps: 8 stage start, 9 entry, 10 L2 loads issued, 11 K/V issued,
    # 12 rope done, 4 decisions synced, 14 scores done, 15 published, 16 peers met,
    # 17 gathered, 5 synced, 6 softmax done, 19 PV done, 20 synced, 21 out written, 7 end
    order = [(8, "start"), (9, "entry"), (10, "L2 loads issued"), (11, "K/V issued"), (12, "rope"),
             (4, "decisions"), (14, "scores"), (15, "published"), (16, "peers met"), (17, "gathered"),
             (5, "synced"), (6, "softmax"), (19, "PV"), (20, "synced"), (21, "out"), (7, "end")]
    a = np.array(att)
    prev = None
    print("attention (CTA 0 = head 0 part 0), mean us per step:")
    for idx, nm in order:
        if prev is not None and a[:, idx].all() and a[:, prev].all():
            print(f"   {nm:18s} {np.mean(a[:, idx] - a[:, prev]) / ghz / 1e3:6.2f}")
        prev = idx
print("step total us", (tr[2 * ns - 1][3] - tr[ns][0]) / 1e3)
