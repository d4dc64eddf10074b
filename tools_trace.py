"""Per-stage phase breakdown of the persistent decode kernel (CTA 0 stamps)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
s = P.InferenceSession(m)
prompt = P.prompt_from_seed(8, cfg.vocab, 16)
s.begin(prompt, 64)
s.prefill()
s.decode(4)
ns = 5 * cfg.n_layers + 1
tr = s.trace(2, 2 * ns).astype(np.int64)
names = ["qkv", "attn", "wo", "gu", "down"]
rows = {}
sub = {}
for i in range(ns, 2 * ns):
    k = i - ns
    name = "head" if k == ns - 1 else names[k % 5]
    t = tr[i]
    nxt = tr[i + 1][0] if i + 1 < 2 * ns else t[3]
    rows.setdefault(name, []).append((t[1] - t[0] if t[1] else 0, t[2] - t[1] if t[2] else 0,
                                      t[3] - (t[2] if t[2] else t[0]), nxt - t[3]))
    if t[4]:
        c = t[8]
        ghz = 1.965e-3  # cycles per ns at max clock (approximate)
        sub.setdefault(name, []).append(((t[4] - c) / ghz, (t[5] - t[4]) / ghz, (t[6] - t[5]) / ghz,
                                         (t[7] - t[6]) / ghz, 0))
print(os.environ.get("DIMG_L2_AHEAD", "0"), os.environ.get("DIMG_BAR_MODE", "0"),
      "stage   prologue  chunks  epilogue  barrier   | copy  reduce  r  norm  pack (us) [attn: rope scores softmax pv tail]")
for k, v in rows.items():
    a = np.array(v).mean(0) / 1e3
    extra = ""
    if k in sub:
        b = np.array(sub[k]).mean(0) / 1e3
        extra = "  | " + " ".join(f"{x:5.2f}" for x in b)
    print(f"{k:6s} {a[0]:9.2f} {a[1]:7.2f} {a[2]:9.2f} {a[3]:8.2f}{extra}")
print("step total us", (tr[2 * ns - 1][3] - tr[ns][0]) / 1e3)
