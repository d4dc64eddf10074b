"""Fused tensor-parallel decode on one GPU (the DIMG_TP_FUSED_LOCAL group):
ms per token at g = 1, 2, 4, 8 against the single-GPU session, tokens checked
against the C2 golden. The g ranks share one GPU's HBM and SMs here, so this
measures the in-kernel exchange's overhead, not multi-GPU scaling.

    python tools/tp_fused_probe.py [steps]
    DIMG_TP_SOLO=1 python tools/tp_fused_probe.py --solo [steps]

--solo: one fused-ipc rank of g = 2, 4, 8 alone on the whole GPU with the
exchange switched off (DIMG_TP_SOLO): the per-GPU time of a g-way shard
without the NVLink latency of the sums -- an estimate of the multi-GPU
per-token time's compute part (tokens are NOT valid in this mode).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_2603_24904_b200 as P  # noqa: E402

solo = "--solo" in sys.argv
argv = [a for a in sys.argv[1:] if a != "--solo"]
steps = int(argv[0]) if argv else 128
g2 = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "models_7b.json")))["c2"]
cfg = P.ModelConfig(*g2["config"])
m = P.gen_toy_model(g2["seed"], cfg, device=0)
prompt = P.prompt_from_seed(g2["prompt_seed"], cfg.vocab, g2["P"])
s = P.InferenceSession(m)
s.begin(prompt, steps)
s.prefill()
s.sync()
ms = s.time_decode(steps)
print(f"single session: {ms / steps * 1e3:.1f} us/token, tokens ok {s.tokens(steps) == g2['tokens'][:steps]}")
if solo:
    assert os.environ.get("DIMG_TP_SOLO") == "1"
    for g in (2, 4, 8):
        tp = P.TensorParallel(m, g, backend="fused-ipc", rank=0)
        tp.time_decode(prompt, 8)
        ms = min(tp.time_decode(prompt, steps) for _ in range(3))
        print(f"solo rank 0 of g={g} (no exchange, whole GPU): {ms / steps * 1e3:7.1f} us/token", flush=True)
        tp.close()
    sys.exit(0)
for backend in ("fused", "local"):
    for g in (1, 2, 4, 8):
        t0 = time.time()
        tp = P.TensorParallel(m, g, backend=backend)
        t1 = time.time()
        tp.time_decode(prompt, 8)
        ms = min(tp.time_decode(prompt, steps) for _ in range(2))
        ok = tp.tokens(steps) == g2["tokens"][:steps]
        print(f"{backend:5s} g={g}: {ms / steps * 1e3:7.1f} us/token  tokens ok {ok}  (create {t1 - t0:.1f} s)", flush=True)
        tp.close()
