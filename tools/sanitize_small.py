"""Small invocations of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck); each result is checked
against the C oracle so a sanitizer run is also a parity run.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py [what...]

what: dense_tokens prefill batch decode sample tp (default: all)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2603_24904_b200 as P  # noqa: E402
from oracle.pyoracle import Config, Oracle  # noqa: E402

orc = Oracle()
what = sys.argv[1:] or ["dense_tokens", "prefill", "batch", "decode", "sample", "tp"]
cfg6 = (2, 128, 2, 256, 100, 96)
m = P.gen_toy_model(21, P.ModelConfig(*cfg6))
om = orc.gen_toy(21, Config(*cfg6))


def want(prompt, n):
    return [int(t) for t in orc.generate_greedy(om, prompt, n)[0]]


if "dense_tokens" in what:
    rng = np.random.default_rng(1)
    for N, K, T in ((100, 300, 7), (33, 17, 1), (130, 4095, 65)):
        w = rng.integers(-127, 128, (N, K), dtype=np.int8)
        s = rng.integers(1, 1 << 12, N, dtype=np.int64)
        x = rng.integers(-0x808080, 0x7F7F80, (T, K), dtype=np.int64)
        got = P.dense_tokens(w, s, x)
        for t in range(T):
            assert np.array_equal(got[t], orc.dense(w, s, x[t])), (N, K, T, t)
    print("dense_tokens ok", flush=True)
if "prefill" in what:
    os.environ["DIMG_PREFILL"] = "1"
    for plen in (6, 40):
        p = P.prompt_from_seed(7 + plen, cfg6[4], plen)
        assert P.generate_greedy(m, p, 4).token_ids == want(p, 4), plen
    os.environ.pop("DIMG_PREFILL")
    print("prefill ok", flush=True)
if "batch" in what:
    prompts = [P.prompt_from_seed(900 + i, cfg6[4], 4 + i % 3) for i in range(5)]
    res, path = P.generate_greedy_batch(m, prompts, 4)
    assert path == "tensor_cores"
    assert [r.token_ids for r in res] == [want(p, 4) for p in prompts]
    print("batch ok", flush=True)
if "decode" in what:
    os.environ["DIMG_PREFILL"] = "2"
    p = P.prompt_from_seed(5, cfg6[4], 5)
    assert P.generate_greedy(m, p, 6).token_ids == want(p, 6)
    os.environ.pop("DIMG_PREFILL")
    print("decode ok", flush=True)
if "sample" in what:
    z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "sample_ops.npz"))
    for row, n, t, d, tok in list(zip(z["logits"], z["lens"], z["temperature"], z["draw"], z["token"]))[:10]:
        assert P.sample_from_logits(row[:n], int(t), int(d)) == int(tok)
    print("sample ok", flush=True)
if "tp" in what and hasattr(P, "TensorParallel"):
    p = P.prompt_from_seed(3, cfg6[4], 5)
    tp = P.TensorParallel(m, 2, backend="local")
    assert tp.generate_greedy(p, 4).token_ids == want(p, 4)
    tp.close()
    print("tp ok", flush=True)
print("sanitize_small done")
