import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import numpy as np
import paper_2603_24904_b200 as P
from oracle.pyoracle import Config, Oracle
orc = Oracle()
for c6, seed, P_len in (((2, 256, 2, 512, 512, 512), 5, 300), ((1, 512, 4, 256, 300, 1024), 6, 700), ((2, 128, 1, 256, 64, 256), 8, 130)):
    cfg = P.ModelConfig(*c6)
    m = P.gen_toy_model(seed, cfg)
    om = orc.gen_toy(seed, Config(*c6))
    prompt = P.prompt_from_seed(seed + 1, cfg.vocab, P_len)
    for pv in ("1", "0"):
        os.environ["DIMG_PF_PV"] = pv
        s = P.InferenceSession(m, keep_logits_cap=4)
        res = s.generate_greedy(prompt, 4, keep_logits=True)
        st = s.stats()
        toks, h, lg = orc.generate_greedy(om, prompt, 4, keep_logits=True)
        print(c6, "pv", pv, "tokens ok", res.token_ids == [int(t) for t in toks], "logits ok",
              bool(np.array_equal(np.stack(res.logits), lg)), "tc_prefills", st["tc_prefills"], "fallbacks", st["tc_fallbacks"], flush=True)
