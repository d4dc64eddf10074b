import sys
sys.path.insert(0, ".")
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(2, 16, 2, 32, 32, 64)
m = P.gen_toy_model(7, cfg)
for n in (4, 8, 12):
    try:
        r = P.generate_greedy(m, [3, 1, 4], n)
        print("gen", n, r.output_hash.hex()[:16])
    except Exception as e:
        print("gen", n, "ERR", e)
s = P.InferenceSession(m)
for args in ((99, 0), (1, 5), (1, 0), (2, 1)):
    try:
        s.forward(*args)
        print("fwd", args, "ok")
    except Exception as e:
        print("fwd", args, type(e).__name__, e)
