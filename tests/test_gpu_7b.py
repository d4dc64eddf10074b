"""GPU parity at the headline shape: the Llama-2-7B-shaped toy model
(BASELINE.json north_star).

* smoke7b and C2 goldens come from the REFERENCE engine itself
  (tests/golden/make_golden_7b.py ref -> oracle/_ref); C2's output hash
  is the one BASELINE.md quotes.
* C4 (1024 new tokens) and the C5 sequences come from the C oracle, which
  is pinned bit-for-bit to the reference on C1 and C2 (tests/test_oracle.py).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


@pytest.fixture(scope="module")
def model7b(P, golden_7b):
    g = golden_7b["c2"]
    m = P.gen_toy_model(g["seed"], P.ModelConfig(*g["config"]), device=0)
    assert m.weight_hash == g["weight_hash"]
    return m


def _digest(P, arrs):
    return P.weight_hash(np.ascontiguousarray(np.stack(arrs), np.int64).tobytes())


@pytest.mark.parametrize("name", ["smoke7b", "c2"])
def test_7b_matches_reference_engine(P, golden_7b, model7b, name):
    g = golden_7b[name]
    prompt = P.prompt_from_seed(g["prompt_seed"], g["config"][4], 16)[:g["P"]]
    res = P.generate_greedy(model7b, prompt, g["max_new"], P.EngineOptions(keep_logits=True))
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]
    assert _digest(P, res.logits) == g["logits_digest"]


def test_7b_c4_long_generation(P, golden_7b, model7b):
    g = golden_7b.get("c4")
    if g is None:
        pytest.skip("c4 golden not generated")
    prompt = P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"])
    res = P.generate_greedy(model7b, prompt, g["max_new"])
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]


def test_7b_c5_sequences(P, golden_7b, model7b):
    names = sorted((k for k in golden_7b if k.startswith("c5_")), key=lambda k: int(k[3:]))
    if not names:
        pytest.skip("c5 goldens not generated")
    s = P.InferenceSession(model7b)
    for k in names:
        g = golden_7b[k]
        prompt = P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"])
        res = s.generate_greedy(prompt, g["max_new"])
        assert res.token_ids == g["tokens"], k
        assert res.output_hash.hex() == g["output_hash"], k


@pytest.mark.parametrize("n_seqs", [8, 16])
def test_7b_c5_batch_on_tensor_cores(P, golden_7b, model7b, n_seqs):
    """C5: the sequences generated together (tensor-core batch path; 8 = the
    per-GPU share of C5's 64 on 8 GPUs), each stream and hash identical to the
    oracle's single-sequence goldens."""
    names = sorted((k for k in golden_7b if k.startswith("c5_")), key=lambda k: int(k[3:]))[:n_seqs]
    if not names:
        pytest.skip("c5 goldens not generated")
    gs = [golden_7b[k] for k in names]
    prompts = [P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"]) for g in gs]
    res, path = P.generate_greedy_batch(model7b, prompts, gs[0]["max_new"])
    assert path == "tensor_cores"
    for g, r in zip(gs, res):
        assert r.token_ids == g["tokens"]
        assert r.output_hash.hex() == g["output_hash"]


def test_7b_c3_prefill_on_tensor_cores(P, golden_7b, model7b):
    """C3: a 2048-token prompt prefilled on the tensor cores, then 8 greedy
    tokens; tokens, hash and the kept logits equal the oracle's."""
    g = golden_7b.get("c3")
    if g is None:
        pytest.skip("c3 golden not generated")
    prompt = P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"])
    s = P.InferenceSession(model7b, keep_logits_cap=g["max_new"])
    res = s.generate_greedy(prompt, g["max_new"], keep_logits=True)
    assert s.stats()["tc_prefills"] == 1
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]
    if g.get("logits_digest"):
        assert _digest(P, res.logits) == g["logits_digest"]


def test_7b_c5_sharded_as_on_8_gpus(P, golden_7b, model7b):
    """C5 as the 8-GPU run deals it (parallel.sequence_shard: 8 sequences per
    rank, each rank one batch call; proj/tests/acceptance.cpp:92-127 deals
    prompts to workers the same way): every shard with goldens, every
    per-sequence hash equal to the oracle's single-sequence golden."""
    from paper_2603_24904_b200.parallel import sequence_shard
    have = {int(k[3:]) for k in golden_7b if k.startswith("c5_")}
    if len(have) < 16:
        pytest.skip("c5 goldens not generated")
    checked = 0
    for rank in range(8):
        ids = sequence_shard(64, 8, rank)
        if not set(ids) <= have:
            continue
        gs = [golden_7b[f"c5_{i}"] for i in ids]
        prompts = [P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"]) for g in gs]
        res, path = P.generate_greedy_batch(model7b, prompts, gs[0]["max_new"])
        assert path == "tensor_cores"
        assert [r.output_hash.hex() for r in res] == [g["output_hash"] for g in gs], rank
        checked += len(ids)
    assert checked >= 16
    if len(have) == 64:  # the full C5 set: all 64 sequences, 8 shards
        assert checked == 64
