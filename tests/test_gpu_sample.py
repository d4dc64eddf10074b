"""Seeded sampling on the GPU: generate_sampled /
sample_from_logits (proj/src/engine.cpp:122-163) against the reference's own
outputs (tests/golden/sample.json, sample_ops.npz from
tests/golden/make_sample_golden.py)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(G, "sample.json")))["cases"]


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def test_selection_matches_reference(P):
    z = np.load(os.path.join(G, "sample_ops.npz"))
    for i, (row, n, t, d, tok) in enumerate(zip(z["logits"], z["lens"], z["temperature"], z["draw"], z["token"])):
        assert P.sample_from_logits(row[:n], int(t), int(d)) == int(tok), i


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['config'][4]}v_T{c['temperature']}")
def test_generate_sampled_matches_reference(P, case):
    m = P.gen_toy_model(case["seed"], P.ModelConfig(*case["config"]))
    assert P.sample_key(m.bytes, case["prompt"]).hex() == case["key"]
    r = P.generate_sampled(m, case["prompt"], case["max_new"], case["temperature"])
    assert r.token_ids == case["tokens"]
    assert r.output_hash.hex() == case["output_hash"]


def test_temperature_must_be_positive(P):
    m = P.gen_toy_model(1001, P.ModelConfig(2, 16, 2, 32, 32, 64))
    with pytest.raises(P.InvalidArgument):
        P.generate_sampled(m, [1, 2], 4, 0)
    with pytest.raises(P.InvalidArgument):
        P.sample_from_logits(np.arange(8), -1, 5)


def test_selection_edges_match_reference(P):
    """sample_edge.npz: the reference's own answers at its edges -- scaled
    logits spanning more than 2^63 (exp_neg_lut's std::domain_error,
    q16.cpp:82) and vocabularies above 65536 whose probabilities all
    truncate to 0 (engine.cpp:138 falls through to V - 1)."""
    z = np.load(os.path.join(G, "sample_edge.npz"))
    for i, (row, n, t, d, st, tok) in enumerate(zip(z["logits"], z["lens"], z["temperature"], z["draw"],
                                                     z["status"], z["token"])):
        if st == 6:
            with pytest.raises(P.DomainError):
                P.sample_from_logits(row[:n], int(t), int(d))
        else:
            assert P.sample_from_logits(row[:n], int(t), int(d)) == int(tok), i
