"""Attest / verify / dispute on the GPU engine, case for case as the
reference's proj/tests/test_attest.cpp (same fixture), with the attestation
bytes and verdict texts equal to the reference's (tests/golden/attest.json)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "attest.json")))


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


@pytest.fixture(scope="module")
def fx(P):
    m = P.gen_toy_model(GOLD["seed"], P.ModelConfig(*GOLD["config"]))
    prompt = GOLD["prompt"]
    res = P.generate_greedy(m, prompt, GOLD["max_new"])
    att = P.make_attestation(m.bytes, prompt, res, GOLD["bond"], GOLD["challenge_period"])
    return m, prompt, res, att


def test_construction_matches_reference(P, fx):
    m, prompt, res, att = fx
    assert att.encode().hex() == GOLD["wire"]
    assert att.to_text() == GOLD["text"]
    assert att.model_id.hex() == m.weight_hash
    assert att == P.make_attestation(m.bytes, prompt, res, GOLD["bond"], GOLD["challenge_period"])
    other = [4, 8, 16]
    o = P.make_attestation(m.bytes, other, P.generate_greedy(m, other, GOLD["max_new"]), 1, 2)
    assert o.input_hash != att.input_hash


def test_honest_confirmed_with_one_reexecution(P, fx):
    m, prompt, _, att = fx
    before = P.generation_counter()
    out = P.verify_by_reexecution(att, m.bytes, prompt, GOLD["max_new"])
    assert out.confirmed and out.to_text() == GOLD["verify"]["honest"]
    assert P.generation_counter() == before + 1


def test_tampered_output_refuted_at_output(P, fx):
    m, prompt, res, att = fx
    bad = bytearray(att.output_hash)
    bad[7] ^= 0x20
    a = P.Attestation(att.model_id, att.input_hash, bytes(bad), att.bond, att.challenge_period)
    out = P.verify_by_reexecution(a, m.bytes, prompt, GOLD["max_new"])
    assert not out.confirmed and out.refuted_stage == "output"
    assert out.expected == bytes(bad) and out.found == res.output_hash
    assert out.to_text() == GOLD["verify"]["tampered_output"]


def test_wrong_model_refuted_before_inference(P, fx):
    _, prompt, _, att = fx
    other = P.gen_toy_model(2002, P.ModelConfig(*GOLD["config"]))
    before = P.generation_counter()
    out = P.verify_by_reexecution(att, other.bytes, prompt, GOLD["max_new"])
    assert not out.confirmed and out.refuted_stage == "model"
    assert P.generation_counter() == before


def test_tampered_prompt_refuted_at_input(P, fx):
    m, _, _, att = fx
    before = P.generation_counter()
    out = P.verify_by_reexecution(att, m.bytes, [4, 9, 15], GOLD["max_new"])
    assert not out.confirmed and out.refuted_stage == "input"
    assert out.to_text() == GOLD["verify"]["tampered_prompt"]
    assert P.generation_counter() == before


def test_single_bit_model_tampering_refuted_at_model(P, fx):
    m, prompt, _, att = fx
    rng = np.random.default_rng(71)
    base = np.frombuffer(m.bytes, np.uint8)
    for _ in range(20):
        b = base.copy()
        bit = int(rng.integers(0, b.size * 8))
        b[bit // 8] ^= np.uint8(1 << (bit % 8))
        out = P.verify_by_reexecution(att, b, prompt, GOLD["max_new"])
        assert not out.confirmed and out.refuted_stage == "model"


def test_unparseable_model_bytes_raise(P, fx):
    _, prompt, _, att = fx
    garbage = bytes([1, 2, 3, 4, 5])
    a = P.Attestation(P.blake3_gpu(garbage), att.input_hash, att.output_hash, att.bond, att.challenge_period)
    with pytest.raises(P.ParseError):
        P.verify_by_reexecution(a, garbage, prompt, GOLD["max_new"])


def test_dispute_game_outcomes(P, fx):
    m, prompt, _, att = fx
    assert P.dispute_game(att, m.bytes, prompt, GOLD["max_new"]).winner == "attester"
    fab = bytearray(att.output_hash)
    fab[0] ^= 1
    cheat = P.dispute_game(P.Attestation(att.model_id, att.input_hash, bytes(fab), att.bond, att.challenge_period),
                           m.bytes, prompt, GOLD["max_new"])
    assert cheat.winner == "challenger" and cheat.outcome.refuted_stage == "output"
    wm = bytearray(att.model_id)
    wm[0] ^= 1
    bound = P.dispute_game(P.Attestation(bytes(wm), att.input_hash, att.output_hash, att.bond, att.challenge_period),
                           m.bytes, prompt, GOLD["max_new"])
    assert bound.winner == "challenger" and bound.outcome.refuted_stage == "model"
    assert bound.outcome.to_text() == GOLD["verify"]["wrong_model"]
