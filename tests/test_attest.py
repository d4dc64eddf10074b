"""Attestation wire format and texts (proj/src/attest.cpp:31-87) against the
reference's own output (tests/golden/attest.json, made by
tests/golden/make_attest_golden.py from the compiled reference). Host-only:
no GPU needed."""
import json
import os

import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "attest.json")))


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def test_wire_round_trip_matches_reference(P):
    wire = bytes.fromhex(GOLD["wire"])
    a = P.Attestation.decode(wire)
    assert a.encode() == wire
    assert a.bond == GOLD["bond"] and a.challenge_period == GOLD["challenge_period"]
    assert a.input_hash == P.prompt_hash(GOLD["prompt"])
    assert a.to_text() == GOLD["text"]


@pytest.mark.parametrize("n", [0, 1, 111, 113, 224])
def test_decode_rejects_bad_sizes(P, n):
    with pytest.raises(P.ParseError) as e:
        P.Attestation.decode(bytes(n))
    assert e.value.kind == "truncated"


def test_outcome_texts_match_reference(P):
    wire = bytes.fromhex(GOLD["wire"])
    a = P.Attestation.decode(wire)
    assert P.VerifyOutcome(True).to_text() == GOLD["verify"]["honest"]
    bad = bytearray(a.output_hash)
    bad[7] ^= 0x20
    o = P.VerifyOutcome(False, "output", bytes(bad), a.output_hash)
    assert o.to_text() == GOLD["verify"]["tampered_output"]
