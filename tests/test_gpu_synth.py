"""Toy-model synthesis on the GPU: gen_toy_model's ChaCha20
weight stream generated on the device gives the same container bytes as the
host generator, and the weight hashes the reference produced
(tests/golden/models.json, models_7b.json)."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def test_matches_reference_weight_hashes(P):
    gold = json.load(open(os.path.join(G, "models.json")))
    n = 0
    for name, g in gold.items():
        if g.get("kind", "toy") != "toy":
            continue
        cfg = P.ModelConfig(*g["config"], rope_theta=g.get("rope_theta", 10000.0))
        m = P.gen_toy_model(g["seed"], cfg, device=0)
        assert m.weight_hash == g["weight_hash"], name
        n += 1
    assert n >= 5


@pytest.mark.parametrize("seed,cfg6", [(1, (1, 8, 1, 8, 8, 8)), (77, (3, 96, 3, 160, 77, 200)),
                                       (5, (2, 256, 4, 700, 1000, 64))])
def test_same_bytes_as_host(P, seed, cfg6):
    cfg = P.ModelConfig(*cfg6)
    assert bytes(P.gen_toy_model(seed, cfg, device=0).bytes) == bytes(P.gen_toy_model(seed, cfg).bytes)


def test_7b_weight_hash(P):
    g = json.load(open(os.path.join(G, "models_7b.json")))["c2"]
    m = P.gen_toy_model(g["seed"], P.ModelConfig(*g["config"]), device=0)
    assert m.weight_hash == g["weight_hash"]
