"""Tensor parallelism on the GPU (BASELINE config C4).

The sharded kernels run through dimg_tp on one GPU: the "local" backend
(per-stage kernels for all tp_size shards on cuda:0, the cross-rank sums of
the pre-scale accumulators done by kernels, no kernel waiting on another) and
the "fused" backend (the persistent decode kernel of every shard in ONE
cooperative launch, CTAs split between the ranks, the sums exchanged inside
the WO / w_down epilogues through each rank's inbox -- the program the
"fused-ipc" backend runs with one process per GPU over peer memory). Every generation must equal
the REFERENCE's goldens -- tokens, BLAKE3 output hash and every kept logit
-- at every tensor-parallel degree (proj/src/kernels.cpp:18-50: the int64
accumulator sum is order-free). The NCCL backend's code path (all-reduce,
all-gather) runs here at world size 1.
"""
import numpy as np
import pytest

from test_gpu_parity import SMALL, _digest, _model_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def _degrees(H):
    return [g for g in (1, 2, 3, 4, 8) if H % g == 0]


BACKENDS = ["local", "fused"]


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("name", [n for n in SMALL if n not in ("micro_s9", "micro_s123456789")])
def test_tp_generation_matches_reference(P, golden_models, name, backend):
    g = golden_models[name]
    m = _model_for(P, g)
    for deg in _degrees(g["config"][2]):
        tp = P.TensorParallel(m, deg, backend=backend, keep_logits_cap=g["max_new"])
        res = tp.generate_greedy(g["prompt"], g["max_new"], keep_logits=True)
        assert res.token_ids == g["tokens"], deg
        assert res.output_hash.hex() == g["output_hash"], deg
        assert _digest(P, res.logits) == g["logits_digest"], deg
        # a second generation on the same group (graphs replayed, caches reused)
        assert tp.generate_greedy(g["prompt"], g["max_new"]).token_ids == g["tokens"], deg
        tp.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_tp_wild_model_takes_the_wide_path(P, golden_models, backend):
    """wild_b's activations need the 8-limb GEMV path on every shard."""
    g = golden_models["wild_b"]
    m = _model_for(P, g)
    for deg in (2, 4, 8):
        res = P.TensorParallel(m, deg, backend=backend).generate_greedy(g["prompt"], g["max_new"])
        assert res.output_hash.hex() == g["output_hash"], deg


@pytest.mark.parametrize("backend", BACKENDS)
def test_tp_uneven_ffn_and_vocab_splits(P, oracle, backend):
    """d_ffn and vocab not divisible by the degree (balanced blocks)."""
    from oracle.pyoracle import Config
    cfg6 = (2, 96, 6, 101, 77, 64)
    m = P.gen_toy_model(5, P.ModelConfig(*cfg6))
    om = oracle.gen_toy(5, Config(*cfg6))
    prompt = P.prompt_from_seed(6, cfg6[4], 9)
    toks, h, lg = oracle.generate_greedy(om, prompt, 7, keep_logits=True)
    for deg in (2, 3, 6):
        res = P.TensorParallel(m, deg, backend=backend, keep_logits_cap=7).generate_greedy(prompt, 7, keep_logits=True)
        assert res.token_ids == [int(t) for t in toks] and res.output_hash.hex() == h, deg
        assert np.array_equal(np.stack(res.logits), lg), deg


def test_tp_nccl_backend_world_one(P, golden_models):
    """The NCCL code path (ncclAllReduce / ncclAllGather in the captured step)
    with one rank."""
    g = golden_models["medium"]
    m = _model_for(P, g)
    tp = P.TensorParallel(m, 1, backend="nccl", rank=0, nccl_id=P.nccl_unique_id(), keep_logits_cap=g["max_new"])
    res = tp.generate_greedy(g["prompt"], g["max_new"], keep_logits=True)
    assert res.output_hash.hex() == g["output_hash"]
    assert _digest(P, res.logits) == g["logits_digest"]
    tp.close()


def test_tp_fused_repeat_and_timing(P, golden_models):
    """The fused group 100x on one group (tags keep advancing across
    launches, inboxes are reused), then the timed-decode entry point."""
    g = golden_models["medium"]
    m = _model_for(P, g)
    tp = P.TensorParallel(m, 2, backend="fused")
    for _ in range(100):
        assert tp.generate_greedy(g["prompt"], g["max_new"]).output_hash.hex() == g["output_hash"]
    ms = tp.time_decode(g["prompt"], g["max_new"])
    assert ms > 0 and tp.tokens(g["max_new"]) == g["tokens"]
    assert tp.info()["launches_per_step"] == 1
    tp.close()


def test_tp_fused_ipc_world_one(P, golden_models):
    """The one-process-per-GPU fused backend's API at world size 1 (nothing
    to map: the group is connected at creation)."""
    g = golden_models["medium"]
    m = _model_for(P, g)
    tp = P.TensorParallel(m, 1, backend="fused-ipc", rank=0)
    assert len(tp.exchange_handle()) == 64
    with pytest.raises(P.LogicError):
        tp.connect([tp.exchange_handle()])  # already connected
    assert tp.generate_greedy(g["prompt"], g["max_new"]).output_hash.hex() == g["output_hash"]
    with pytest.raises(P.InvalidArgument):
        tp.generate_greedy(g["prompt"], 2, keep_logits=True)  # each process holds only its vocab slice
    tp.close()
    # a two-rank group is not usable before connect
    tp2 = P.TensorParallel(m, 2, backend="fused-ipc", rank=0)
    with pytest.raises(P.LogicError):
        tp2.generate_greedy(g["prompt"], 2)
    tp2.close()


def test_tp_errors(P):
    m = P.gen_toy_model(1, P.ModelConfig(2, 16, 2, 32, 32, 64))
    with pytest.raises(P.InvalidArgument):
        P.TensorParallel(m, 3)  # does not divide n_heads
    tp = P.TensorParallel(m, 2)
    with pytest.raises(P.InvalidArgument):
        tp.generate_greedy([], 3)
    with pytest.raises(P.OutOfRange):
        tp.generate_greedy([1, 40], 3)
    with pytest.raises(P.ContextOverflow):
        tp.generate_greedy([1, 2], 63)
    assert tp.generate_greedy([1, 2], 4).token_ids == P.generate_greedy(m, [1, 2], 4).token_ids


# ---- the 7B shape: C2 (reference golden) and C4 (1024 tokens) at 2 / 4 / 8 ----

@pytest.fixture(scope="module")
def model7b(P, golden_7b):
    g = golden_7b["c2"]
    m = P.gen_toy_model(g["seed"], P.ModelConfig(*g["config"]), device=0)
    assert m.weight_hash == g["weight_hash"]
    return m


@pytest.mark.slow
@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("deg", [2, 4, 8])
def test_tp_7b_c2_and_c4(P, golden_7b, model7b, deg, backend):
    tp = P.TensorParallel(model7b, deg, backend=backend, keep_logits_cap=128)
    g = golden_7b["c2"]
    prompt = P.prompt_from_seed(g["prompt_seed"], g["config"][4], g["P"])
    res = tp.generate_greedy(prompt, g["max_new"], keep_logits=True)
    assert res.token_ids == g["tokens"]
    assert res.output_hash.hex() == g["output_hash"]
    assert _digest(P, res.logits) == g["logits_digest"]
    g4 = golden_7b.get("c4")
    if g4 is not None:
        prompt = P.prompt_from_seed(g4["prompt_seed"], g4["config"][4], g4["P"])
        res = tp.generate_greedy(prompt, g4["max_new"])
        assert res.token_ids == g4["tokens"]
        assert res.output_hash.hex() == g4["output_hash"]
    tp.close()
