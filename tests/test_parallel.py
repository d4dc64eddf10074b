"""Multi-rank host logic on CPU (gloo, world size 2).

A tensor-parallel greedy generation: each rank computes its shard of every
layer with the C oracle's operators, the pre-scale int64 accumulators of wo
and w_down are summed with a real gloo allreduce, and the argmax is picked
from gathered (value, index) pairs. The tokens, output hash and every
logit must equal the UNSHARDED reference goldens bit for bit -- the
exactness argument the device tensor-parallel path rests on."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_sequence_shard():
    from paper_2603_24904_b200.parallel import sequence_shard
    parts = [sequence_shard(64, 8, r) for r in range(8)]
    assert sum(parts, []) == list(range(64))
    assert all(len(p) == 8 for p in parts)
    parts = [sequence_shard(10, 4, r) for r in range(4)]
    assert sum(parts, []) == list(range(10))


def test_tp_plan_slices_cover_the_model():
    from paper_2603_24904_b200 import ModelConfig
    from paper_2603_24904_b200.parallel import TPPlan
    cfg = ModelConfig(2, 16, 4, 37, 33, 64)
    for tp in (1, 2, 4):
        plans = [TPPlan(cfg, tp, r) for r in range(tp)]
        assert [p.heads for p in plans][0][0] == 0 and plans[-1].heads[1] == 4
        assert sum(p.ffn[1] - p.ffn[0] for p in plans) == 37
        assert sum(p.vocab[1] - p.vocab[0] for p in plans) == 33
    with pytest.raises(ValueError):
        TPPlan(cfg, 3, 0)


def _scale(acc, s):
    # (int128(acc) * s) >> 16 truncated to int64 (proj/src/kernels.cpp:27)
    v = (int(acc) * int(s)) >> 16
    return np.int64(((v + (1 << 63)) % (1 << 64)) - (1 << 63))


def _tp_worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json
        import sys
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import ctypes as C

        import paper_2603_24904_b200 as P
        from oracle.pyoracle import Oracle, _ptr, i64p
        from paper_2603_24904_b200.parallel import TPPlan, pick_argmax, shard_tensors

        g = json.load(open(os.path.join(ROOT, "tests", "golden", "models.json")))[name]
        cfg = P.ModelConfig(*g["config"])
        mf = P.gen_toy_model(g["seed"], cfg)
        plan = TPPlan(cfg, world, rank)
        sh = shard_tensors(mf, plan)
        orc = Oracle()
        L, D, dh = cfg.n_layers, cfg.d_model, cfg.d_head
        h0, h1 = plan.heads
        Hl = h1 - h0
        c0, c1 = plan.head_cols
        norms = sh["norms"].reshape(2 * L + 1, D)
        kc = [np.zeros((cfg.max_ctx, Hl * dh), np.int64) for _ in range(L)]
        vc = [np.zeros((cfg.max_ctx, Hl * dh), np.int64) for _ in range(L)]
        rc, rs = orc.rope_tables(cfg.rope_theta, dh, cfg.max_ctx)
        E, Es = sh["tok_embd"]

        def allreduce(v):
            t = torch.from_numpy(np.ascontiguousarray(v, np.int64))
            dist.all_reduce(t)  # int64 sum: wraps like the reference's accumulator
            return t.numpy()

        def forward(tok, pos):
            x = (E[tok].astype(np.int64) * Es[tok]).astype(np.int64)  # embed_token
            for l in range(L):
                xn = orc.rmsnorm(x, norms[2 * l])
                q = orc.dense(*sh[f"layers.{l}.wq"], xn)
                k = orc.dense(*sh[f"layers.{l}.wk"], xn)
                v = orc.dense(*sh[f"layers.{l}.wv"], xn)
                att = np.empty(Hl * dh, np.int64)
                orc.lib.orc_attention_step(_ptr(q, i64p), _ptr(k, i64p), _ptr(v, i64p), C.c_uint32(Hl),
                                           C.c_uint32(dh), C.c_uint32(cfg.max_ctx), _ptr(kc[l], i64p),
                                           _ptr(vc[l], i64p), C.c_uint32(pos), _ptr(rc, i64p), _ptr(rs, i64p),
                                           _ptr(att, i64p))
                wo, so = sh[f"layers.{l}.wo"]
                acc = allreduce(wo.astype(np.int64) @ att)  # pre-scale partial sums
                x = np.clip(x + np.array([_scale(a, s) for a, s in zip(acc, so)], np.int64),
                            -(256 << 16), 256 << 16)
                xf = orc.rmsnorm(x, norms[2 * l + 1])
                gate = orc.dense(*sh[f"layers.{l}.w_gate"], xf)
                up = orc.dense(*sh[f"layers.{l}.w_up"], xf)
                hh = np.array([orc.lib.orc_q16_mul(orc.lib.orc_silu(int(a)), int(b)) for a, b in zip(gate, up)],
                              np.int64)
                wd, sd = sh[f"layers.{l}.w_down"]
                acc = allreduce(wd.astype(np.int64) @ hh)
                x = np.clip(x + np.array([_scale(a, s) for a, s in zip(acc, sd)], np.int64),
                            -(256 << 16), 256 << 16)
            xo = orc.rmsnorm(x, norms[2 * L])
            local = orc.dense(*sh["output"], xo)  # this rank's vocab slice
            return local

        v0, v1 = plan.vocab
        prompt, N = g["prompt"], g["max_new"]
        toks, kept, pos = [], [], 0
        for i, t in enumerate(prompt):
            local = forward(t, pos)
            pos += 1
        for n in range(N):
            lb = int(np.argmax(local))  # first maximum = lowest index
            cands = [None] * world
            dist.all_gather_object(cands, (int(local[lb]), v0 + lb))
            full = [None] * world
            dist.all_gather_object(full, local.tolist())
            kept.append(sum(full, []))
            nxt = pick_argmax(cands)
            toks.append(nxt)
            if n + 1 == N:
                break
            local = forward(nxt, pos)
            pos += 1
        if rank == 0:
            q.put((toks, P.hash_token_ids(toks).hex(),
                   P.weight_hash(np.array(kept, np.int64).tobytes())))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["small_s7", "accept_102"])
def test_tensor_parallel_generation_is_bit_exact(golden_models, name):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_tp_worker, args=(2, _free_port(), name, q), nprocs=2, join=True,
                       start_method="spawn")
    toks, h, logits_digest = q.get(timeout=60)
    g = golden_models[name]
    assert toks == g["tokens"]
    assert h == g["output_hash"]
    assert logits_digest == g["logits_digest"]
