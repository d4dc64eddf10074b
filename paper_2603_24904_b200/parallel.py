"""Partitioning of the decode path across GPUs.

* Sequence sharding (C5): independent sequences are dealt to ranks; no
  data-path collective. `sequence_shard`.
* Tensor parallel (C4), Megatron style:
  - column-parallel: wq/wk/wv by heads (rank r owns heads [r*H/g, (r+1)*H/g)),
    w_gate/w_up by FFN rows, the lm_head by vocab rows;
  - row-parallel: wo by the same head columns, w_down by the same FFN columns;
  - after wo and after w_down the PRE-SCALE int64 accumulators are summed
    across ranks (allreduce): `(acc * s) >> 16` is nonlinear, so the sum must
    come first; integer addition is associative, so the result is
    bit-identical at every g (the reference's chunk-invariance argument,
    proj/tests/test_kernels.cpp:79-97);
  - argmax: rank-local (max, lowest index) then a deterministic global pick.
`TPPlan` states these slices for the host-side sharding (`shard_tensors`)
and its gloo tests (tests/test_parallel.py); the device shards are cut by
dimg_model_upload with the same balanced blocks.

`TensorParallel` runs the sharded model on the GPU (dimg_tp_*):
  - "fused-ipc": this process is one rank (one process per GPU); its shard
    runs the persistent decode kernel, and the WO / w_down epilogues store
    their rows' pre-scale partials straight into every peer's inbox over
    NVLink (CUDA IPC peer memory, `connect_group`) and poll their own: the
    all-reduce is fused into the GEMV, no collective call per layer;
  - "fused": the same kernel program for all shards on one device (one
    cooperative launch split between the ranks) -- the one-GPU test of it;
  - "nccl": one process per GPU, per-stage GEMV kernels and an NCCL
    all-reduce of the pre-scale accumulators (the collective-library
    baseline); "local": that chain for all shards on one device.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import ctypes as C

import numpy as np

from ._lib import ModelDesc, check, i64p, lib, ptr, u32p, u64p
from .model import LAYER_TENSORS, ModelConfig, ModelFile


def sequence_shard(n_seqs: int, world: int, rank: int) -> List[int]:
    """Contiguous balanced block of sequence ids for `rank` (C5: 64 over 8)."""
    lo = n_seqs * rank // world
    hi = n_seqs * (rank + 1) // world
    return list(range(lo, hi))


def _block(n: int, parts: int, i: int) -> Tuple[int, int]:
    return n * i // parts, n * (i + 1) // parts


@dataclass(frozen=True)
class TPPlan:
    cfg: ModelConfig
    tp: int
    rank: int

    def __post_init__(self):
        if not (1 <= self.tp and 0 <= self.rank < self.tp):
            raise ValueError("bad tp rank/size")
        if self.cfg.n_heads % self.tp:
            raise ValueError("n_heads must be divisible by the tensor-parallel degree")

    @property
    def heads(self) -> Tuple[int, int]:
        return _block(self.cfg.n_heads, self.tp, self.rank)

    @property
    def head_cols(self) -> Tuple[int, int]:
        """d_model columns (= q/k/v rows) owned: whole heads."""
        h0, h1 = self.heads
        return h0 * self.cfg.d_head, h1 * self.cfg.d_head

    @property
    def ffn(self) -> Tuple[int, int]:
        return _block(self.cfg.d_ffn, self.tp, self.rank)

    @property
    def vocab(self) -> Tuple[int, int]:
        return _block(self.cfg.vocab, self.tp, self.rank)

    def slice_layer(self, name: str, w: np.ndarray, s: np.ndarray):
        """The rank's part of a layer tensor (int8 weights, int64 row scales).
        Column-parallel tensors keep their row scales; row-parallel ones keep
        all rows (scales applied after the allreduce) and a column slice."""
        c0, c1 = self.head_cols
        f0, f1 = self.ffn
        if name in ("wq", "wk", "wv"):
            return w[c0:c1], s[c0:c1]
        if name == "wo":
            return w[:, c0:c1], s
        if name in ("w_gate", "w_up"):
            return w[f0:f1], s[f0:f1]
        if name == "w_down":
            return w[:, f0:f1], s
        raise KeyError(name)

    def slice_head(self, w: np.ndarray, s: np.ndarray):
        v0, v1 = self.vocab
        return w[v0:v1], s[v0:v1]


def shard_tensors(model: ModelFile, plan: TPPlan):
    """Directory-order (weights, scales) of the rank's shard, plus the
    replicated embedding and gains."""
    out = {"tok_embd": model.tensor("tok_embd"), "norms": model.norms()}
    for l in range(model.config.n_layers):
        for t in LAYER_TENSORS:
            out[f"layers.{l}.{t}"] = plan.slice_layer(t, *model.tensor(f"layers.{l}.{t}"))
    out["output"] = plan.slice_head(*model.tensor("output"))
    return out


def pick_argmax(candidates) -> int:
    """Deterministic global argmax from per-rank (value, index) pairs:
    largest value, lowest index on ties (proj/src/engine.cpp:113-120)."""
    best = None
    for v, i in candidates:
        if best is None or v > best[0] or (v == best[0] and i < best[1]):
            best = (v, i)
    return int(best[1])


# "local" / "nccl": per-stage GEMV kernels + collectives (NCCL between
# processes); "fused" / "fused-ipc": the persistent decode kernel on every
# shard with the sums inside it (one device / one process per GPU over CUDA
# IPC peer memory), include/dimg.h dimg_tp_backend.
BACKENDS = {"local": 0, "nccl": 1, "fused": 2, "fused-ipc": 3}


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it; the caller broadcasts it)."""
    b = (C.c_uint8 * 128)()
    check(lib.dimg_nccl_unique_id(b))
    return bytes(b)


class TensorParallel:
    """generate_greedy (proj/src/engine.cpp:31-54) on a model sharded over
    tp_size ranks. Tokens and hashes equal the
    single-GPU engine's at every tp_size."""

    def __init__(self, model: ModelFile, tp_size: int, backend: str = "local", rank: int = 0,
                 nccl_id: bytes = None, device: int = 0, keep_logits_cap: int = 0):
        from .engine import GenerationResult  # noqa: F401  (import cycle)
        model.config.validate()
        d = ModelDesc()
        check(lib.dimg_host_model_desc(model._h, C.byref(d)))
        idb = (C.c_uint8 * 128)(*nccl_id) if nccl_id is not None else None
        h = C.c_void_p()
        check(lib.dimg_tp_create(device, C.byref(d), BACKENDS[backend], rank, tp_size, idb, keep_logits_cap,
                                 C.byref(h)))
        self._h = h
        self._model = model  # the desc's host buffers are borrowed during upload only
        self.tp_size, self.backend, self.rank = tp_size, backend, rank
        self.vocab = model.config.vocab

    def generate_greedy(self, prompt, max_new: int, keep_logits: bool = False):
        from .engine import GenerationResult
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        toks = np.zeros(max(1, max_new), np.uint32)
        h = (C.c_uint8 * 32)()
        logits = np.empty((max_new, self.vocab), np.int64) if keep_logits else None
        check(lib.dimg_tp_generate_greedy(self._h, ptr(p, u32p), p.size, max_new, ptr(toks, u32p), h,
                                          ptr(logits, i64p) if keep_logits else None))
        res = GenerationResult([int(t) for t in toks[:max_new]], bytes(h))
        if keep_logits:
            res.logits = [logits[i] for i in range(max_new)]
        return res

    def time_decode(self, prompt, n_steps: int) -> float:
        """ms of n_steps decode steps (CUDA events on the group's stream)."""
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        ms = C.c_float()
        check(lib.dimg_tp_time_decode(self._h, ptr(p, u32p), p.size, n_steps, C.byref(ms)))
        return ms.value

    def tokens(self, n: int):
        out = np.zeros(max(1, n), np.uint32)
        check(lib.dimg_tp_tokens(self._h, ptr(out, u32p), n))
        return [int(t) for t in out[:n]]

    def exchange_handle(self) -> bytes:
        """fused-ipc: this rank's exchange-block handle (64 bytes)."""
        h = (C.c_uint8 * 64)()
        check(lib.dimg_tp_exchange_handle(self._h, h))
        return bytes(h)

    def connect(self, handles) -> None:
        """fused-ipc: map the peers' exchange blocks (handles in rank order)."""
        if len(handles) != self.tp_size or any(len(h) != 64 for h in handles):
            raise ValueError("connect: one 64-byte handle per rank")
        buf = (C.c_uint8 * (64 * self.tp_size))(*b"".join(handles))
        check(lib.dimg_tp_connect(self._h, buf))

    def connect_group(self, group=None) -> None:
        """fused-ipc: exchange the handles over torch.distributed and connect."""
        import torch.distributed as dist
        hs = [None] * self.tp_size
        dist.all_gather_object(hs, self.exchange_handle(), group=group)
        self.connect(hs)

    def info(self):
        b, n = C.c_uint64(), C.c_uint64()
        check(lib.dimg_tp_info(self._h, C.byref(b), C.byref(n)))
        return {"weight_bytes": b.value, "launches_per_step": n.value}

    def close(self):
        if getattr(self, "_h", None):
            lib.dimg_tp_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
