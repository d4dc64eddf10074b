"""The reference's engine API (proj/include/dim/engine.hpp) over the B200 C ABI.

Same names, argument meaning and error behaviour as dim::InferenceSession,
dim::generate_greedy, dim::hash_token_ids and dim::select_greedy, so the
reference's tests (proj/tests/test_engine.cpp) read the same against it.
Every forward pass runs on the GPU through libdimg.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import errors
from ._lib import QTensor, check, i8p, i64p, lib, ptr, u8p, u32p, u64p
from .model import ModelFile

def generation_counter() -> int:
    """Count of generation runs in this process (engine.cpp:165-168): kept by
    the library (dimg_generate_greedy, the batch call, re-execution)."""
    n = C.c_uint64()
    check(lib.dimg_generation_counter(C.byref(n)))
    return n.value


@dataclass
class EngineOptions:
    """EngineOptions (engine.hpp:20-24). `threads` and `chunk` select the
    reference's head-thread pool and chunked matvec; integer sums make both
    invisible in the output, so the GPU path accepts and ignores them."""

    threads: int = 1
    chunk: int = 0
    keep_logits: bool = False
    device: int = 0


@dataclass
class GenerationResult:
    token_ids: List[int]
    output_hash: bytes
    logits: List[np.ndarray] = field(default_factory=list)

    @property
    def output_hash_hex(self) -> str:
        return self.output_hash.hex()


def hash_token_ids(ids: Sequence[int]) -> bytes:
    """BLAKE3 over u32-LE ids (engine.cpp:104-111)."""
    a = np.ascontiguousarray(ids, dtype=np.uint32)
    out = (C.c_uint8 * 32)()
    check(lib.dimg_hash_token_ids(ptr(a, u32p), a.size, out))
    return bytes(out)


def select_greedy(logits) -> int:
    """Argmax, lowest index on ties (engine.cpp:113-120)."""
    a = np.ascontiguousarray(logits, dtype=np.int64)
    out = C.c_uint32()
    check(lib.dimg_select_greedy(ptr(a, i64p), a.size, C.byref(out)))
    return out.value


def parse_prompt(prompt_csv: str = "", bytes_str: str = "") -> List[int]:
    """parse_prompt (proj/tools/dim_cli.cpp:56-70)."""
    cap = max(16, len(prompt_csv) + len(bytes_str.encode()) + 1)
    out = np.zeros(cap, np.uint32)
    n = C.c_size_t()
    check(lib.dimg_parse_prompt(prompt_csv.encode(), bytes_str.encode() if bytes_str else None,
                                ptr(out, u32p), cap, C.byref(n)))
    return [int(v) for v in out[:n.value]]


def prompt_from_seed(seed: int, vocab: int, n: int) -> List[int]:
    out = np.zeros(max(1, n), np.uint32)
    check(lib.dimg_prompt_from_seed(C.c_uint64(seed), vocab, n, ptr(out, u32p)))
    return [int(v) for v in out[:n]]


def build_rope_tables(theta: float, d_head: int, max_ctx: int):
    """RopeTables cos/sin [max_ctx][d_head/2] (proj/src/rope.cpp:17-39)."""
    c = np.empty(max_ctx * (d_head // 2), np.int64)
    s = np.empty_like(c)
    check(lib.dimg_rope_tables(theta, d_head, max_ctx, ptr(c, i64p), ptr(s, i64p)))
    return c, s


class RopeTables:
    """RopeTables (proj/include/dim/rope.hpp:15-26): Q16 cos/sin
    [max_ctx][half_dim]. Unpacks as (cos_raw, sin_raw), the form
    InferenceSession's imported_tables takes."""

    def __init__(self, max_ctx: int, half_dim: int, theta_base: float, cos_raw, sin_raw):
        self.max_ctx, self.half_dim, self.theta_base = int(max_ctx), int(half_dim), float(theta_base)
        self.cos_raw = np.ascontiguousarray(cos_raw, np.int64).reshape(-1)
        self.sin_raw = np.ascontiguousarray(sin_raw, np.int64).reshape(-1)

    @classmethod
    def build(cls, theta: float, d_head: int, max_ctx: int) -> "RopeTables":
        c, s = build_rope_tables(theta, d_head, max_ctx)
        return cls(max_ctx, d_head // 2, theta, c, s)

    def __iter__(self):
        return iter((self.cos_raw, self.sin_raw))

    def __eq__(self, o):
        return (isinstance(o, RopeTables) and (self.max_ctx, self.half_dim) == (o.max_ctx, o.half_dim)
                and np.float64(self.theta_base).tobytes() == np.float64(o.theta_base).tobytes()
                and np.array_equal(self.cos_raw, o.cos_raw) and np.array_equal(self.sin_raw, o.sin_raw))


def serialize_rope_tables(t: RopeTables) -> bytes:
    """The RTAB artifact (proj/src/rope.cpp:41-51), byte-exact."""
    n = C.c_size_t()
    check(lib.dimg_rtab_serialize(t.theta_base, t.max_ctx, t.half_dim, ptr(t.cos_raw, i64p),
                                  ptr(t.sin_raw, i64p), None, 0, C.byref(n)))
    out = np.empty(n.value, np.uint8)
    check(lib.dimg_rtab_serialize(t.theta_base, t.max_ctx, t.half_dim, ptr(t.cos_raw, i64p),
                                  ptr(t.sin_raw, i64p), ptr(out, u8p), out.size, C.byref(n)))
    return out.tobytes()


def deserialize_rope_tables(data: bytes) -> RopeTables:
    """deserialize_rope_tables (proj/src/rope.cpp:53-78): ParseError with the
    reference's kind on bad magic / version, truncation, empty dims or
    trailing bytes."""
    b = np.frombuffer(bytes(data), np.uint8).copy()
    if b.size == 0:
        b = np.zeros(1, np.uint8)[:0]
    mc, hd, th = C.c_uint32(), C.c_uint32(), C.c_double()
    bp = ptr(b, u8p) if b.size else None
    check(lib.dimg_rtab_deserialize(bp, b.size, C.byref(mc), C.byref(hd), C.byref(th), None, None, 0))
    cells = mc.value * hd.value
    c = np.empty(cells, np.int64)
    s = np.empty(cells, np.int64)
    check(lib.dimg_rtab_deserialize(bp, b.size, C.byref(mc), C.byref(hd), C.byref(th), ptr(c, i64p),
                                    ptr(s, i64p), cells))
    return RopeTables(mc.value, hd.value, th.value, c, s)


def save_rope_tables(t: RopeTables, path: str) -> None:
    """save_rope_tables (proj/src/rope.cpp:80-86); IOFailure if unwritable."""
    check(lib.dimg_rtab_save(path.encode(), t.theta_base, t.max_ctx, t.half_dim, ptr(t.cos_raw, i64p),
                             ptr(t.sin_raw, i64p)))


def load_rope_tables(path: str) -> RopeTables:
    """load_rope_tables (proj/src/rope.cpp:88-93)."""
    n = C.c_size_t()
    check(lib.dimg_rtab_load(path.encode(), None, 0, C.byref(n)))
    out = np.empty(max(1, n.value), np.uint8)
    check(lib.dimg_rtab_load(path.encode(), ptr(out, u8p), out.size, C.byref(n)))
    return deserialize_rope_tables(out[:n.value].tobytes())


class InferenceSession:
    """Owns one sequence's KV cache on a GPU; single writer (engine.hpp:41-57)."""

    def __init__(self, model: ModelFile, opts: Optional[EngineOptions] = None,
                 imported_tables=None, keep_logits_cap: int = 0):
        self.opts = opts or EngineOptions()
        model.config.validate()
        if imported_tables is not None:
            c, s = imported_tables
            half = model.config.d_head // 2
            if c.size % max(1, half) or c.size // max(1, half) < model.config.max_ctx:
                raise errors.InvalidArgument("session: imported tables do not fit the model")
        self.model = model
        self._dm = model.device_model(self.opts.device, imported_tables)
        h = C.c_void_p()
        check(lib.dimg_session_create(self._dm._h, keep_logits_cap, C.byref(h)))
        self._h = h
        self.vocab = model.config.vocab

    def forward(self, token: int, pos: int) -> np.ndarray:
        """Runs token at position pos (== cache length); returns the logits."""
        out = np.empty(self.vocab, np.int64)
        check(lib.dimg_session_forward(self._h, token, pos, ptr(out, i64p)))
        return out

    @property
    def cache_len(self) -> int:
        n = C.c_uint32()
        check(lib.dimg_session_len(self._h, C.byref(n)))
        return n.value

    def reset(self):
        check(lib.dimg_session_reset(self._h))

    def generate_greedy(self, prompt: Sequence[int], max_new: int, keep_logits: bool = False):
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        toks = np.zeros(max(1, max_new), np.uint32)
        h = (C.c_uint8 * 32)()
        logits = np.empty((max_new, self.vocab), np.int64) if keep_logits else None
        check(lib.dimg_generate_greedy(self._h, ptr(p, u32p), p.size, max_new, ptr(toks, u32p), h,
                                       ptr(logits, i64p) if keep_logits else None))
        res = GenerationResult([int(t) for t in toks[:max_new]], bytes(h))
        if keep_logits:
            res.logits = [logits[i] for i in range(max_new)]
        return res

    def generate_sampled(self, prompt: Sequence[int], max_new: int, temperature: int, key: bytes):
        """generate_sampled (engine.cpp:148-163) with the RNG key given
        (sample_key); tokens drawn on the device step by step."""
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        toks = np.zeros(max(1, max_new), np.uint32)
        h = (C.c_uint8 * 32)()
        k = (C.c_uint8 * 32)(*key)
        check(lib.dimg_generate_sampled(self._h, ptr(p, u32p), p.size, max_new, int(temperature), k,
                                        ptr(toks, u32p), h))
        return GenerationResult([int(t) for t in toks[:max_new]], bytes(h))

    # ---- device-resident stepping (bench)
    def begin(self, prompt: Sequence[int], max_new: int):
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        check(lib.dimg_session_begin(self._h, ptr(p, u32p), p.size, max_new))

    def prefill(self):
        check(lib.dimg_session_prefill(self._h))

    def decode(self, n: int):
        check(lib.dimg_session_decode(self._h, n))

    def time_decode(self, n: int) -> float:
        ms = C.c_float()
        check(lib.dimg_session_time_decode(self._h, n, C.byref(ms)))
        return ms.value

    KERNELS = ("qkv_gemv", "wo_gemv", "gate_up_gemv", "down_gemv", "lm_head_gemv")

    def time_prefill(self):
        """(ms, tensor_cores) of the prefill of the begun prompt (CUDA events)."""
        ms = C.c_float()
        tc = C.c_uint32()
        check(lib.dimg_session_time_prefill(self._h, C.byref(ms), C.byref(tc)))
        return ms.value, bool(tc.value)

    def time_kernel(self, which: int, n: int):
        """(ms per launch, algorithmic bytes per launch) of kernel class `which`."""
        ms = C.c_float()
        b = C.c_uint64()
        check(lib.dimg_session_time_kernel(self._h, which, n, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def trace(self, n_steps: int, cap: int):
        """Per-stage %globaltimer stamps of CTA 0 over n decode steps: [cap, 4]
        = (start, prologue done, chunks done, epilogue done) in ns, [4..31] clock64 sub-stamps."""
        out = np.zeros(cap * 32, np.uint64)
        check(lib.dimg_session_trace(self._h, n_steps, ptr(out, u64p), cap))
        return out.reshape(cap, 32)

    def sync(self):
        check(lib.dimg_session_sync(self._h))

    def tokens(self, n: int) -> List[int]:
        out = np.zeros(max(1, n), np.uint32)
        check(lib.dimg_session_tokens(self._h, ptr(out, u32p), n))
        return [int(t) for t in out[:n]]

    def stream(self) -> int:
        p = C.c_void_p()
        check(lib.dimg_session_stream(self._h, C.byref(p)))
        return p.value or 0

    def launches(self):
        d, p = C.c_uint32(), C.c_uint32()
        check(lib.dimg_session_launches(self._h, C.byref(d), C.byref(p)))
        return d.value, p.value

    def stats(self):
        out = np.zeros(4, np.uint64)
        check(lib.dimg_session_stats(self._h, ptr(out, u64p)))
        return {"wide_limb_ctas": int(out[0]), "err": int(out[1]), "wide_kv_ctas": int(out[2]),
                "tc_prefills": int(out[3]) & 0xFFFFFFFF, "tc_fallbacks": int(out[3]) >> 32}

    def __del__(self):
        try:
            lib.dimg_session_free(self._h)
        except Exception:
            pass


_session_cache = {}


def _cached_session(model: ModelFile, opts: EngineOptions, keep: int, tables):
    key = (id(model), opts.device, None if tables is None else id(tables))
    s = _session_cache.get(key)
    if s is None or s.model is not model:
        s = InferenceSession(model, EngineOptions(device=opts.device), tables, keep_logits_cap=keep)
        _session_cache[key] = s
    return s


def generate_greedy(model: ModelFile, prompt: Sequence[int], max_new: int,
                    opts: Optional[EngineOptions] = None, imported_tables=None) -> GenerationResult:
    """generate_greedy (engine.cpp:142-147) on the GPU: prompt + greedy
    continuation + BLAKE3 output hash; logits when opts.keep_logits."""
    opts = opts or EngineOptions()
    sess = _cached_session(model, opts, max_new if opts.keep_logits else 0, imported_tables)
    return sess.generate_greedy(prompt, max_new, keep_logits=opts.keep_logits)


def generate_greedy_batch(model: ModelFile, prompts: Sequence[Sequence[int]], max_new: int,
                          device: int = 0):
    """generate_greedy for many independent sequences at once (C5): stepped
    together on the tensor cores (one limb GEMM per matrix per step for all
    sequences), bit-identical to separate generate_greedy calls. Returns
    (results, path) with path "tensor_cores" or "per_sequence"."""
    dm = model.device_model(device)
    n = len(prompts)
    lens = np.array([len(p) for p in prompts], np.uint32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.uint32) for p in prompts]) if n else
                                np.zeros(1, np.uint32), np.uint32)
    toks = np.zeros((max(1, n), max(1, max_new)), np.uint32)
    hashes = np.zeros((max(1, n), 32), np.uint8)
    path = C.c_uint32()
    check(lib.dimg_generate_greedy_batch(dm._h, n, ptr(flat, u32p), ptr(lens, u32p), max_new, ptr(toks, u32p),
                                         ptr(hashes, u8p), C.byref(path)))
    res = [GenerationResult([int(t) for t in toks[i, :max_new]], bytes(hashes[i])) for i in range(n)]
    return res, "tensor_cores" if path.value else "per_sequence"


def release_sessions():
    _session_cache.clear()


# ---- operator-level entry points (proj/src/kernels.cpp), GPU kernels --------

def _qt(w, s):
    w = np.ascontiguousarray(w, np.int8)
    s = np.ascontiguousarray(s, np.int64)
    return QTensor(w.shape[0], w.shape[1], ptr(w, i8p), ptr(s, i64p)), (w, s)


def dense_forward(w, scales, x, device: int = 0) -> np.ndarray:
    qt, keep = _qt(w, scales)
    x = np.ascontiguousarray(x, np.int64)
    if x.size != qt.cols:
        raise errors.InvalidArgument("dense_forward: dimension mismatch")
    out = np.empty(qt.rows, np.int64)
    check(lib.dimg_op_dense(device, C.byref(qt), ptr(x, i64p), ptr(out, i64p)))
    return out


def sample_key(model_bytes, prompt: Sequence[int], device: int = 0) -> bytes:
    """generate_sampled's RNG key (engine.cpp:151-157): BLAKE3(model bytes ||
    prompt ids u32 LE), hashed on the GPU."""
    mb = np.frombuffer(memoryview(model_bytes).cast("B"), np.uint8) if not isinstance(model_bytes, np.ndarray) \
        else np.ascontiguousarray(model_bytes).view(np.uint8).reshape(-1)
    p = np.ascontiguousarray(prompt, np.uint32)
    out = (C.c_uint8 * 32)()
    check(lib.dimg_sample_key(device, mb.ctypes.data_as(u8p), mb.size, ptr(p, u32p), p.size, out))
    return bytes(out)


def sample_from_logits(logits, temperature: int, draw: int, device: int = 0) -> int:
    """sample_from_logits (engine.cpp:122-139) of one row with the given
    ChaCha20 draw, on the GPU."""
    a = np.ascontiguousarray(logits, np.int64)
    out = C.c_uint32()
    check(lib.dimg_op_sample(device, ptr(a, i64p), a.size, int(temperature), int(draw), C.byref(out)))
    return out.value


def generate_sampled(model: ModelFile, prompt: Sequence[int], max_new: int, temperature: int,
                     opts: Optional[EngineOptions] = None) -> GenerationResult:
    """generate_sampled (engine.cpp:148-163): Q16 temperature > 0, the RNG
    keyed by BLAKE3(model bytes || prompt)."""
    opts = opts or EngineOptions()
    if temperature <= 0:
        raise errors.InvalidArgument("sample: temperature must be positive")
    key = sample_key(model.bytes, prompt, opts.device)
    sess = _cached_session(model, opts, 0, None)
    return sess.generate_sampled(prompt, max_new, temperature, key)


def blake3_gpu(data, device: int = 0) -> bytes:
    """BLAKE3 of host bytes on the GPU (upload + device tree hash): the
    model-bytes hash of weight_hash (proj/src/model.cpp:310-316)."""
    buf = np.frombuffer(memoryview(data).cast("B"), np.uint8) if not isinstance(data, np.ndarray) \
        else np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    out = (C.c_uint8 * 32)()
    check(lib.dimg_blake3_gpu(device, buf.ctypes.data_as(C.c_void_p), buf.size, out))
    return bytes(out)


def blake3_device(ptr: int, length: int, device: int = 0, timed: bool = False):
    """BLAKE3 of `length` bytes at device pointer `ptr` (e.g. a CUDA tensor's
    data_ptr()); with timed=True returns (digest, kernel ms)."""
    out = (C.c_uint8 * 32)()
    ms = C.c_float()
    check(lib.dimg_blake3_device(device, C.c_void_p(ptr), length, out, C.byref(ms) if timed else None))
    return (bytes(out), ms.value) if timed else bytes(out)


def dense_tokens(w, scales, x, device: int = 0) -> np.ndarray:
    """dense_forward for every row of x [T, cols] -> [T, rows]: the prefill
    GEMM on the tensor cores (exact byte-limb int8 products)."""
    qt, keep = _qt(w, scales)
    x = np.ascontiguousarray(x, np.int64)
    if x.ndim != 2 or x.shape[1] != qt.cols:
        raise errors.InvalidArgument("dense_tokens: dimension mismatch")
    out = np.empty((x.shape[0], qt.rows), np.int64)
    check(lib.dimg_op_dense_tokens(device, C.byref(qt), ptr(x, i64p), x.shape[0], ptr(out, i64p)))
    return out


def rmsnorm(x, gamma, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, np.int64)
    g = np.ascontiguousarray(gamma, np.int64)
    if x.size != g.size:
        raise errors.InvalidArgument("rmsnorm: gamma size mismatch")
    out = np.empty_like(x)
    check(lib.dimg_op_rmsnorm(device, ptr(x, i64p), ptr(g, i64p), x.size, ptr(out, i64p)))
    return out


def softmax_q16(scores, device: int = 0) -> np.ndarray:
    s = np.ascontiguousarray(scores, np.int64)
    out = np.empty_like(s)
    check(lib.dimg_op_softmax(device, ptr(s, i64p), s.size, ptr(out, i64p)))
    return out


def attention_steps(n_heads, d_head, max_ctx, theta, q, k, v, device: int = 0) -> np.ndarray:
    q, k, v = (np.ascontiguousarray(a, np.int64) for a in (q, k, v))
    out = np.empty_like(q)
    check(lib.dimg_op_attention(device, n_heads, d_head, max_ctx, theta, q.shape[0], ptr(q, i64p),
                                ptr(k, i64p), ptr(v, i64p), ptr(out, i64p)))
    return out


def ffn_silu(x, wg, sg, wu, su, wd, sd, device: int = 0) -> np.ndarray:
    g, k1 = _qt(wg, sg)
    u, k2 = _qt(wu, su)
    d, k3 = _qt(wd, sd)
    x = np.ascontiguousarray(x, np.int64)
    out = np.empty(d.rows, np.int64)
    check(lib.dimg_op_ffn(device, C.byref(g), C.byref(u), C.byref(d), ptr(x, i64p), ptr(out, i64p)))
    return out


def device_count() -> int:
    n = C.c_int()
    check(lib.dimg_device_count(C.byref(n)))
    return n.value
