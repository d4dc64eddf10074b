"""TEST INFRASTRUCTURE ONLY: ctypes front-end for the two CPU checkers.

* ``Oracle`` -- the plain-C restatement (oracle/dim_oracle.c), built on demand
  with gcc (present here and on the GPU box).
* ``Reference`` -- the unmodified reference engine compiled from
  /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdimref.so.
  That file is built in this container and shipped to the GPU box by gpurun;
  where it is absent ``Reference.available()`` is False.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libdim_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdimref.so")
_lock = threading.Lock()

u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
i64p = C.POINTER(C.c_int64)
u32p = C.POINTER(C.c_uint32)


def chacha20_u32s(key32: bytes, n: int):
    """The first n next_u32() of ChaCha20Rng(key) (proj/src/chacha20.cpp:48-78):
    RFC 8439 blocks, key words little-endian, nonce 0, counter from 0, bytes
    consumed in order, u32 = 4 bytes LE. Pure Python (small n)."""
    M = 0xFFFFFFFF
    key = [int.from_bytes(key32[4 * i:4 * i + 4], "little") for i in range(8)]

    def rotl(x, r):
        return ((x << r) | (x >> (32 - r))) & M

    def qr(s, a, b, c, d):
        s[a] = (s[a] + s[b]) & M; s[d] = rotl(s[d] ^ s[a], 16)
        s[c] = (s[c] + s[d]) & M; s[b] = rotl(s[b] ^ s[c], 12)
        s[a] = (s[a] + s[b]) & M; s[d] = rotl(s[d] ^ s[a], 8)
        s[c] = (s[c] + s[d]) & M; s[b] = rotl(s[b] ^ s[c], 7)

    out, ctr = bytearray(), 0
    while len(out) < 4 * n:
        init = [0x61707865, 0x3320646E, 0x79622D32, 0x6B206574] + key + [ctr, 0, 0, 0]
        s = list(init)
        for _ in range(10):
            qr(s, 0, 4, 8, 12); qr(s, 1, 5, 9, 13); qr(s, 2, 6, 10, 14); qr(s, 3, 7, 11, 15)
            qr(s, 0, 5, 10, 15); qr(s, 1, 6, 11, 12); qr(s, 2, 7, 8, 13); qr(s, 3, 4, 9, 14)
        for i in range(16):
            out += ((s[i] + init[i]) & M).to_bytes(4, "little")
        ctr += 1
    return [int.from_bytes(out[4 * i:4 * i + 4], "little") for i in range(n)]


def _ptr(a, t):
    return a.ctypes.data_as(t)


def build_oracle(force: bool = False) -> str:
    with _lock:
        src = os.path.join(HERE, "dim_oracle.c")
        if force or not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return ORACLE_SO


class Config:
    """ModelConfig (proj/include/dim/model.hpp:15-29)."""

    def __init__(self, n_layers, d_model, n_heads, d_ffn, vocab, max_ctx, rope_theta=10000.0):
        self.n_layers, self.d_model, self.n_heads = n_layers, d_model, n_heads
        self.d_ffn, self.vocab, self.max_ctx, self.rope_theta = d_ffn, vocab, max_ctx, rope_theta

    def tuple6(self):
        return (self.n_layers, self.d_model, self.n_heads, self.d_ffn, self.vocab, self.max_ctx)

    @property
    def d_head(self):
        return self.d_model // self.n_heads

    def tensor_shapes(self):
        """Quantised tensors in directory order (proj/src/model.cpp:41-61)."""
        D, F, V = self.d_model, self.d_ffn, self.vocab
        s = [(V, D)]
        for _ in range(self.n_layers):
            s += [(D, D)] * 4 + [(F, D), (F, D), (D, F)]
        s.append((V, D))
        return s

    def n_weights(self):
        return sum(r * c for r, c in self.tensor_shapes())

    def n_scales(self):
        return sum(r for r, _ in self.tensor_shapes())


class _QT(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("data", i8p), ("scales", i64p)]


class _Model(C.Structure):
    _fields_ = [
        ("n_layers", C.c_uint32), ("d_model", C.c_uint32), ("n_heads", C.c_uint32),
        ("d_ffn", C.c_uint32), ("vocab", C.c_uint32), ("max_ctx", C.c_uint32),
        ("rope_theta", C.c_double), ("tok_embd", _QT), ("output", _QT),
        ("layers", C.POINTER(_QT)), ("norms", i64p),
    ]


class OracleModel:
    """Directory-order weights/scales/norms plus the bound C descriptor."""

    def __init__(self, lib, cfg: Config, weights, scales, norms):
        self.lib, self.cfg = lib, cfg
        self.weights = np.ascontiguousarray(weights, dtype=np.int8)
        self.scales = np.ascontiguousarray(scales, dtype=np.int64)
        self.norms = np.ascontiguousarray(norms, dtype=np.int64)
        self._layers = (_QT * max(1, 7 * cfg.n_layers))()
        m = _Model()
        (m.n_layers, m.d_model, m.n_heads, m.d_ffn, m.vocab, m.max_ctx) = cfg.tuple6()
        m.rope_theta = cfg.rope_theta
        m.norms = _ptr(self.norms, i64p)
        lib.orc_bind(C.byref(m), self._layers, _ptr(self.weights, i8p), _ptr(self.scales, i64p))
        self.c = m

    def weight_hash(self) -> str:
        out = (C.c_uint8 * 32)()
        self.lib.orc_weight_hash(C.byref(self.c), out)
        return bytes(out).hex()

    def serialize(self) -> bytes:
        n = self.lib.orc_serialized_size(C.byref(self.c))
        buf = np.empty(n, dtype=np.uint8)
        self.lib.orc_serialize(C.byref(self.c), _ptr(buf, u8p))
        return buf.tobytes()

    def tensor(self, idx):
        """(int8 [rows, cols], int64 [rows]) of quantised tensor idx (directory order)."""
        shapes = self.cfg.tensor_shapes()
        wo = sum(r * c for r, c in shapes[:idx])
        so = sum(r for r, _ in shapes[:idx])
        r, c = shapes[idx]
        return self.weights[wo:wo + r * c].reshape(r, c), self.scales[so:so + r]


class Oracle:
    def __init__(self):
        lib = C.CDLL(build_oracle())
        lib.orc_inv_sqrt.restype = C.c_int64
        lib.orc_inv_sqrt.argtypes = [C.c_int64]
        lib.orc_invsqrt_seed.restype = C.c_int64
        lib.orc_invsqrt_seed.argtypes = [C.c_int]
        lib.orc_exp_entry.restype = C.c_int64
        lib.orc_exp_entry.argtypes = [C.c_int]
        for f in ("orc_exp_neg", "orc_sigmoid", "orc_silu"):
            getattr(lib, f).restype = C.c_int64
            getattr(lib, f).argtypes = [C.c_int64]
        lib.orc_q16_from_ratio.restype = C.c_int64
        lib.orc_q16_from_ratio.argtypes = [C.c_int64, C.c_int64]
        lib.orc_q16_mul.restype = C.c_int64
        lib.orc_q16_mul.argtypes = [C.c_int64, C.c_int64]
        lib.orc_rope_tables.argtypes = [C.c_double, C.c_uint32, C.c_uint32, i64p, i64p]
        lib.orc_gen_toy.argtypes = [C.c_uint64, C.c_void_p, i8p, i64p]
        lib.orc_serialized_size.restype = C.c_uint64
        lib.orc_session_new.restype = C.c_void_p
        lib.orc_session_new.argtypes = [C.c_void_p]
        lib.orc_session_free.argtypes = [C.c_void_p]
        lib.orc_session_forward.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, i64p]
        lib.orc_select_greedy.restype = C.c_uint32
        lib.orc_generate_greedy.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_uint32, u32p,
                                            u8p, i64p]
        lib.orc_rng_u32.restype = C.c_uint32
        self.lib = lib

    # ---- primitives
    def blake3(self, data: bytes) -> str:
        out = (C.c_uint8 * 32)()
        self.lib.orc_blake3_oneshot(C.c_char_p(bytes(data)), C.c_size_t(len(data)), out)
        return bytes(out).hex()

    def blake3_array(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        out = (C.c_uint8 * 32)()
        self.lib.orc_blake3_oneshot(C.c_void_p(a.ctypes.data), C.c_size_t(a.nbytes), out)
        return bytes(out).hex()

    def exp_lut(self):
        return np.array([self.lib.orc_exp_entry(i) for i in range(257)], dtype=np.int64)

    def invsqrt_seeds(self):
        return np.array([self.lib.orc_invsqrt_seed(b) for b in range(64)], dtype=np.int64)

    def rope_tables(self, theta, d_head, max_ctx):
        c = np.empty(max_ctx * (d_head // 2), np.int64)
        s = np.empty_like(c)
        self.lib.orc_rope_tables(theta, d_head, max_ctx, _ptr(c, i64p), _ptr(s, i64p))
        return c, s

    def prompt(self, seed, vocab, n):
        class Rng(C.Structure):
            _fields_ = [("key", C.c_uint32 * 8), ("counter", C.c_uint32),
                        ("buf", C.c_uint8 * 64), ("pos", C.c_uint32)]
        r = Rng()
        self.lib.orc_rng_from_seed(C.byref(r), C.c_uint64(seed))
        return np.array([self.lib.orc_rng_u32(C.byref(r)) % vocab for _ in range(n)], np.uint32)

    # ---- model
    def gen_toy(self, seed: int, cfg: Config) -> OracleModel:
        w = np.empty(cfg.n_weights(), np.int8)
        s = np.empty(cfg.n_scales(), np.int64)
        probe = _Model()
        (probe.n_layers, probe.d_model, probe.n_heads, probe.d_ffn, probe.vocab,
         probe.max_ctx) = cfg.tuple6()
        self.lib.orc_gen_toy(C.c_uint64(seed), C.byref(probe), _ptr(w, i8p), _ptr(s, i64p))
        norms = np.full((2 * cfg.n_layers + 1) * cfg.d_model, 65536, np.int64)
        return OracleModel(self.lib, cfg, w, s, norms)

    def model(self, cfg: Config, weights, scales, norms) -> OracleModel:
        return OracleModel(self.lib, cfg, weights, scales, norms)

    def generate_greedy(self, m: OracleModel, prompt, max_new, keep_logits=False):
        p = np.ascontiguousarray(prompt, dtype=np.uint32)
        toks = np.zeros(max(1, max_new), np.uint32)
        h = (C.c_uint8 * 32)()
        logits = np.zeros((max_new, m.cfg.vocab), np.int64) if keep_logits else None
        rc = self.lib.orc_generate_greedy(C.byref(m.c), _ptr(p, u32p), len(p), max_new,
                                          _ptr(toks, u32p), h,
                                          _ptr(logits, i64p) if keep_logits else None)
        if rc:
            raise RuntimeError(f"oracle generate rc={rc}")
        return toks[:max_new], bytes(h).hex(), logits

    def session(self, m: OracleModel):
        return OracleSession(self, m)

    # ---- operators
    def dense(self, w, s, x):
        w = np.ascontiguousarray(w, np.int8)
        s = np.ascontiguousarray(s, np.int64)
        x = np.ascontiguousarray(x, np.int64)
        qt = _QT(w.shape[0], w.shape[1], _ptr(w, i8p), _ptr(s, i64p))
        out = np.empty(w.shape[0], np.int64)
        self.lib.orc_dense(C.byref(qt), _ptr(x, i64p), _ptr(out, i64p))
        return out

    def rmsnorm(self, x, g):
        x = np.ascontiguousarray(x, np.int64)
        g = np.ascontiguousarray(g, np.int64)
        out = np.empty_like(x)
        self.lib.orc_rmsnorm(_ptr(x, i64p), _ptr(g, i64p), C.c_uint32(len(x)), _ptr(out, i64p))
        return out

    def softmax(self, s):
        s = np.ascontiguousarray(s, np.int64)
        out = np.empty_like(s)
        self.lib.orc_softmax(_ptr(s, i64p), C.c_uint32(len(s)), _ptr(out, i64p))
        return out

    def sample_from_logits(self, logits, temperature: int, draw: int) -> int:
        """sample_from_logits (proj/src/engine.cpp:122-139) given the step's
        ChaCha20 u32: truncating int128 temperature division (low 64 bits),
        softmax_q16 (the C oracle's), threshold (draw * sum p) >> 32, first
        index whose cumulative mass exceeds it."""
        if temperature <= 0 or len(logits) == 0:
            raise ValueError("sample: temperature must be positive / empty logits")
        scaled = []
        for v in logits:
            num = int(v) << 16
            q = abs(num) // temperature
            q = q if num >= 0 else -q
            q &= (1 << 64) - 1
            scaled.append(q - (1 << 64) if q >= 1 << 63 else q)
        self.lib.orc_domain_error()  # clear
        p = self.softmax(np.array(scaled, np.int64))
        if self.lib.orc_domain_error():  # exp_neg_lut's std::domain_error (q16.cpp:82)
            raise ArithmeticError("exp_neg_lut: argument outside [0, 8]")
        total = int(sum(int(x) for x in p))
        threshold = (int(draw) * total) >> 32
        cum = 0
        for i, x in enumerate(p):
            cum += int(x)
            if cum > threshold:
                return i
        return len(p) - 1

    def attention(self, H, dh, max_ctx, theta, q, k, v):
        """Consecutive attention steps at pos 0..T-1; q/k/v [T, H*dh]."""
        q, k, v = (np.ascontiguousarray(a, np.int64) for a in (q, k, v))
        T, D = q.shape
        c, s = self.rope_tables(theta, dh, max_ctx)
        kc = np.zeros((max_ctx, D), np.int64)
        vc = np.zeros((max_ctx, D), np.int64)
        out = np.empty((T, D), np.int64)
        for t in range(T):
            self.lib.orc_attention_step(_ptr(q[t], i64p), _ptr(k[t], i64p), _ptr(v[t], i64p),
                                        C.c_uint32(H), C.c_uint32(dh), C.c_uint32(max_ctx),
                                        _ptr(kc, i64p), _ptr(vc, i64p), C.c_uint32(t),
                                        _ptr(c, i64p), _ptr(s, i64p), _ptr(out[t], i64p))
        return out

    def ffn(self, wg, sg, wu, su, wd, sd, x):
        arrs = [np.ascontiguousarray(a) for a in (wg, sg, wu, su, wd, sd, x)]
        wg, sg, wu, su, wd, sd, x = arrs
        g = _QT(wg.shape[0], wg.shape[1], _ptr(wg, i8p), _ptr(sg, i64p))
        u = _QT(wu.shape[0], wu.shape[1], _ptr(wu, i8p), _ptr(su, i64p))
        d = _QT(wd.shape[0], wd.shape[1], _ptr(wd, i8p), _ptr(sd, i64p))
        out = np.empty(wd.shape[0], np.int64)
        self.lib.orc_ffn(C.byref(g), C.byref(u), C.byref(d), _ptr(x, i64p), _ptr(out, i64p))
        return out


class OracleSession:
    ERRORS = {-1: IndexError, -2: OverflowError, -3: RuntimeError}

    def __init__(self, orc: Oracle, m: OracleModel):
        self.orc, self.m = orc, m
        self.h = orc.lib.orc_session_new(C.byref(m.c))

    def forward(self, token, pos, want_logits=True):
        out = np.empty(self.m.cfg.vocab, np.int64) if want_logits else None
        rc = self.orc.lib.orc_session_forward(self.h, token, pos,
                                              _ptr(out, i64p) if want_logits else None)
        if rc:
            raise self.ERRORS[rc](f"oracle forward rc={rc}")
        return out

    def __del__(self):
        try:
            self.orc.lib.orc_session_free(self.h)
        except Exception:
            pass


# --------------------------------------------------------------------------
class Reference:
    """The reference engine itself (oracle/_ref/libdimref.so)."""

    @staticmethod
    def available() -> bool:
        if os.path.exists(REF_SO):
            return True
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-C", HERE, "ref"], check=False)
        return os.path.exists(REF_SO)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        lib.ref_sigmoid.restype = C.c_int64
        lib.ref_sigmoid.argtypes = [C.c_int64]
        lib.ref_silu.restype = C.c_int64
        lib.ref_silu.argtypes = [C.c_int64]
        lib.ref_inv_sqrt.argtypes = [C.c_int64, i64p]
        lib.ref_exp_neg.argtypes = [C.c_int64, i64p]
        lib.ref_q16_from_ratio.argtypes = [C.c_int64, C.c_int64, i64p]
        lib.ref_rope_tables.argtypes = [C.c_double, C.c_uint32, C.c_uint32, i64p, i64p]
        lib.ref_gen_toy_model.argtypes = [C.c_uint64, u32p, C.c_double, C.POINTER(C.c_void_p)]
        lib.ref_model_from_arrays.argtypes = [u32p, C.c_double, i8p, i64p, i64p,
                                              C.POINTER(C.c_void_p)]
        lib.ref_deserialize.argtypes = [u8p, C.c_size_t, C.POINTER(C.c_void_p)]
        lib.ref_model_free.argtypes = [C.c_void_p]
        lib.ref_model_weight_hash.argtypes = [C.c_void_p, u8p]
        lib.ref_model_bytes.restype = C.c_size_t
        lib.ref_model_bytes.argtypes = [C.c_void_p, u8p]
        lib.ref_model_export.argtypes = [C.c_void_p, i8p, i64p, i64p]
        lib.ref_generate_greedy.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_uint32, C.c_int,
                                            C.c_size_t, u32p, u8p, i64p]
        lib.ref_session_new.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        lib.ref_session_free.argtypes = [C.c_void_p]
        lib.ref_session_forward.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, i64p, u32p]
        lib.ref_prompt.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p]
        lib.ref_dense.argtypes = [C.c_uint32, C.c_uint32, i8p, i64p, i64p, C.c_size_t, i64p]
        lib.ref_rmsnorm.argtypes = [i64p, i64p, C.c_uint32, i64p]
        lib.ref_softmax.argtypes = [i64p, C.c_uint32, i64p]
        lib.ref_attention.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint32,
                                      i64p, i64p, i64p, C.c_int, i64p]
        lib.ref_ffn.argtypes = [C.c_uint32, C.c_uint32, i8p, i64p, i8p, i64p, i8p, i64p, i64p, i64p]
        lib.ref_generation_counter.restype = C.c_uint64
        lib.ref_sample_from_logits.argtypes = [i64p, C.c_uint32, C.c_int64, u8p, u32p]
        self.lib = lib

    def sample_from_logits(self, logits, temperature: int, key32: bytes):
        """The reference's sample_from_logits with ChaCha20Rng(key32): (status,
        token); status 0 ok, 1 invalid_argument, 6 domain_error."""
        a = np.ascontiguousarray(logits, np.int64)
        out = C.c_uint32(0xFFFFFFFF)
        k = (C.c_uint8 * 32)(*key32)
        rc = self.lib.ref_sample_from_logits(_ptr(a, i64p), len(a), int(temperature), k, C.byref(out))
        return rc, out.value

    def blake3(self, data: bytes) -> str:
        out = (C.c_uint8 * 32)()
        self.lib.ref_blake3(C.c_char_p(bytes(data)), C.c_size_t(len(data)), out)
        return bytes(out).hex()

    def exp_lut(self):
        out = np.empty(257, np.int64)
        self.lib.ref_exp_lut(_ptr(out, i64p))
        return out

    def inv_sqrt(self, x):
        out = C.c_int64()
        rc = self.lib.ref_inv_sqrt(x, C.byref(out))
        if rc:
            raise ValueError(rc)
        return out.value

    def rope_tables(self, theta, d_head, max_ctx):
        c = np.empty(max_ctx * (d_head // 2), np.int64)
        s = np.empty_like(c)
        rc = self.lib.ref_rope_tables(theta, d_head, max_ctx, _ptr(c, i64p), _ptr(s, i64p))
        if rc:
            raise ValueError(rc)
        return c, s

    def prompt(self, seed, vocab, n):
        out = np.empty(n, np.uint32)
        self.lib.ref_prompt(seed, vocab, n, _ptr(out, u32p))
        return out

    def gen_toy(self, seed, cfg: Config):
        c6 = np.array(cfg.tuple6(), np.uint32)
        h = C.c_void_p()
        rc = self.lib.ref_gen_toy_model(seed, _ptr(c6, u32p), cfg.rope_theta, C.byref(h))
        if rc:
            raise ValueError(rc)
        return RefModel(self, cfg, h)

    def model_from_arrays(self, cfg: Config, weights, scales, norms):
        c6 = np.array(cfg.tuple6(), np.uint32)
        h = C.c_void_p()
        rc = self.lib.ref_model_from_arrays(_ptr(c6, u32p), cfg.rope_theta,
                                            _ptr(np.ascontiguousarray(weights, np.int8), i8p),
                                            _ptr(np.ascontiguousarray(scales, np.int64), i64p),
                                            _ptr(np.ascontiguousarray(norms, np.int64), i64p),
                                            C.byref(h))
        if rc:
            raise ValueError(rc)
        return RefModel(self, cfg, h)

    def generate_greedy(self, m: "RefModel", prompt, max_new, threads=1, chunk=0,
                        keep_logits=False):
        p = np.ascontiguousarray(prompt, np.uint32)
        toks = np.zeros(max(1, max_new), np.uint32)
        h = (C.c_uint8 * 32)()
        logits = np.zeros((max_new, m.cfg.vocab), np.int64) if keep_logits else None
        rc = self.lib.ref_generate_greedy(m.h, _ptr(p, u32p), len(p), max_new, threads, chunk,
                                          _ptr(toks, u32p), h,
                                          _ptr(logits, i64p) if keep_logits else None)
        if rc:
            raise RuntimeError(f"reference generate rc={rc}")
        return toks[:max_new], bytes(h).hex(), logits


class RefModel:
    def __init__(self, ref: Reference, cfg: Config, h):
        self.ref, self.cfg, self.h = ref, cfg, h

    def weight_hash(self):
        out = (C.c_uint8 * 32)()
        self.ref.lib.ref_model_weight_hash(self.h, out)
        return bytes(out).hex()

    def export(self):
        w = np.empty(self.cfg.n_weights(), np.int8)
        s = np.empty(self.cfg.n_scales(), np.int64)
        n = np.empty((2 * self.cfg.n_layers + 1) * self.cfg.d_model, np.int64)
        self.ref.lib.ref_model_export(self.h, _ptr(w, i8p), _ptr(s, i64p), _ptr(n, i64p))
        return w, s, n

    def __del__(self):
        try:
            self.ref.lib.ref_model_free(self.h)
        except Exception:
            pass
