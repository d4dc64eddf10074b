"""Host model container and configuration (proj/include/dim/model.hpp).

``ModelFile`` holds the canonical DIM1 bytes in the C++ host library (the
reference's ModelFile keeps the same pair: tensors + ``bytes``) and lazily
uploads itself to a GPU the first time a session needs it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Optional, Tuple

import numpy as np

from ._lib import Config, ModelDesc, QTensor, check, i8p, i64p, lib, ptr, u8p

ONE = 1 << 16


@dataclass(frozen=True)
class ModelConfig:
    """ModelConfig (proj/include/dim/model.hpp:15-29)."""

    n_layers: int = 0
    d_model: int = 0
    n_heads: int = 0
    d_ffn: int = 0
    vocab: int = 0
    max_ctx: int = 0
    rope_theta: float = 10000.0

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    def to_c(self) -> Config:
        return Config(self.n_layers, self.d_model, self.n_heads, self.d_ffn, self.vocab,
                      self.max_ctx, self.rope_theta)

    def validate(self) -> None:
        """model.cpp:95-109; raises InvalidArgument."""
        c = self.to_c()
        check(lib.dimg_config_validate(C.byref(c)))

    def tensor_shapes(self):
        D, F, V = self.d_model, self.d_ffn, self.vocab
        s = [(V, D)]
        for _ in range(self.n_layers):
            s += [(D, D)] * 4 + [(F, D), (F, D), (D, F)]
        s.append((V, D))
        return s

    @staticmethod
    def tinyllama(max_ctx=2048):
        return ModelConfig(22, 2048, 32, 5632, 32000, max_ctx)

    @staticmethod
    def llama2_7b(max_ctx=4096):
        return ModelConfig(32, 4096, 32, 11008, 32000, max_ctx)


LAYER_TENSORS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")


class ModelFile:
    """Byte-exact model container (proj/include/dim/model.hpp:50-60)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if isinstance(handle, int) else handle
        d = ModelDesc()
        check(lib.dimg_host_model_desc(self._h, C.byref(d)))
        c = d.cfg
        self.config = ModelConfig(c.n_layers, c.d_model, c.n_heads, c.d_ffn, c.vocab, c.max_ctx,
                                  c.rope_theta)
        self._desc = d
        self._device_models: Dict[Tuple[int, Optional[int]], "DeviceModel"] = {}
        self._weight_hash: Optional[str] = None

    # ---- construction (model.cpp:189-215, 217-334)
    @classmethod
    def gen_toy(cls, seed: int, config: ModelConfig, threads: int = 0, device: Optional[int] = None) -> "ModelFile":
        """gen_toy_model; device=N synthesises the weight stream on GPU N."""
        h = C.c_void_p()
        c = config.to_c()
        if device is None:
            check(lib.dimg_host_model_gen_toy(C.c_uint64(seed), C.byref(c), threads, C.byref(h)))
        else:
            check(lib.dimg_host_model_gen_toy_gpu(device, C.c_uint64(seed), C.byref(c), C.byref(h)))
        return cls(h)

    @classmethod
    def from_bytes(cls, data) -> "ModelFile":
        buf = np.frombuffer(bytes(data) if not isinstance(data, (bytes, bytearray)) else data,
                            dtype=np.uint8)
        h = C.c_void_p()
        check(lib.dimg_host_model_from_bytes(ptr(buf, u8p), buf.size, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "ModelFile":
        h = C.c_void_p()
        check(lib.dimg_host_model_load(path.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, config: ModelConfig, tensors, norms) -> "ModelFile":
        """tensors: directory-order list of (int8 [rows, cols], int64 [rows]);
        norms: int64 [(2L+1) * d_model]."""
        keep = []
        qts = []
        for w, s in tensors:
            w = np.ascontiguousarray(w, np.int8)
            s = np.ascontiguousarray(s, np.int64)
            keep += [w, s]
            qts.append(QTensor(w.shape[0], w.shape[1], ptr(w, i8p), ptr(s, i64p)))
        norms = np.ascontiguousarray(norms, np.int64)
        layers = (QTensor * max(1, 7 * config.n_layers))(*qts[1:-1])
        d = ModelDesc(config.to_c(), qts[0], qts[-1], layers, ptr(norms, i64p), None, None, 0)
        h = C.c_void_p()
        check(lib.dimg_host_model_from_desc(C.byref(d), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        check(lib.dimg_host_model_save(self._h, path.encode()))

    # ---- views
    @property
    def bytes(self) -> memoryview:
        p = u8p()
        n = C.c_size_t()
        check(lib.dimg_host_model_bytes(self._h, C.byref(p), C.byref(n)))
        return memoryview((C.c_uint8 * n.value).from_address(C.addressof(p.contents))).cast("B")

    @property
    def weight_hash(self) -> str:
        """BLAKE3 of the exact container bytes (model.cpp:310,325-327)."""
        if self._weight_hash is None:
            out = (C.c_uint8 * 32)()
            check(lib.dimg_host_model_weight_hash(self._h, out))
            self._weight_hash = bytes(out).hex()
        return self._weight_hash

    def tensor(self, name: str):
        """(int8 [rows, cols], int64 [rows]) views of a quantised tensor."""
        if name == "tok_embd":
            t = self._desc.tok_embd
        elif name == "output":
            t = self._desc.output
        else:
            _, l, what = name.split(".")
            t = self._desc.layers[7 * int(l) + LAYER_TENSORS.index(what)]
        w = np.ctypeslib.as_array(t.data, shape=(t.rows, t.cols))
        s = np.ctypeslib.as_array(t.scales, shape=(t.rows,))
        return w, s

    def norms(self):
        n = (2 * self.config.n_layers + 1) * self.config.d_model
        return np.ctypeslib.as_array(self._desc.norms, shape=(n,))

    # ---- device copies
    def device_model(self, device: int = 0, rope: Optional[Tuple[np.ndarray, np.ndarray]] = None):
        key = (device, None if rope is None else id(rope))
        dm = self._device_models.get(key)
        if dm is None:
            dm = DeviceModel(self, device, rope)
            self._device_models[key] = dm
        return dm

    def __del__(self):
        try:
            self._device_models.clear()
            lib.dimg_host_model_free(self._h)
        except Exception:
            pass


class DeviceModel:
    """The model re-laid out in one GPU's HBM (dimg_model_upload)."""

    def __init__(self, mf: ModelFile, device: int, rope=None, tp_rank: int = 0, tp_size: int = 1):
        d = ModelDesc()
        check(lib.dimg_host_model_desc(mf._h, C.byref(d)))
        self._rope = rope
        if rope is not None:
            c, s = (np.ascontiguousarray(a, np.int64) for a in rope)
            self._rope = (c, s)
            d.rope_cos, d.rope_sin = ptr(c, i64p), ptr(s, i64p)
            d.rope_max_ctx = c.size // max(1, mf.config.d_head // 2)
        h = C.c_void_p()
        check(lib.dimg_model_upload(device, C.byref(d), tp_rank, tp_size, C.byref(h)))
        self._h = h
        self.device = device
        self.config = mf.config
        self._mf = mf

    def bytes_on_device(self) -> int:
        n = C.c_uint64()
        check(lib.dimg_model_bytes_on_device(self._h, C.byref(n)))
        return n.value

    def __del__(self):
        try:
            lib.dimg_model_free(self._h)
        except Exception:
            pass


def gen_toy_model(seed: int, config: ModelConfig, threads: int = 0, device: Optional[int] = None) -> ModelFile:
    """gen_toy_model (proj/src/model.cpp:189-215): all host cores, or the
    weight stream synthesised on GPU `device`."""
    return ModelFile.gen_toy(seed, config, threads, device)


def deserialize(data) -> ModelFile:
    return ModelFile.from_bytes(data)


def load_model(path: str) -> ModelFile:
    return ModelFile.load(path)


def weight_hash(data) -> str:
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    out = (C.c_uint8 * 32)()
    check(lib.dimg_blake3(buf.ctypes.data_as(C.c_void_p), buf.size, out))
    return bytes(out).hex()
