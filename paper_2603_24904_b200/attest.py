"""Attestation and re-execution verification (proj/include/dim/attest.hpp,
proj/src/attest.cpp): the direct callers of the generation hot path.

The 112-byte wire format and texts are the reference's; the model id is the
GPU BLAKE3 of the model bytes and the re-execution runs on the GPU engine
(dimg_verify_by_reexecution), so a 7B verification costs one upload, a
few-millisecond hash and one generation instead of minutes of host work.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from ._lib import Attestation as _CAtt
from ._lib import VerifyOutcome as _COut
from ._lib import check, lib
from .engine import EngineOptions, GenerationResult, hash_token_ids

_STAGES = ("model", "input", "output")


def _buf(model_bytes):
    if isinstance(model_bytes, np.ndarray):
        return np.ascontiguousarray(model_bytes).view(np.uint8).reshape(-1)
    return np.frombuffer(memoryview(model_bytes).cast("B"), np.uint8)


@dataclass(frozen=True)
class Attestation:
    """Attestation (attest.hpp:16-30)."""
    model_id: bytes
    input_hash: bytes
    output_hash: bytes
    bond: int
    challenge_period: int

    def _c(self) -> _CAtt:
        a = _CAtt()
        C.memmove(a.model_id, self.model_id, 32)
        C.memmove(a.input_hash, self.input_hash, 32)
        C.memmove(a.output_hash, self.output_hash, 32)
        a.bond, a.challenge_period = self.bond, self.challenge_period
        return a

    @staticmethod
    def _from_c(a: _CAtt) -> "Attestation":
        return Attestation(bytes(a.model_id), bytes(a.input_hash), bytes(a.output_hash), int(a.bond),
                           int(a.challenge_period))

    def encode(self) -> bytes:
        out = (C.c_uint8 * 112)()
        a = self._c()
        check(lib.dimg_attestation_encode(C.byref(a), out))
        return bytes(out)

    @staticmethod
    def decode(data) -> "Attestation":
        """Raises ParseError(kind=truncated) unless exactly 112 bytes."""
        buf = np.frombuffer(bytes(data), np.uint8)
        a = _CAtt()
        check(lib.dimg_attestation_decode(buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size, C.byref(a)))
        return Attestation._from_c(a)

    def to_text(self) -> str:
        a = self._c()
        n = C.c_size_t()
        buf = C.create_string_buffer(512)
        check(lib.dimg_attestation_text(C.byref(a), buf, 512, C.byref(n)))
        return buf.value.decode()


@dataclass(frozen=True)
class VerifyOutcome:
    """VerifyOutcome (attest.hpp:40-52)."""
    confirmed: bool
    refuted_stage: Optional[str] = None  # "model" | "input" | "output"
    expected: bytes = b""
    found: bytes = b""

    def to_text(self) -> str:
        if self.confirmed:
            return "Confirmed"
        return f"Refuted({self.refuted_stage}) expected={self.expected.hex()} found={self.found.hex()}"


@dataclass(frozen=True)
class DisputeResult:
    """DisputeResult (attest.hpp:58-68): winner "attester" or "challenger"."""
    winner: str
    outcome: VerifyOutcome


def prompt_hash(prompt_ids: Sequence[int]) -> bytes:
    """prompt_hash (attest.cpp:64-66) = hash_token_ids."""
    return hash_token_ids(prompt_ids)


def make_attestation(model_bytes, prompt_ids: Sequence[int], result: GenerationResult, bond: int,
                     challenge_period: int, device: int = 0) -> Attestation:
    """make_attestation (attest.cpp:68-78); the model id hashed on the GPU."""
    mb = _buf(model_bytes)
    p = np.ascontiguousarray(prompt_ids, np.uint32)
    oh = (C.c_uint8 * 32)(*result.output_hash)
    a = _CAtt()
    check(lib.dimg_make_attestation(device, mb.ctypes.data_as(C.c_void_p), mb.size,
                                    p.ctypes.data_as(C.POINTER(C.c_uint32)), p.size, oh, bond, challenge_period,
                                    C.byref(a)))
    return Attestation._from_c(a)


def _outcome(o: _COut) -> VerifyOutcome:
    if o.confirmed:
        return VerifyOutcome(True)
    return VerifyOutcome(False, _STAGES[o.refuted_stage], bytes(o.expected), bytes(o.found))


def verify_by_reexecution(att: Attestation, model_bytes, prompt_ids: Sequence[int], max_new: int,
                          opts: Optional[EngineOptions] = None) -> VerifyOutcome:
    """verify_by_reexecution (attest.cpp:89-117): ParseError for unparseable
    model bytes (after the model id matched), else a verdict."""
    opts = opts or EngineOptions()
    mb = _buf(model_bytes)
    p = np.ascontiguousarray(prompt_ids, np.uint32)
    a, o = att._c(), _COut()
    check(lib.dimg_verify_by_reexecution(opts.device, C.byref(a), mb.ctypes.data_as(C.c_void_p), mb.size,
                                         p.ctypes.data_as(C.POINTER(C.c_uint32)), p.size, max_new, C.byref(o)))
    return _outcome(o)


def dispute_game(att: Attestation, model_bytes, prompt_ids: Sequence[int], max_new: int,
                 opts: Optional[EngineOptions] = None) -> DisputeResult:
    """dispute_game (attest.cpp:119-125)."""
    opts = opts or EngineOptions()
    mb = _buf(model_bytes)
    p = np.ascontiguousarray(prompt_ids, np.uint32)
    a, o, w = att._c(), _COut(), C.c_uint32()
    check(lib.dimg_dispute_game(opts.device, C.byref(a), mb.ctypes.data_as(C.c_void_p), mb.size,
                                p.ctypes.data_as(C.POINTER(C.c_uint32)), p.size, max_new, C.byref(w), C.byref(o)))
    return DisputeResult("attester" if w.value == 0 else "challenger", _outcome(o))
