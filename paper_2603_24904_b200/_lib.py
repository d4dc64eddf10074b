"""ctypes binding of include/dimg.h (libdimg.so, built in-tree).

The library is the product: sm_100a kernels plus the C++ host half. If it is
missing, importing this module raises -- there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# DIMG_LIB: an instrumented experiment build (tools/); the product is libdimg.so
LIB_PATH = os.environ.get("DIMG_LIB") or os.path.join(HERE, "libdimg.so")

u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
i64p = C.POINTER(C.c_int64)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class Config(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("d_model", C.c_uint32), ("n_heads", C.c_uint32),
                ("d_ffn", C.c_uint32), ("vocab", C.c_uint32), ("max_ctx", C.c_uint32),
                ("rope_theta", C.c_double)]


class QTensor(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("data", i8p), ("scales", i64p)]


class ModelDesc(C.Structure):
    _fields_ = [("cfg", Config), ("tok_embd", QTensor), ("output", QTensor),
                ("layers", C.POINTER(QTensor)), ("norms", i64p), ("rope_cos", i64p),
                ("rope_sin", i64p), ("rope_max_ctx", C.c_uint32)]


class Attestation(C.Structure):
    _fields_ = [("model_id", C.c_uint8 * 32), ("input_hash", C.c_uint8 * 32), ("output_hash", C.c_uint8 * 32),
                ("bond", C.c_uint64), ("challenge_period", C.c_uint64)]


class VerifyOutcome(C.Structure):
    _fields_ = [("confirmed", C.c_uint32), ("refuted_stage", C.c_uint32), ("expected", C.c_uint8 * 32),
                ("found", C.c_uint8 * 32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2603_24904_b200/csrc` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    pp = C.POINTER(C.c_void_p)
    sigs = {
        "dimg_last_error": ([], C.c_char_p),
        "dimg_last_parse_kind": ([], C.c_int),
        "dimg_version": ([], C.c_char_p),
        "dimg_config_validate": ([C.POINTER(Config)], C.c_int),
        "dimg_blake3": ([vp, C.c_size_t, u8p], C.c_int),
        "dimg_hash_token_ids": ([u32p, C.c_size_t, u8p], C.c_int),
        "dimg_select_greedy": ([i64p, C.c_size_t, u32p], C.c_int),
        "dimg_prompt_from_seed": ([C.c_uint64, C.c_uint32, C.c_uint32, u32p], C.c_int),
        "dimg_parse_prompt": ([C.c_char_p, C.c_char_p, u32p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "dimg_rope_tables": ([C.c_double, C.c_uint32, C.c_uint32, i64p, i64p], C.c_int),
        "dimg_rtab_serialize": ([C.c_double, C.c_uint32, C.c_uint32, i64p, i64p, u8p, C.c_size_t,
                                 C.POINTER(C.c_size_t)], C.c_int),
        "dimg_rtab_deserialize": ([u8p, C.c_size_t, u32p, u32p, C.POINTER(C.c_double), i64p, i64p, C.c_size_t],
                                  C.c_int),
        "dimg_rtab_save": ([C.c_char_p, C.c_double, C.c_uint32, C.c_uint32, i64p, i64p], C.c_int),
        "dimg_rtab_load": ([C.c_char_p, u8p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "dimg_exp_lut": ([i64p], C.c_int),
        "dimg_invsqrt_seeds": ([i64p], C.c_int),
        "dimg_host_model_gen_toy": ([C.c_uint64, C.POINTER(Config), C.c_int, pp], C.c_int),
        "dimg_host_model_gen_toy_gpu": ([C.c_int, C.c_uint64, C.POINTER(Config), pp], C.c_int),
        "dimg_host_model_from_bytes": ([u8p, C.c_size_t, pp], C.c_int),
        "dimg_host_model_load": ([C.c_char_p, pp], C.c_int),
        "dimg_host_model_save": ([vp, C.c_char_p], C.c_int),
        "dimg_host_model_from_desc": ([C.POINTER(ModelDesc), pp], C.c_int),
        "dimg_host_model_bytes": ([vp, C.POINTER(u8p), C.POINTER(C.c_size_t)], C.c_int),
        "dimg_host_model_weight_hash": ([vp, u8p], C.c_int),
        "dimg_host_model_desc": ([vp, C.POINTER(ModelDesc)], C.c_int),
        "dimg_host_model_free": ([vp], C.c_int),
        "dimg_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "dimg_model_upload": ([C.c_int, C.POINTER(ModelDesc), C.c_int, C.c_int, pp], C.c_int),
        "dimg_model_free": ([vp], C.c_int),
        "dimg_model_bytes_on_device": ([vp, u64p], C.c_int),
        "dimg_session_create": ([vp, C.c_uint32, pp], C.c_int),
        "dimg_session_free": ([vp], C.c_int),
        "dimg_session_reset": ([vp], C.c_int),
        "dimg_session_len": ([vp, u32p], C.c_int),
        "dimg_session_forward": ([vp, C.c_uint32, C.c_uint32, i64p], C.c_int),
        "dimg_generate_greedy": ([vp, u32p, C.c_uint32, C.c_uint32, u32p, u8p, i64p], C.c_int),
        "dimg_generate_greedy_batch": ([vp, C.c_uint32, u32p, u32p, C.c_uint32, u32p, u8p, u32p], C.c_int),
        "dimg_session_begin": ([vp, u32p, C.c_uint32, C.c_uint32], C.c_int),
        "dimg_session_prefill": ([vp], C.c_int),
        "dimg_session_decode": ([vp, C.c_uint32], C.c_int),
        "dimg_session_sync": ([vp], C.c_int),
        "dimg_session_tokens": ([vp, u32p, C.c_uint32], C.c_int),
        "dimg_session_stream": ([vp, pp], C.c_int),
        "dimg_session_time_decode": ([vp, C.c_uint32, C.POINTER(C.c_float)], C.c_int),
        "dimg_session_time_prefill": ([vp, C.POINTER(C.c_float), C.POINTER(C.c_uint32)], C.c_int),
        "dimg_session_launches": ([vp, u32p, u32p], C.c_int),
        "dimg_session_time_kernel": ([vp, C.c_int, C.c_uint32, C.POINTER(C.c_float), u64p], C.c_int),
        "dimg_session_stats": ([vp, u64p], C.c_int),
        "dimg_session_trace": ([vp, C.c_uint32, u64p, C.c_uint32], C.c_int),
        "dimg_session_trace_all": ([vp, C.c_uint32, u64p, C.c_uint32], C.c_int),
        "dimg_nccl_unique_id": ([u8p], C.c_int),
        "dimg_tp_create": ([C.c_int, C.POINTER(ModelDesc), C.c_int, C.c_int, C.c_int, u8p, C.c_uint32, pp],
                           C.c_int),
        "dimg_tp_free": ([vp], C.c_int),
        "dimg_tp_generate_greedy": ([vp, u32p, C.c_uint32, C.c_uint32, u32p, u8p, i64p], C.c_int),
        "dimg_tp_time_decode": ([vp, u32p, C.c_uint32, C.c_uint32, C.POINTER(C.c_float)], C.c_int),
        "dimg_tp_tokens": ([vp, u32p, C.c_uint32], C.c_int),
        "dimg_tp_stream": ([vp, pp], C.c_int),
        "dimg_tp_info": ([vp, u64p, u64p], C.c_int),
        "dimg_tp_exchange_handle": ([vp, u8p], C.c_int),
        "dimg_inv_sqrt_q16": ([C.c_int64, i64p], C.c_int),
        "dimg_tp_connect": ([vp, u8p], C.c_int),
        "dimg_op_dense": ([C.c_int, C.POINTER(QTensor), i64p, i64p], C.c_int),
        "dimg_op_dense_tokens": ([C.c_int, C.POINTER(QTensor), i64p, C.c_uint32, i64p], C.c_int),
        "dimg_blake3_device": ([C.c_int, vp, C.c_size_t, u8p, C.POINTER(C.c_float)], C.c_int),
        "dimg_blake3_gpu": ([C.c_int, vp, C.c_size_t, u8p], C.c_int),
        "dimg_attestation_encode": ([C.POINTER(Attestation), u8p], C.c_int),
        "dimg_attestation_decode": ([u8p, C.c_size_t, C.POINTER(Attestation)], C.c_int),
        "dimg_attestation_text": ([C.POINTER(Attestation), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
        "dimg_make_attestation": ([C.c_int, vp, C.c_size_t, u32p, C.c_size_t, u8p, C.c_uint64, C.c_uint64,
                                   C.POINTER(Attestation)], C.c_int),
        "dimg_verify_by_reexecution": ([C.c_int, C.POINTER(Attestation), vp, C.c_size_t, u32p, C.c_size_t,
                                        C.c_uint32, C.POINTER(VerifyOutcome)], C.c_int),
        "dimg_dispute_game": ([C.c_int, C.POINTER(Attestation), vp, C.c_size_t, u32p, C.c_size_t, C.c_uint32,
                               u32p, C.POINTER(VerifyOutcome)], C.c_int),
        "dimg_generation_counter": ([u64p], C.c_int),
        "dimg_sample_key": ([C.c_int, u8p, C.c_size_t, u32p, C.c_size_t, u8p], C.c_int),
        "dimg_generate_sampled": ([vp, u32p, C.c_uint32, C.c_uint32, C.c_int64, u8p, u32p, u8p], C.c_int),
        "dimg_op_sample": ([C.c_int, i64p, C.c_uint32, C.c_int64, C.c_uint32, u32p], C.c_int),
        "dimg_op_rmsnorm": ([C.c_int, i64p, i64p, C.c_uint32, i64p], C.c_int),
        "dimg_op_softmax": ([C.c_int, i64p, C.c_uint32, i64p], C.c_int),
        "dimg_op_attention": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint32,
                               i64p, i64p, i64p, i64p], C.c_int),
        "dimg_op_ffn": ([C.c_int, C.POINTER(QTensor), C.POINTER(QTensor), C.POINTER(QTensor),
                         i64p, i64p], C.c_int),
    }
    for name, (args, res) in sigs.items():
        if os.environ.get("DIMG_LIB") and not hasattr(lib, name):
            continue  # an older experiment build (tools/ab_decode.py); the product library has every symbol
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib, list(sigs)


lib, EXPORTED = _load()


def check(rc: int):
    """Raises the Python mirror of the reference exception for a status."""
    if rc != 0:
        msg = (lib.dimg_last_error() or b"").decode(errors="replace")
        raise errors.from_status(rc, msg, lib.dimg_last_parse_kind())


def ptr(a, t):
    return a.ctypes.data_as(t)
