"""B200-native integer transformer engine (the hot path of arXiv 2603.24904's
ARC engine, as re-created by the reference `dim`).

Public API mirrors proj/include/dim/{engine,model}.hpp; everything executes in
libdimg.so (sm_100a kernels + C++ host library) through include/dimg.h.
"""
from . import attest, errors
from .attest import (Attestation, DisputeResult, VerifyOutcome, dispute_game, make_attestation, prompt_hash,
                     verify_by_reexecution)
from ._lib import LIB_PATH, lib
from .engine import (EngineOptions, GenerationResult, InferenceSession, attention_steps, blake3_device,
                     blake3_gpu, build_rope_tables, generate_sampled, sample_from_logits, sample_key, dense_forward, dense_tokens, device_count, ffn_silu, generate_greedy,
                     generate_greedy_batch, generation_counter, hash_token_ids, parse_prompt, prompt_from_seed,
                     release_sessions, rmsnorm, select_greedy, softmax_q16, RopeTables, serialize_rope_tables,
                     deserialize_rope_tables, save_rope_tables, load_rope_tables)
from .errors import (ContextOverflow, DomainError, InvalidArgument, LengthError, LogicError,
                     OutOfRange, ParseError)
from .parallel import TensorParallel, nccl_unique_id
from .model import (ONE, DeviceModel, ModelConfig, ModelFile, deserialize, gen_toy_model,
                    load_model, weight_hash)

__all__ = [
    "EngineOptions", "GenerationResult", "InferenceSession", "generate_greedy", "generate_greedy_batch",
    "generation_counter", "hash_token_ids", "select_greedy", "parse_prompt", "prompt_from_seed",
    "build_rope_tables", "blake3_device", "blake3_gpu", "generate_sampled", "sample_from_logits", "sample_key", "dense_forward", "dense_tokens", "rmsnorm", "softmax_q16", "attention_steps", "ffn_silu",
    "device_count", "release_sessions", "ModelConfig", "ModelFile", "DeviceModel",
    "gen_toy_model", "deserialize", "load_model", "weight_hash", "ONE", "errors",
    "ContextOverflow", "DomainError", "InvalidArgument", "LengthError", "LogicError",
    "OutOfRange", "ParseError", "LIB_PATH", "lib", "attest", "Attestation", "VerifyOutcome", "DisputeResult",
    "make_attestation", "verify_by_reexecution", "dispute_game", "prompt_hash",
    "TensorParallel", "nccl_unique_id", "RopeTables", "serialize_rope_tables", "deserialize_rope_tables", "save_rope_tables", "load_rope_tables",
]
