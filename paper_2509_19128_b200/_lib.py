"""ctypes binding of ``libsrl_b200.so`` (the C ABI in include/streamrl_b200.h).

There is deliberately no fallback: if the shared library is missing or a
symbol is absent this module raises at import/first use, and every compute
entry point returns SRL_NO_DEVICE / SRL_CUDA_ERROR without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libsrl_b200.so"
HEADER = HERE.parent / "include" / "streamrl_b200.h"

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
P = C.POINTER

STATUS = {}


class SrlError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.error = _error_string(status)
        super().__init__(f"{self.error} ({status}) {what}".strip())


_lib = None


def _error_string(status: int) -> str:
    return lib().srl_status_string(status).decode()



class DecoderConfigC(C.Structure):
    _fields_ = [("vocab_size", i32), ("hidden", i32), ("layers", i32), ("q_heads", i32),
                ("kv_heads", i32), ("head_dim", i32), ("intermediate", i32),
                ("tie_embeddings", i32), ("bos_token", i32), ("max_positions", i32),
                ("rope_theta", f64), ("rms_eps", f64)]


class EngineOptionsC(C.Structure):
    _fields_ = [("max_streams", i32), ("max_seq_len", i32), ("greedy", i32),
                ("rounds_per_sync", i32), ("use_graphs", i32), ("device", i32),
                ("event_ring", i32), ("prefill_budget", i32), ("precise", i32)]


class TokenEventC(C.Structure):
    _fields_ = [("stream", i64), ("position", i32), ("token", i32), ("logprob", f64),
                ("weight_version", i32), ("reserved", i32)]


class EngineStatsC(C.Structure):
    _fields_ = [("rounds", i64), ("tokens", i64), ("updates", i64), ("decode_ms", f64),
                ("last_pause_ms", f64), ("max_pause_ms", f64), ("launches", i64),
                ("prefill_rounds", i64), ("prefill_rows", i64), ("prefill_ms", f64)]


class TrainerOptionsC(C.Structure):
    _fields_ = [("max_tokens", i32), ("device", i32), ("fast_bf16", i32), ("logit_chunk", i32)]


class TrainerStatsC(C.Structure):
    _fields_ = [("objective", f64), ("ess", f64), ("clamped", i32), ("tokens", i32),
                ("forward_ms", f64), ("step_ms", f64)]


class KernelProfileC(C.Structure):
    _fields_ = [("ms", f64 * 10), ("launches", i32 * 10), ("valid", i32), ("rows", i32),
                ("fused", i32), ("fused_ms", f64)]


KERNEL_CLASSES = ["plan", "embed", "qkv_gemm", "rope_kv_append", "attention", "o_gemm",
                  "gate_up_gemm", "down_gemm", "lm_head_gemm", "sample"]


I = C.c_int
# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "srl_status_string": (cp, [I]),
    "srl_last_error": (cp, []),
    "srl_kernel_gemm_mn": (I, [vp, vp, i32, i32, i32, i32, i32, i32, f32, vp, vp]),
    "srl_kernel_gemm_bf16": (I, [vp, vp, i32, i32, i32, i32, i32, vp, vp, i32, f32, f32,
                                 vp, vp, vp, vp, vp, vp]),
    "srl_policy_tabular_create": (I, [i32, i32, vp, i32, P(cp), vp, vp, vp, P(vp)]),
    "srl_policy_recurrent_create": (I, [i32, i32, vp, vp, vp, P(vp)]),
    "srl_policy_decoder_create": (I, [P(DecoderConfigC), u64, f64, i32, P(vp)]),
    "srl_policy_decoder_from_buffer": (I, [P(DecoderConfigC), vp, sz, i32, i32, P(vp)]),
    "srl_decoder_weight_bytes": (sz, [P(DecoderConfigC)]),
    "srl_policy_decoder_weights": (I, [vp, P(vp), P(sz)]),
    "srl_policy_decoder_device": (I, [vp, P(i32)]),
    "srl_policy_decoder_offset": (I, [vp, cp, P(sz)]),
    "srl_policy_decoder_perturb": (I, [vp, u64, f64]),
    "srl_policy_type": (I, [vp]),
    "srl_policy_vocab_size": (i32, [vp]),
    "srl_policy_validate": (I, [vp]),
    "srl_policy_destroy": (None, [vp]),
    "srl_engine_create": (I, [vp, i32, i32, P(EngineOptionsC), P(vp)]),
    "srl_engine_destroy": (None, [vp]),
    "srl_engine_open_stream": (I, [vp, cp, i32, u64, i32, vp, i32, P(i64)]),
    "srl_engine_wait_events": (I, [vp, i64, P(TokenEventC), i32, P(i32), P(i32), P(i32)]),
    "srl_engine_wait_events_many": (I, [vp, vp, i32, P(TokenEventC), i32, vp, vp, vp]),
    "srl_engine_poll_events_many": (I, [vp, vp, i32, P(TokenEventC), i32, vp, vp, vp]),
    "srl_engine_apply_weight_update": (I, [vp, i32, vp, P(i32)]),
    "srl_engine_begin_weight_update": (I, [vp, i32, P(vp), P(sz)]),
    "srl_engine_commit_weight_update": (I, [vp, i32, P(i32), P(f64)]),
    "srl_engine_abort_weight_update": (I, [vp]),
    "srl_engine_standby_bytes": (I, [vp, P(sz)]),
    "srl_engine_advance": (I, [vp, i32, P(i64)]),
    "srl_engine_pause": (I, [vp]),
    "srl_engine_resume": (I, [vp]),
    "srl_engine_weight_version": (I, [vp, P(i32)]),
    "srl_engine_active_streams": (I, [vp, P(i32)]),
    "srl_engine_total_streams": (I, [vp, P(i64)]),
    "srl_engine_rounds_done": (I, [vp, P(i64)]),
    "srl_engine_recompute_state_mode": (I, [vp, P(i32)]),
    "srl_engine_set_process_group": (I, [vp, cp, P(cp), i32]),
    "srl_engine_process_group_id": (I, [vp, cp, sz, P(i32)]),
    "srl_engine_stop": (I, [vp]),
    "srl_engine_stream_tokens": (I, [vp, i64, vp, i32, P(i32)]),
    "srl_engine_stats_get": (I, [vp, P(EngineStatsC)]),
    "srl_policy_logprobs": (I, [vp, cp, vp, i32, vp]),
    "srl_truncated_is_weight": (I, [f64, f64, f64, P(f64)]),
    "srl_ess": (I, [vp, i32, P(f64)]),
    "srl_decoder_kl_per_position": (I, [vp, i32, vp, i32, i32, vp, vp, vp, i32, vp, i32]),
    "srl_tabular_is_reinforce_gradient": (I, [vp, i32, P(cp), vp, vp, vp, vp, vp, i32, f64, i32, vp, vp]),
    "srl_lag_stats": (I, [vp, vp, i32, i32, vp, i32, vp, vp, vp]),
    "srl_crc32": (C.c_uint32, [vp, sz]),
    "srl_process_group_id": (I, [P(cp), i32, cp, sz]),
    "srl_kernel_attention_decode": (I, [vp, vp, vp, vp, i32, vp, vp, i32, i32, i32, i32, i32, vp, vp]),
    "srl_kernel_attention_prefill": (I, [vp, vp, vp, vp, i32, vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, vp,
                                         i32, vp]),
    "srl_device_copy_async": (I, [vp, vp, sz, vp]),
    "srl_kernel_sample_logits": (I, [vp, i32, i32, vp, vp, i32, vp, vp, vp]),
    "srl_engine_profile_next_round": (I, [vp]),
    "srl_trainer_create": (I, [vp, P(TrainerOptionsC), P(vp)]),
    "srl_trainer_destroy": (None, [vp]),
    "srl_trainer_step": (I, [vp, vp, vp, i32, vp, vp, vp, i32, f64, i32, vp, P(TrainerStatsC)]),
    "srl_trainer_gradient": (I, [vp, P(vp), P(sz)]),
    "srl_trainer_apply_adam": (I, [vp, f64, f64, f64, f64]),
    "srl_trainer_weights": (I, [vp, P(vp), P(sz)]),
    "srl_engine_kernel_profile": (I, [vp, P(KernelProfileC)]),
    "srl_comm_unique_id": (I, [vp]),
    "srl_comm_init": (I, [vp, i32, i32, i32, P(vp)]),
    "srl_comm_destroy": (None, [vp]),
    "srl_comm_size": (I, [vp, P(i32), P(i32)]),
    "srl_comm_broadcast_bytes": (I, [vp, i32, vp, sz]),
    "srl_comm_send_weights": (I, [vp, vp]),
    "srl_comm_recv_weights_begin": (I, [vp, i32, vp, i32, P(i32)]),
    "srl_comm_recv_weights_finish": (I, [vp, vp, i32, P(i32), P(i32), P(f64), P(f64)]),
    "srl_comm_wait": (I, [vp, P(f64)]),
    "srl_comm_allreduce_gradient": (I, [vp, vp]),
}


def declared_symbols() -> list[str]:
    """Every function name declared in include/streamrl_b200.h."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srl_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        detail = lib().srl_last_error().decode()
        raise SrlError(status, (what + " " + detail).strip())


def call(name: str, *args):
    """Call an entry point that returns srl_status; raise SrlError on failure."""
    st = getattr(lib(), name)(*args)
    check(st, name)
    return st
