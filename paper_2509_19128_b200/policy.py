"""Policy checkpoints: the reference ``rlmath::Policy`` variant
(/root/reference/proj/core/include/streamrl/policy.hpp:16-82) plus the
decoder policy this framework adds, all behind the ``streamrl.policy/1``
document schema (src/policy.cpp:136-206).

Tabular and recurrent policies are plain host data (numpy, fp64) that are
uploaded to the device when an engine or a trainer-math call uses them.  A
decoder policy owns a flat bf16 weight buffer on the GPU (``srl_policy``).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib

SCHEMA = "streamrl.policy/1"


@dataclass
class TabularPolicy:
    """TabularPolicy (policy.hpp:16-47): (prompt_id, context window) -> logits row."""

    vocab_size: int
    context_order: int = 0
    logits: dict = field(default_factory=dict)  # {(prompt_id, (ctx...)): np.ndarray[V]}
    default_logits: np.ndarray | None = None    # None/empty -> uniform fallback

    def rows(self):
        """Rows in std::map<ContextKey> order (prompt_id, then context)."""
        return sorted(self.logits.items(), key=lambda kv: (kv[0][0], tuple(kv[0][1])))


@dataclass
class RecurrentToyPolicy:
    """RecurrentToyPolicy (policy.hpp:52-72): h <- tanh(R h + E[tok]); logits = h^T O."""

    vocab_size: int
    hidden_dim: int
    input_embedding: np.ndarray  # [V x D] row-major (flat or 2-D)
    recurrence: np.ndarray       # [D x D]
    output: np.ndarray           # [D x V]


@dataclass(frozen=True)
class DecoderConfig:
    """Shape of the decoder policy (Qwen2.5 family)."""

    name: str
    vocab_size: int
    hidden: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    tie_embeddings: bool = True
    bos_token: int = 0
    max_positions: int = 8192
    rope_theta: float = 1_000_000.0
    rms_eps: float = 1e-6

    def native(self):
        return _lib.DecoderConfigC(self.vocab_size, self.hidden, self.layers, self.q_heads,
                                   self.kv_heads, self.head_dim, self.intermediate,
                                   int(self.tie_embeddings), self.bos_token, self.max_positions,
                                   self.rope_theta, self.rms_eps)

    def params(self) -> int:
        h, i, v = self.hidden, self.intermediate, self.vocab_size
        qkv = (self.q_heads + 2 * self.kv_heads) * self.head_dim
        per_layer = 2 * h + qkv * h + qkv + h * self.q_heads * self.head_dim + 3 * i * h
        return v * h * (1 if self.tie_embeddings else 2) + self.layers * per_layer + h

    def matmul_params(self) -> int:
        """Weights streamed by one decode step (all GEMM operands incl. LM head)."""
        h, i = self.hidden, self.intermediate
        qkv = (self.q_heads + 2 * self.kv_heads) * self.head_dim
        per_layer = qkv * h + h * self.q_heads * self.head_dim + 3 * i * h
        return self.layers * per_layer + self.vocab_size * h

    def to_dict(self):
        d = dict(self.__dict__)
        return d


# The builder-defined tiny config (BASELINE.json configs[0]) and the
# Qwen2.5 shapes of configs[1..4] (public architecture constants).
TINY = DecoderConfig("tiny", 256, 128, 2, 2, 1, 64, 512, True, 0, 4096, 10000.0, 1e-6)
QWEN25_05B = DecoderConfig("qwen2.5-0.5b", 151936, 896, 24, 14, 2, 64, 4864, True, 151643, 8192)
QWEN25_15B = DecoderConfig("qwen2.5-1.5b", 151936, 1536, 28, 12, 2, 128, 8960, True, 151643, 16384)
QWEN25_7B = DecoderConfig("qwen2.5-7b", 152064, 3584, 28, 28, 4, 128, 18944, False, 151643, 16384)
PRESETS = {c.name: c for c in (TINY, QWEN25_05B, QWEN25_15B, QWEN25_7B)}


class DecoderPolicy:
    """A decoder checkpoint: flat bf16 weights on the device (``srl_policy``)."""

    def __init__(self, config: DecoderConfig, handle, init: dict | None = None):
        self.config = config
        self._h = handle
        self.init = init or {}

    @classmethod
    def random(cls, config: DecoderConfig, seed: int = 0, scale: float = 0.02, device: int = 0):
        h = C.c_void_p()
        cfg = config.native()
        _lib.call("srl_policy_decoder_create", C.byref(cfg), seed, scale, device, C.byref(h))
        return cls(config, h, {"seed": seed, "scale": scale})

    @classmethod
    def from_buffer(cls, config: DecoderConfig, ptr: int, nbytes: int, on_device=True, device=0):
        h = C.c_void_p()
        cfg = config.native()
        _lib.call("srl_policy_decoder_from_buffer", C.byref(cfg), C.c_void_p(ptr), nbytes,
                  int(on_device), device, C.byref(h))
        return cls(config, h)

    @property
    def handle(self):
        return self._h

    def weights(self):
        """(device pointer, nbytes) of the flat bf16 buffer."""
        p, n = C.c_void_p(), C.c_size_t()
        _lib.call("srl_policy_decoder_weights", self._h, C.byref(p), C.byref(n))
        return p.value, n.value

    def offset(self, name: str) -> int:
        o = C.c_size_t()
        _lib.call("srl_policy_decoder_offset", self._h, name.encode(), C.byref(o))
        return o.value

    def perturb(self, seed: int, magnitude: float):
        _lib.call("srl_policy_decoder_perturb", self._h, seed, magnitude)
        return self

    @property
    def device(self) -> int:
        """CUDA device index of the weights."""
        d = C.c_int32()
        _lib.call("srl_policy_decoder_device", self._h, C.byref(d))
        return d.value

    def clone(self, device: int | None = None):
        """A copy on `device` (default: this policy's device)."""
        p, n = self.weights()
        return DecoderPolicy.from_buffer(self.config, p, n, True,
                                         self.device if device is None else device)

    def torch_weights(self):
        """Zero-copy torch view (uint16 -> bf16) of the flat weight buffer."""
        import torch

        p, n = self.weights()

        class _Arr:
            __cuda_array_interface__ = {"shape": (n // 2,), "typestr": "<u2", "data": (p, False),
                                        "version": 3}

            def __init__(self, owner):
                self.owner = owner  # the tensor keeps _Arr alive, _Arr keeps the buffer's owner alive

        return torch.as_tensor(_Arr(self), device=f"cuda:{self.device}").view(torch.bfloat16)

    def __del__(self):
        try:
            if self._h:
                _lib.lib().srl_policy_destroy(self._h)
                self._h = None
        except Exception:
            pass


Policy = TabularPolicy | RecurrentToyPolicy | DecoderPolicy


def vocab_size_of(policy) -> int:
    if isinstance(policy, DecoderPolicy):
        return policy.config.vocab_size
    return policy.vocab_size


# ----------------------------------------------------------- native handles
class NativePolicy:
    """Temporary ``srl_policy`` for a host (tabular / recurrent) policy."""

    def __init__(self, policy):
        self.owned = not isinstance(policy, DecoderPolicy)
        if not self.owned:
            self.h = policy.handle
            return
        h = C.c_void_p()
        if isinstance(policy, RecurrentToyPolicy):
            e = np.ascontiguousarray(policy.input_embedding, dtype=np.float64).ravel()
            r = np.ascontiguousarray(policy.recurrence, dtype=np.float64).ravel()
            o = np.ascontiguousarray(policy.output, dtype=np.float64).ravel()
            self._keep = (e, r, o)
            _lib.call("srl_policy_recurrent_create", policy.vocab_size, policy.hidden_dim,
                      e.ctypes.data, r.ctypes.data, o.ctypes.data, C.byref(h))
        else:
            rows = policy.rows()
            V, order = policy.vocab_size, policy.context_order
            n = len(rows)
            ids = (C.c_char_p * max(n, 1))(*[k[0].encode() for k, _ in rows])
            lens = np.array([len(k[1]) for k, _ in rows] or [0], dtype=np.int32)
            width = max(order, 1)
            ctx = np.zeros((max(n, 1), width), dtype=np.int32)
            for i, (k, _) in enumerate(rows):
                c = list(k[1])[:width]
                ctx[i, :len(c)] = c
            lg = np.ascontiguousarray(np.array([np.asarray(v, dtype=np.float64) for _, v in rows]
                                               or [np.zeros(max(V, 1))], dtype=np.float64)).ravel()
            d = policy.default_logits
            dptr = None
            if d is not None and len(d):
                d = np.ascontiguousarray(d, dtype=np.float64)
                dptr = d.ctypes.data
            self._keep = (ids, lens, ctx, lg, d)
            _lib.call("srl_policy_tabular_create", V, order, dptr, n, ids, lens.ctypes.data,
                      ctx.ctypes.data, lg.ctypes.data, C.byref(h))
        self.h = h

    def __enter__(self):
        return self.h

    def __exit__(self, *exc):
        self.close()

    def close(self):
        if self.owned and self.h:
            _lib.lib().srl_policy_destroy(self.h)
            self.h = None


# ---------------------------------------------------------- JSON documents
def _row_list(a):
    return [float(x) for x in np.asarray(a, dtype=np.float64).ravel()]


def policy_to_dict(policy) -> dict:
    if isinstance(policy, TabularPolicy):
        rows = [{"prompt_id": k[0], "context": list(k[1]), "logits": _row_list(v)}
                for k, v in policy.rows()]
        d = policy.default_logits
        return {"schema": SCHEMA, "type": "tabular", "vocab_size": policy.vocab_size,
                "context_order": policy.context_order,
                "default_logits": [] if d is None else _row_list(d), "rows": rows}
    if isinstance(policy, RecurrentToyPolicy):
        return {"schema": SCHEMA, "type": "recurrent", "vocab_size": policy.vocab_size,
                "hidden_dim": policy.hidden_dim,
                "input_embedding": _row_list(policy.input_embedding),
                "recurrence": _row_list(policy.recurrence), "output": _row_list(policy.output)}
    if isinstance(policy, DecoderPolicy):
        return {"schema": SCHEMA, "type": "decoder", "config": policy.config.to_dict(),
                "init": policy.init}
    raise TypeError(type(policy))


def policy_to_json(policy) -> str:
    return json.dumps(policy_to_dict(policy), indent=2)


def policy_from_dict(doc: dict):
    """policy_from_json (policy.cpp:163-192) plus the decoder type."""
    if doc.get("schema") != SCHEMA:
        raise ValueError("policy document: unknown schema id")
    t = doc["type"]
    if t == "tabular":
        logits = {}
        for row in doc.get("rows", []):
            logits[(row["prompt_id"], tuple(int(x) for x in row["context"]))] = np.array(
                row["logits"], dtype=np.float64)
        d = doc.get("default_logits", [])
        return TabularPolicy(int(doc["vocab_size"]), int(doc["context_order"]), logits,
                             np.array(d, dtype=np.float64) if len(d) else None)
    if t == "recurrent":
        V, D = int(doc["vocab_size"]), int(doc["hidden_dim"])
        return RecurrentToyPolicy(V, D, np.array(doc["input_embedding"], dtype=np.float64),
                                  np.array(doc["recurrence"], dtype=np.float64),
                                  np.array(doc["output"], dtype=np.float64))
    if t == "decoder":
        cfg = DecoderConfig(**doc["config"])
        init = doc.get("init", {})
        return DecoderPolicy.random(cfg, int(init.get("seed", 0)), float(init.get("scale", 0.02)))
    raise ValueError("policy document: unknown type " + t)


def policy_from_json(text: str):
    return policy_from_dict(json.loads(text))


def validate(policy) -> None:
    """Raises SrlError(invalid_policy) like rlmath::validate."""
    with NativePolicy(policy) as h:
        _lib.call("srl_policy_validate", h)
