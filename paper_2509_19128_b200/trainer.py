"""Trainer step for the decoder policy: current-policy log-prob recompute,
truncated importance-weighted REINFORCE objective and its gradient on the
device (``srl_trainer_*``), plus the Adam update whose bf16 weights are the
in-flight update payload.

Semantics follow rlmath::is_reinforce_gradient
(/root/reference/proj/core/src/rl_math.cpp:211-276): ascent gradient of
J = (1/m) sum_traj sum_t w * (R - b_t) * log pi(y_t), stop-gradient on the
truncated weight w = min(c, exp(log pi - log mu)) taken per sequence
(default, rl_math.hpp:57-60) or per token.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .policy import DecoderPolicy

GRANULARITY = {"sequence": 0, "per_token": 1}


@dataclass
class TrainStep:
    objective: float
    ess: float
    clamped: int
    tokens: int
    forward_ms: float
    step_ms: float
    logprobs: list  # per trajectory, log pi of every token (index 0 = bos -> 0.0)


class Trainer:
    def __init__(self, policy: DecoderPolicy, max_tokens: int = 4096, device: int | None = None,
                 precise: bool = True, logit_chunk: int = 0):
        """precise (default): activations and backward operands as bf16 hi + lo
        pairs -- the 1e-3 parity mode; precise=False: single bf16 operands
        (faster, ~1e-2 gradient agreement).  logit_chunk: LM-head rows per pass
        (0 = 16384)."""
        if not isinstance(policy, DecoderPolicy):
            raise TypeError("Trainer needs a DecoderPolicy")
        self.config = policy.config
        self.device = policy.device if device is None else device
        self.precise = precise
        opts = _lib.TrainerOptionsC(max_tokens, self.device, 0 if precise else 1, logit_chunk)
        h = C.c_void_p()
        _lib.call("srl_trainer_create", policy.handle, C.byref(opts), C.byref(h))
        self._h = h

    def step(self, trajectories, n_trajectories: int | None = None, clamp: float = 5.0,
             granularity: str = "sequence") -> TrainStep:
        """trajectories: dicts with tokens (bos + prompt + generated), loss_begin
        (index of the first generated token), behavior_logprobs and advantages
        (one per token, entries before loss_begin ignored)."""
        toks = np.concatenate([np.asarray(t["tokens"], dtype=np.int32) for t in trajectories])
        offs = np.concatenate([[0], np.cumsum([len(t["tokens"]) for t in trajectories])]).astype(np.int64)
        lb = np.array([t["loss_begin"] for t in trajectories], dtype=np.int32)
        mu = np.concatenate([np.asarray(t["behavior_logprobs"], dtype=np.float64) for t in trajectories])
        adv = np.concatenate([np.asarray(t["advantages"], dtype=np.float64) for t in trajectories])
        out = np.zeros(len(toks), dtype=np.float64)
        stats = _lib.TrainerStatsC()
        m = len(trajectories) if n_trajectories is None else n_trajectories
        st = _lib.lib().srl_trainer_step(self._h, toks.ctypes.data, offs.ctypes.data, len(trajectories),
                                         lb.ctypes.data, mu.ctypes.data, adv.ctypes.data, m, clamp,
                                         GRANULARITY[granularity], out.ctypes.data, C.byref(stats))
        if st == 5:
            raise ValueError(_lib.lib().srl_last_error().decode())
        _lib.check(st, "srl_trainer_step")
        lps = [out[offs[i]:offs[i + 1]].tolist() for i in range(len(trajectories))]
        return TrainStep(stats.objective, stats.ess, stats.clamped, stats.tokens, stats.forward_ms,
                         stats.step_ms, lps)

    def step_data_parallel(self, trajectories, rank: int, world: int, group=None, **kw) -> TrainStep:
        """One data-parallel trainer step: this rank's shard of the consumed
        batch (weight_sync.shard), the objective normalised by the GLOBAL
        trajectory count, then the gradient all-reduce over the trainer group
        (weight_sync.GradientSync).  Every rank then applies the same Adam step."""
        from .weight_sync import GradientSync, shard

        res = self.step(shard(trajectories, rank, world), n_trajectories=len(trajectories), **kw)
        GradientSync(group).allreduce_(self.gradient())
        return res

    def gradient(self):
        """Zero-copy torch view (fp32, flat weight layout) of the last gradient."""
        import torch

        p, n = C.c_void_p(), C.c_size_t()
        _lib.call("srl_trainer_gradient", self._h, C.byref(p), C.byref(n))

        class _Arr:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f4",
                                        "data": (p.value, False), "version": 3}
        return torch.as_tensor(_Arr(), device=f"cuda:{self.device}")

    def apply_adam(self, lr: float, betas=(0.9, 0.999), eps: float = 1e-8):
        _lib.call("srl_trainer_apply_adam", self._h, lr, betas[0], betas[1], eps)

    def weights(self):
        """(device pointer, nbytes) of the bf16 weights -- the broadcast payload."""
        p, n = C.c_void_p(), C.c_size_t()
        _lib.call("srl_trainer_weights", self._h, C.byref(p), C.byref(n))
        return p.value, n.value

    def policy(self) -> DecoderPolicy:
        p, n = self.weights()
        return DecoderPolicy.from_buffer(self.config, p, n, True, self.device)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().srl_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
