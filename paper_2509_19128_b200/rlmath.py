"""Trainer math: the ``streamrl::rlmath`` free functions
(/root/reference/proj/core/include/streamrl/rl_math.hpp:20-121) over the
native library.  Same names, argument meaning and exceptions: ValueError for
std::invalid_argument, EssUndefinedError for the all-zero ESS case.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .policy import NativePolicy


class EssUndefinedError(ValueError):
    """EssUndefinedError (rl_math.hpp:30-32)."""


def _check(st: int, what: str):
    if st == 0:
        return
    detail = _lib.lib().srl_last_error().decode()
    if st in (5, 2):
        raise ValueError(f"{what}: {detail}")
    if st == 8:
        raise EssUndefinedError(detail)
    raise _lib.SrlError(st, f"{what}: {detail}")


def policy_logprobs(policy, prompt_id: str, tokens) -> np.ndarray:
    """log pi(y_t | x, y_<t) for every position (rl_math.cpp:128-142), on the device."""
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    out = np.zeros(len(t), dtype=np.float64)
    with NativePolicy(policy) as h:
        st = _lib.lib().srl_policy_logprobs(h, prompt_id.encode(), t.ctypes.data, len(t),
                                            out.ctypes.data)
    _check(st, "policy_logprobs")
    return out


def truncated_is_weight(pi_logprob_sum: float, mu_logprob_sum: float, clamp: float) -> float:
    """min(c, exp(pi - mu)) (rl_math.cpp:144-150)."""
    out = C.c_double()
    _check(_lib.lib().srl_truncated_is_weight(pi_logprob_sum, mu_logprob_sum, clamp, C.byref(out)),
           "truncated_is_weight")
    return out.value


def ess(weights) -> float:
    """(sum w)^2 / (N sum w^2) (rl_math.cpp:152-163)."""
    a = np.ascontiguousarray(weights, dtype=np.float64)
    out = C.c_double()
    _check(_lib.lib().srl_ess(a.ctypes.data if len(a) else None, len(a), C.byref(out)), "ess")
    return out.value


@dataclass
class Trajectory:
    """Trajectory (trajectory.hpp:15-25)."""

    prompt_id: str
    tokens: list
    behavior_logprobs: list
    behavior_versions: list
    reward: float = 0.0

    def validate(self):  # trajectory.cpp:14-25
        n = len(self.tokens)
        if n < 1:
            raise ValueError("Trajectory: empty token sequence")
        if len(self.behavior_logprobs) != n or len(self.behavior_versions) != n:
            raise ValueError("Trajectory: field lengths differ")
        if any(b < a for a, b in zip(self.behavior_versions, self.behavior_versions[1:])):
            raise ValueError("Trajectory: behavior_versions decrease")
        if any(np.isnan(self.behavior_logprobs)):
            raise ValueError("Trajectory: NaN behavior logprob")
        if not np.isfinite(self.reward):
            raise ValueError("Trajectory: non-finite reward")

    def length(self) -> int:
        return len(self.tokens)

    def behavior_logprob_sum(self) -> float:
        s = 0.0
        for v in self.behavior_logprobs:
            s += v
        return s


@dataclass
class BaselineTable:
    """Per-(prompt, position) mean reward (trajectory.hpp:29-35)."""

    values: dict = field(default_factory=dict)

    def at(self, prompt_id: str, position: int) -> float:
        try:
            return self.values[(prompt_id, position)]
        except KeyError:
            raise ValueError(f"BaselineTable: missing cell ({prompt_id}, {position})") from None


def fit_baseline(trajectories) -> BaselineTable:
    """fit_baseline (rl_math.cpp:165-179): exact per-cell mean (host-side actor queue logic)."""
    if not trajectories:
        raise ValueError("fit_baseline: no trajectories")
    cells: dict = {}
    for t in trajectories:
        t.validate()
        for p in range(t.length()):
            s, n = cells.get((t.prompt_id, p), (0.0, 0))
            cells[(t.prompt_id, p)] = (s + t.reward, n + 1)
    return BaselineTable({k: s / n for k, (s, n) in cells.items()})


@dataclass
class GradientTable:
    """GradientTable (rl_math.hpp:39-46): rows keyed by (prompt_id, context
    tuple); contributions through the fallback row land in default_row."""

    rows: dict = field(default_factory=dict)
    default_row: np.ndarray | None = None

    def max_abs(self) -> float:
        m = 0.0
        for r in self.rows.values():
            m = max(m, float(np.abs(r).max(initial=0.0)))
        if self.default_row is not None:
            m = max(m, float(np.abs(self.default_row).max(initial=0.0)))
        return m


def _tabular_gradient(policy, trajectories, baseline, clamp, use_is, granularity):
    from .policy import TabularPolicy

    if not isinstance(policy, TabularPolicy):
        raise TypeError("is_reinforce_gradient needs a TabularPolicy")
    if not trajectories:
        raise ValueError("reinforce_gradient: no trajectories")
    for t in trajectories:
        t.validate()
    toks = np.concatenate([np.asarray(t.tokens, dtype=np.int32) for t in trajectories])
    offs = np.concatenate([[0], np.cumsum([t.length() for t in trajectories])]).astype(np.int64)
    mu = np.concatenate([np.asarray(t.behavior_logprobs, dtype=np.float64) for t in trajectories])
    rew = np.array([t.reward for t in trajectories], dtype=np.float64)
    base = np.array([baseline.at(t.prompt_id, p) for t in trajectories for p in range(t.length())],
                    dtype=np.float64)  # BaselineTable::at throws on a missing cell
    ids = (C.c_char_p * len(trajectories))(*[t.prompt_id.encode() for t in trajectories])
    keys = sorted(k for k, _ in policy.rows())  # std::map<ContextKey> order
    V = policy.vocab_size
    grad = np.zeros((len(keys) + 1, V))
    touched = np.zeros(len(keys) + 1, dtype=np.int32)
    with NativePolicy(policy) as h:
        st = _lib.lib().srl_tabular_is_reinforce_gradient(
            h, len(trajectories), ids, toks.ctypes.data, offs.ctypes.data, mu.ctypes.data,
            rew.ctypes.data, base.ctypes.data, 1 if use_is else 0, float(clamp),
            1 if granularity in (1, "per_token") else 0, grad.ctypes.data, touched.ctypes.data)
    _check(st, "is_reinforce_gradient")
    out = GradientTable({k: grad[i] for i, k in enumerate(keys) if touched[i]},
                        grad[-1] if touched[-1] else None)
    return out


def reinforce_gradient(policy, trajectories, baseline) -> GradientTable:
    """reinforce_gradient (rl_math.cpp:264-269) for a TabularPolicy, on the device."""
    return _tabular_gradient(policy, trajectories, baseline, 1.0, False, 0)


def is_reinforce_gradient(policy, trajectories, baseline, clamp: float,
                          granularity="sequence") -> GradientTable:
    """is_reinforce_gradient (rl_math.cpp:271-276) for a TabularPolicy, on the
    device: (1/m) w (R - b_t) (onehot(y_t) - softmax(row)), stop-gradient on
    the truncated IS weight w (per sequence by default, or per token)."""
    return _tabular_gradient(policy, trajectories, baseline, clamp, True, granularity)


def mixed_schedule(max_len: int, max_lag: int) -> list:
    """MixedPolicySchedule::make switch points (rl_math.cpp:286-301): the first
    segment 2L/g long (the warm-up bubble), then every L/g tokens."""
    if max_len < 1:
        raise ValueError("schedule: max_len must be positive")
    if max_lag < 1:
        raise ValueError("schedule: max_lag must be positive")
    first, step = (2 * max_len) // max_lag, max_len // max_lag
    pts, t = [], first
    while t < max_len and len(pts) < max_lag:
        pts.append(t)
        if step == 0:
            break
        t += step
    return pts


def kl_per_position(checkpoints, switch_points, recompute_state: bool, target, prefixes) -> np.ndarray:
    """kl_per_position (rl_math.cpp:336-372) for decoder policies, on the
    device: mean exact KL(behaviour || target) per position over the token
    prefixes; the behaviour switches checkpoint at switch_points with a stale
    (PipelineRL) or recomputed KV cache.  One checkpoint and no switch points =
    BehaviorSpec::single."""
    from .policy import DecoderPolicy

    cks = list(checkpoints)
    if not cks:
        raise ValueError("kl: empty behavior spec")
    if not all(isinstance(p, DecoderPolicy) for p in cks + [target]):
        raise TypeError("kl_per_position: decoder policies (tabular / recurrent: the reference's own)")
    toks = np.concatenate([np.asarray(p, dtype=np.int32) for p in prefixes]) if prefixes else \
        np.zeros(1, dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum([len(p) for p in prefixes])]).astype(np.int64)
    n = max((len(p) for p in prefixes), default=0)
    out = np.zeros(max(n, 1))
    hs = (C.c_void_p * len(cks))(*[p.handle.value if hasattr(p.handle, "value") else p.handle for p in cks])
    sw = np.asarray(switch_points, dtype=np.int32)
    st = _lib.lib().srl_decoder_kl_per_position(hs, len(cks), sw.ctypes.data if len(sw) else None, len(sw),
                                               int(recompute_state), target.handle, toks.ctypes.data,
                                               offs.ctypes.data, len(prefixes), out.ctypes.data, len(out))
    _check(st, "kl_per_position")
    return out[:n]


def pipeline_max_lag_steps(gen_batch: int, inference_count: int, max_len: float, mean_len: float,
                           train_batch: int) -> int:
    """g_max = ceil(H * I * L / (mean L * B)) (throughput.cpp:260-269): the
    analytic maximum token lag, in optimizer steps, of a pipeline with I
    generators of constant batch H and a trainer consuming B sequences per
    step -- the cross-check for the lag the loop measures (test_sim.cpp:233-242)."""
    import math

    if gen_batch < 1 or inference_count < 1 or train_batch < 1 or not max_len > 0 or not mean_len > 0:
        raise ValueError("pipeline_max_lag_steps: invalid arguments")
    return int(math.ceil(float(gen_batch) * float(inference_count) * max_len / (mean_len * float(train_batch))))
