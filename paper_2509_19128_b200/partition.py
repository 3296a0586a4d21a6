"""Generator / trainer partitioning of one box (north_star: 1+1, 2+2, 4+4,
6+2, 7+1) from the paper's analytical pipeline model, fed with curves
measured on the B200 (tools/utilization_curve.py) instead of the
reference's default curve (assets/curves/default_utilization.csv).

Restates the reference's throughput model pieces this choice needs, same
semantics and tie-breaking:
  UtilizationCurve.value_at     throughput.cpp:36-65 (padding window)
  LengthDistribution.mean       throughput.cpp:123-137
  pipeline_max_lag_steps        throughput.cpp:260-269
  search_configs                throughput.cpp:288-330
Units are the reference's "flashes" (throughput.hpp:12-20): one flash is the
minimal amortised time of one token forward pass, flops_per_token /
peak_flops, so U(h) = tokens/s at batch h x flash seconds and the trainer's
tau = flashes per trained token.  tests/test_partition_cpu.py checks
search_configs against the reference itself (oracle/_ref).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass
class UtilizationCurve:
    samples: list  # [(h, utilization)], h strictly increasing, utilization in (0, 1]
    padding_window: int = 64

    def validate(self):
        if not self.samples:
            raise ValueError("UtilizationCurve: no samples")
        if self.padding_window < 0:
            raise ValueError("UtilizationCurve: negative padding window")
        prev = 0.0
        for h, u in self.samples:
            if h <= prev:
                raise ValueError("UtilizationCurve: batch sizes must be strictly increasing")
            if not (0.0 < u <= 1.0):
                raise ValueError("UtilizationCurve: utilization must be in (0, 1]")
            prev = h

    def last_batch_size(self) -> float:
        self.validate()
        return self.samples[-1][0]

    def _value(self, h: float) -> float:
        if not h > 0.0:
            raise ValueError("UtilizationCurve: batch size must be positive")
        h0, u0 = self.samples[0]
        if h <= h0:  # linear through the origin below the first sample
            return u0 * (h / h0)
        if h >= self.samples[-1][0]:
            return self.samples[-1][1]
        for (hl, ul), (hh, uh) in zip(self.samples, self.samples[1:]):
            if h <= hh:
                w = (h - hl) / (hh - hl)
                return ul + w * (uh - ul)
        return self.samples[-1][1]

    def value_at(self, h: float, use_padding: bool = False) -> float:
        self.validate()
        best = self._value(h)
        if not use_padding:
            return best
        for hp in range(max(math.ceil(h), 1), math.floor(h) + self.padding_window + 1):
            best = max(best, (h / hp) * self._value(float(hp)))
        return best


@dataclass
class LengthDistribution:
    kind: str = "constant"  # "uniform" | "constant" | "empirical"
    max_len: int = 1
    values: list = field(default_factory=list)

    def mean(self) -> float:
        if self.max_len < 1:
            raise ValueError("LengthDistribution: max_len must be positive")
        if self.kind == "uniform":
            return (1.0 + self.max_len) / 2.0
        if self.kind == "constant":
            return float(self.max_len)
        s = 0.0
        for v in self.values:
            s += v
        return s / len(self.values)


def pipeline_max_lag_steps(gen_batch: int, inference_count: int, max_len: float, mean_len: float,
                           train_batch: int) -> int:
    """ceil(H * I * L / (mean L * B)) (throughput.cpp:260-269)."""
    if gen_batch < 1 or inference_count < 1 or train_batch < 1 or not max_len > 0 or not mean_len > 0:
        raise ValueError("pipeline_max_lag_steps: invalid arguments")
    return int(math.ceil(float(gen_batch) * float(inference_count) * max_len / (mean_len * float(train_batch))))


@dataclass
class SearchResult:
    feasible: bool = False
    gen_batch: int = 0
    inference_count: int = 0
    r_gen: float = 0.0
    r_train: float = 0.0
    r_total: float = 0.0
    max_lag: int = 0


def search_configs(n_accelerators: int, train_batch: int, curve: UtilizationCurve, tau: float,
                   lengths: LengthDistribution, max_lag_steps_cap: int,
                   use_padding: bool = False) -> SearchResult:
    """Exhaustive (H, I) search (throughput.cpp:288-330): I generators over
    [1, N-1], H over every integer up to the curve's last sample; keep
    max lag <= cap; maximise r_total = min(U(H) I, (N - I) / tau), ties to
    smaller lag, then smaller I, then smaller H."""
    if n_accelerators < 2:
        raise ValueError("search_configs: need n_accelerators >= 2")
    if train_batch < 1:
        raise ValueError("search_configs: train_batch must be >= 1")
    if max_lag_steps_cap < 1:
        raise ValueError("search_configs: cap must be >= 1")
    h_limit = int(math.floor(curve.last_batch_size()))
    mean_len = lengths.mean()
    best = SearchResult()
    for inference in range(1, n_accelerators):
        r_train = float(n_accelerators - inference) / tau
        for h in range(1, h_limit + 1):
            lag = pipeline_max_lag_steps(h, inference, lengths.max_len, mean_len, train_batch)
            if lag > max_lag_steps_cap:
                break  # lag grows with h
            r_gen = curve.value_at(h, use_padding) * inference
            r_total = min(r_gen, r_train)
            better = (not best.feasible or r_total > best.r_total or
                      (r_total == best.r_total and
                       (lag < best.max_lag or
                        (lag == best.max_lag and
                         (inference < best.inference_count or
                          (inference == best.inference_count and h < best.gen_batch))))))
            if better:
                best = SearchResult(True, h, inference, r_gen, r_train, r_total, lag)
    return best


def curve_from_measurement(points, flops_per_token: float, peak_flops: float,
                           padding_window: int = 64) -> UtilizationCurve:
    """U(h) from measured (h, tokens/s) of one generator GPU: tokens/s x flash
    seconds (throughput.hpp:12-20), clamped into (0, 1]."""
    flash = flops_per_token / peak_flops
    out = []
    for h, tps in sorted(points):
        out.append((float(h), min(1.0, max(1e-12, tps * flash))))
    return UtilizationCurve(out, padding_window)
