"""Host stand-ins for the generator engine and the trainer, with the interfaces
the partitioned PipelineRL loop (paper_2509_19128_b200/pipeline_dist.py) uses,
so its real code runs in multi-process gloo tests on CPU.

FakeEngine: constant-batch streams, one token per live stream per round,
tokens a deterministic function of (seed, position) and log-probs of the
ACTIVE weights (so a stream that keeps going after a swap shows the new
weights in its next log-prob); standby buffer + pointer swap.
FakeTrainer: fp32 weights viewed as bytes for the broadcast, a gradient that
is linear in the consumed trajectories (so data-parallel shards sum to the
full-batch gradient) and an ascent step."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class Ev:
    token: int
    logprob: float
    weight_version: int


class FakeEngine:
    def __init__(self, n_params: int, vocab: int, version_offset: int = 0):
        self.V = vocab
        self.active = torch.zeros(n_params, dtype=torch.float32)
        self.standby = torch.zeros(n_params, dtype=torch.float32)
        self.version = version_offset
        self.staged = None
        self.streams = {}
        self.next = 0

    # engine.hpp interface (subset)
    def open_stream(self, prompt_id, max_tokens, seed, terminator=-1, prompt=None):
        sid = f"s{self.next}"
        self.next += 1
        self.streams[sid] = dict(seed=seed, max=max_tokens, pos=0, out=[], done=False)
        return sid

    def advance(self, rounds):
        n = 0
        for _ in range(rounds):
            for s in self.streams.values():
                if s["done"]:
                    continue
                tok = int((s["seed"] * 2654435761 + s["pos"] * 40503) % self.V)
                lp = -float(np.log(self.V)) + 0.01 * float(self.active[tok % len(self.active)])
                s["out"].append(Ev(tok, lp, self.version))
                s["pos"] += 1
                n += 1
                if s["pos"] >= s["max"]:
                    s["done"] = True
        return n

    def wait_events_many(self, ids, columns=False):
        out = {}
        for sid in ids:
            s = self.streams[sid]
            evs, s["out"] = s["out"], []
            out[sid] = (evs, "length" if s["done"] else "running", not s["done"] or bool(evs))
            if s["done"] and not evs:
                out[sid] = (evs, "length", False)
        return out

    def weight_version(self):
        return self.version

    # standby adapter used by TorchTransport
    def standby_bytes(self):
        return self.standby.numel() * 4

    def stage(self, version):
        if version != self.version + 1 or self.staged is not None:
            raise ValueError("version_conflict")  # as EngineStandby.stage
        self.staged = version
        return self.standby.view(torch.uint8)

    def commit(self, version):
        if self.staged != version:
            return False, 0.0
        self.active, self.standby = self.standby, self.active
        self.version = version
        self.staged = None
        return True, 0.0


@dataclass
class FakeStep:
    objective: float
    ess: float


class FakeTrainer:
    def __init__(self, n_params: int):
        self.w = torch.zeros(n_params, dtype=torch.float32)
        self.g = torch.zeros(n_params, dtype=torch.float32)
        self.steps = []

    def step(self, packed, n_trajectories, clamp=5.0, granularity="sequence"):
        self.g.zero_()
        n = self.g.numel()
        idx = torch.arange(n, dtype=torch.float64)
        acc = torch.zeros(n, dtype=torch.float64)
        for t in packed:
            lb = t["loss_begin"]
            for tok, a in zip(t["tokens"][lb:], t["advantages"][lb:]):
                acc += a * (((idx + tok) % 7) - 3.0)
        self.g.copy_((acc / n_trajectories).float())
        self.steps.append(len(packed))
        return FakeStep(float(acc.sum()), 1.0)

    def apply_adam(self, lr):
        self.w += lr * self.g

    def weights_tensor(self):
        return self.w.view(torch.uint8)

    def gradient_tensor(self):
        return self.g
