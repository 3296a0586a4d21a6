"""PipelineRL (arXiv 2509.19128, Algorithm 2) end to end on the device path:

    generator Engine (constant batch, in-flight weight updates)
      -> host actor queue (preprocessor delay, bounded ring, oldest-first eviction)
      -> Trainer (log-prob recompute, truncated-IS REINFORCE, backward, Adam)
      -> WeightChannel (standby buffer + swap at a token boundary)
      -> generator, which keeps decoding its in-progress sequences on the stale KV cache.

The queue restates the reference tick simulator's actor queue
(/root/reference/proj/core/src/sim.cpp:265-369): finished sequences wait out a
preprocessor delay, then enter a ring of `queue_capacity` sequences; a full
ring evicts its oldest entry (:309-315); the trainer takes `train_batch`
sequences oldest-first when a batch is available and otherwise stalls
(:321-353).  Time is measured in generator rounds (the simulator's ticks).
Per consumed batch the lag bookkeeping of make_step_record / fill_sample_lags
(sim.cpp:63-104) is computed on the device (srl_lag_stats).

The generator and the trainer time-share one GPU here (the round-end driver
has one); with a partition (weight_sync.partition) each side runs on its own
ranks and the channel is an ncclBroadcast.
"""
from __future__ import annotations

import collections
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import Engine
from .rlmath import Trajectory, fit_baseline
from .trainer import Trainer
from .weight_sync import EngineStandby, WeightChannel


@dataclass
class QueuedSequence:
    """A finished generation: Trajectory (trajectory.hpp:15-25) + bookkeeping."""

    id: int
    prompt_id: str
    prompt: list               # prompt tokens (without bos)
    tokens: list               # generated tokens
    behavior_logprobs: list    # log mu of each generated token (event log-probs)
    versions: list             # weight version of each generated token
    consumed_at_emit: list     # sequences consumed by the trainer when each token was emitted
    reward: float = 0.0
    finish_round: int = 0


class ActorQueue:
    """Preprocessor delay + bounded ring with oldest-first eviction (sim.cpp:302-317)."""

    def __init__(self, capacity: int, preprocessor_delay: int = 0):
        if capacity < 1:
            raise ValueError("ActorQueue: capacity must be >= 1")
        self.capacity = capacity
        self.delay = preprocessor_delay
        self.preprocessor = collections.deque()  # (ready_round, seq)
        self.ring = collections.deque()
        self.evicted = []

    def push(self, seq: QueuedSequence, now: int):
        self.preprocessor.append((now + self.delay, seq))

    def advance(self, now: int):
        while self.preprocessor and self.preprocessor[0][0] <= now:
            if len(self.ring) == self.capacity:
                self.evicted.append(self.ring.popleft())
            self.ring.append(self.preprocessor.popleft()[1])

    def pop_batch(self, n: int):
        if len(self.ring) < n:
            return None
        return [self.ring.popleft() for _ in range(n)]


@dataclass
class StepReport:
    step: int
    round: int
    version_before: int
    reward_mean: float
    objective: float
    ess: float
    clamped: int
    tokens: int
    max_lag_steps: int
    mean_lag_steps: float
    lag_histogram: dict
    sample_max_lag: int
    pause_ms: float
    train_ms: float
    post_warmup: bool
    mean_length: float = 0.0   # mean generated length of the consumed batch


@dataclass
class PipelineReport:
    steps: list = field(default_factory=list)
    rounds: int = 0
    generated_tokens: int = 0
    generated_sequences: int = 0
    evicted: int = 0
    stalls: int = 0
    wall_s: float = 0.0
    generate_s: float = 0.0
    train_s: float = 0.0


def target_fraction_reward(target_mod: int = 4):
    """Synthetic task: reward = fraction of generated tokens t with t % target_mod == 0."""
    def reward(prompt, tokens):
        if not tokens:
            return 0.0
        return float(np.mean([(t % target_mod) == 0 for t in tokens]))
    return reward


class PipelineRL:
    """One generator engine + one trainer + the actor queue between them."""

    def __init__(self, policy, batch: int = 64, prompt_len: int = 16, max_tokens: int = 64,
                 train_batch: int = 32, queue_capacity: int = 256, preprocessor_delay: int = 0,
                 rounds_per_poll: int = 8, n_prompts: int = 8, clamp: float = 5.0,
                 granularity: str = "sequence", lr: float = 1e-4, reward_fn=None, seed: int = 0,
                 device: int = 0):
        self.cfg = policy.config
        self.B, self.prompt_len, self.max_tokens = batch, prompt_len, max_tokens
        self.train_batch, self.rounds_per_poll = train_batch, rounds_per_poll
        self.clamp, self.granularity, self.lr = clamp, granularity, lr
        self.reward_fn = reward_fn or target_fraction_reward()
        self.rng = np.random.default_rng(seed)
        # a small pool of prompts: several trajectories share a prompt, so the
        # per-(prompt, position) baseline of fit_baseline is informative
        self.prompts = {f"p{i}": self.rng.integers(0, self.cfg.vocab_size, size=prompt_len).tolist()
                        for i in range(n_prompts)}
        self.engine = Engine(policy, start_paused=True, max_streams=batch,
                             max_seq_len=1 + prompt_len + max_tokens + 1, rounds_per_sync=rounds_per_poll,
                             event_ring=max(64, rounds_per_poll), device=device,
                             prefill_budget=batch * (prompt_len + 1))
        self.trainer = Trainer(policy.clone(), max_tokens=train_batch * (1 + prompt_len + max_tokens),
                               device=device)
        self.channel = WeightChannel(src=0)
        self.standby = EngineStandby(self.engine, f"cuda:{device}")
        self.queue = ActorQueue(queue_capacity, preprocessor_delay)
        self.live = {}       # stream id -> QueuedSequence under construction
        self.next_id = 0
        self.consumed = 0
        self.round = 0
        self.device = device

    # ---------------------------------------------------------- generator ---
    def _open(self, staggered: int = 0):
        pid = f"p{int(self.rng.integers(0, len(self.prompts)))}"
        n = self.max_tokens if not staggered else max(4, self.max_tokens - staggered)
        sid = self.engine.open_stream(pid, n, int(self.rng.integers(0, 2**63)), -1, self.prompts[pid])
        self.live[sid] = QueuedSequence(self.next_id, pid, self.prompts[pid], [], [], [], [])
        self.next_id += 1

    def _generate(self, report: PipelineReport):
        t0 = time.perf_counter()
        self.engine.advance(self.rounds_per_poll)
        self.round += self.rounds_per_poll
        finished = []
        drained = self.engine.wait_events_many(list(self.live))
        for sid, seq in list(self.live.items()):
            evs, reason, more = drained[sid]
            for e in evs:
                seq.tokens.append(e.token)
                seq.behavior_logprobs.append(e.logprob)
                seq.versions.append(e.weight_version)
                seq.consumed_at_emit.append(self.consumed)
            report.generated_tokens += len(evs)
            if not more or reason != "running":
                finished.append(sid)
        for sid in finished:
            seq = self.live.pop(sid)
            seq.reward = self.reward_fn(seq.prompt, seq.tokens)
            seq.finish_round = self.round
            self.queue.push(seq, self.round)
            report.generated_sequences += 1
            self._open()  # constant generation batch (Algorithm 2)
        self.queue.advance(self.round)
        report.generate_s += time.perf_counter() - t0

    # ------------------------------------------------------------ trainer ---
    def _train(self, batch, report: PipelineReport, step: int):
        import torch

        t0 = time.perf_counter()
        version_before = self.channel.version
        trajs = [Trajectory(s.prompt_id, s.tokens, s.behavior_logprobs, s.versions, s.reward) for s in batch]
        base = fit_baseline(trajs)  # b(prompt, t): mean reward of the batch (rl_math.cpp:165-179)
        packed = []
        for s, t in zip(batch, trajs):
            P = 1 + len(s.prompt)
            toks = [self.cfg.bos_token] + s.prompt + s.tokens
            mu = [0.0] * P + list(s.behavior_logprobs)
            adv = [0.0] * P + [s.reward - base.at(s.prompt_id, p) for p in range(len(s.tokens))]
            packed.append(dict(tokens=toks, loss_begin=P, behavior_logprobs=mu, advantages=adv))
        res = self.trainer.step(packed, clamp=self.clamp, granularity=self.granularity)
        self.trainer.apply_adam(self.lr)
        # lag bookkeeping of the consumed batch (sim.cpp:63-104), on the device
        vers = torch.tensor(np.concatenate([np.asarray(s.versions, np.int32) for s in batch]),
                            device=f"cuda:{self.device}")
        offs = torch.tensor(np.concatenate([[0], np.cumsum([len(s.versions) for s in batch])]),
                            dtype=torch.int64, device=vers.device)
        hist = torch.zeros(1024, dtype=torch.int64, device=vers.device)
        sums = torch.zeros(len(batch), dtype=torch.int64, device=vers.device)
        tot = torch.zeros(4, dtype=torch.int64, device=vers.device)
        _lib.call("srl_lag_stats", vers.data_ptr(), offs.data_ptr(), len(batch), version_before,
                  hist.data_ptr(), 1024, sums.data_ptr(), tot.data_ptr(), None)
        # in-flight update: trainer weights -> standby buffer -> swap at the next token boundary
        src, n = self.trainer.weights()

        class _Raw:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (src, False), "version": 3}
        payload = torch.as_tensor(_Raw(), device=vers.device)
        applied, _, pause = self.channel.publish(0, None, payload, engine=self.standby)
        if not applied:
            raise RuntimeError("in-flight weight update rejected")
        torch.cuda.synchronize()
        t = tot.cpu().tolist()
        h = {i: int(c) for i, c in enumerate(hist.cpu().tolist()) if c}
        # fill_sample_lags (sim.cpp:89-104): the i-th sequence of the batch is
        # sample number consumed + i
        lags = [self.consumed + i - c for i, s in enumerate(batch) for c in s.consumed_at_emit]
        sample_lag = max(lags) if lags else 0
        self.consumed += len(batch)
        report.train_s += time.perf_counter() - t0
        return StepReport(step, self.round, version_before, float(np.mean([s.reward for s in batch])),
                          res.objective, res.ess, res.clamped, res.tokens, int(t[2]),
                          t[1] / max(t[0], 1), h, int(sample_lag), pause, res.step_ms,
                          all(s.versions and s.versions[0] >= 1 for s in batch),  # sim.cpp:106-110
                          float(np.mean([len(s.tokens) for s in batch])))

    # --------------------------------------------------------------- loop ---
    def run(self, optimizer_steps: int, max_rounds: int = 1_000_000) -> PipelineReport:
        report = PipelineReport()
        t0 = time.perf_counter()
        for i in range(self.B - len(self.live)):  # staggered initial lengths
            self._open(staggered=(i * self.max_tokens) // self.B)
        step = 0
        while step < optimizer_steps and self.round < max_rounds:
            self._generate(report)
            batch = self.queue.pop_batch(self.train_batch)
            if batch is None:
                report.stalls += 1  # the trainer waits for a full batch (sim.cpp:350-353)
                continue
            report.steps.append(self._train(batch, report, step))
            step += 1
        report.rounds = self.round
        report.evicted = len(self.queue.evicted)
        report.wall_s = time.perf_counter() - t0
        return report

    def close(self):
        self.engine.close()
        self.trainer.close()
