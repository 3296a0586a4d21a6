"""PipelineRL over a generator / trainer partition of one node (arXiv
2509.19128 Algorithm 2 with I generator GPUs and a data-parallel trainer
group; 1+1, 2+2, 4+4, 6+2, 7+1).

One process per GPU.  ``weight_sync.partition(world, trainers)`` puts the
trainer ranks first and the generator ranks after.  The loop advances in
periods of R generator rounds (the reference simulator's ticks,
/root/reference/proj/core/src/sim.cpp:265-369); in period k:

* every rank pops the next training batch from its replica of the host actor
  queue (preprocessor delay, bounded ring, oldest-first eviction,
  sim.cpp:302-353) -- the replicas see the same finished sequences in the same
  order, so every rank knows whether the trainer steps this period;
* if the trainer stepped in period k-1, its new weights (version v) are
  broadcast from trainer rank 0 into every generator's standby buffer
  (``srl_comm_send_weights`` / ``srl_comm_recv_weights_begin``), overlapped
  with the generators' decode of this period, and swapped in at the token
  boundary after it (``srl_comm_recv_weights_finish``): the in-flight update,
  the sequences in progress keep their stale KV cache;
* generator ranks decode R rounds of their constant batch, drain the token
  events (each stamped with the weight version that emitted it) and refill
  finished streams;
* trainer ranks (if a batch was popped) take their shard of it
  (``weight_sync.shard``), run the IS-REINFORCE step normalised by the GLOBAL
  trajectory count (rl_math.cpp:211-276), all-reduce the fp32 gradient over
  the trainer group (``srl_comm_allreduce_gradient``) and apply Adam;
* the finished sequences of every generator are exchanged on the host
  (torch.distributed all_gather_object over a gloo group: control data only)
  and enter every queue replica in rank order.

Per consumed batch, trainer rank 0 records the lag statistics of
make_step_record / fill_sample_lags / batch_post_warmup (sim.cpp:63-110).

The transports are pluggable: ``NcclTransport`` (the C ABI of csrc/comm.cpp,
NCCL over NVLink) on the box, ``TorchTransport`` (torch.distributed, gloo on
CPU tensors) for the multi-process CPU tests, which drive this same loop with
host stand-ins for the engine and the trainer.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .pipeline import ActorQueue, QueuedSequence, target_fraction_reward
from .rlmath import Trajectory, fit_baseline
from .weight_sync import partition, shard


# ------------------------------------------------------------ lag record ---
def step_record(version_before: int, token_versions, consumed_at_emit, consumed_before: int):
    """make_step_record + fill_sample_lags + batch_post_warmup (sim.cpp:63-110)
    of one consumed batch: lag = version_before - token version (sim.cpp:74);
    the i-th sequence of the batch is sample number consumed_before + i and a
    token's sample lag is that minus the samples consumed when it was emitted
    (sim.cpp:89-104); post-warmup = every sequence's first token has version
    >= 1 (sim.cpp:106-110).  Integer bookkeeping on the host (the trainer's
    actor side), the same arithmetic as srl_lag_stats."""
    hist: dict = {}
    tokens = lag_sum = max_lag = 0
    seq_sums = []
    for vers in token_versions:
        ss = 0
        for v in vers:
            lag = version_before - int(v)
            hist[lag] = hist.get(lag, 0) + 1
            max_lag = max(max_lag, lag)
            lag_sum += lag
            ss += lag
        tokens += len(vers)
        seq_sums.append(ss)
    smax = ssum = scount = 0
    for i, cae in enumerate(consumed_at_emit):
        for c in cae:
            lag = consumed_before + i - int(c)
            smax = max(smax, lag)
            ssum += lag
            scount += 1
    return {"histogram": hist, "tokens": tokens, "max_lag_steps": max_lag,
            "mean_lag_steps": lag_sum / tokens if tokens else 0.0, "sequence_lag_sums": seq_sums,
            "max_lag_samples": smax, "mean_lag_samples": ssum / scount if scount else 0.0,
            "post_warmup": all(len(v) and int(v[0]) >= 1 for v in token_versions)}


# ------------------------------------------------------------ transports ---
class NcclTransport:
    """The C-ABI channel (csrc/comm.cpp): one communicator for the broadcast
    group (trainer rank 0 + the generators) and one for the trainer group."""

    def __init__(self, part, rank: int, device: int, pg=None):
        import torch.distributed as dist

        from .comm import NcclComm, unique_id

        self.root = 0  # trainer rank 0 is index 0 of the broadcast group
        self.bcast_ranks = [part.trainers[0], *part.generators]
        ids = [None, None]
        if rank == part.trainers[0]:  # a member of both groups generates both ids
            ids = [unique_id(), unique_id()]
        dist.broadcast_object_list(ids, src=part.trainers[0], group=pg)
        self.bcast = NcclComm(ids[0], len(self.bcast_ranks), self.bcast_ranks.index(rank), device) \
            if rank in self.bcast_ranks else None
        self.train = NcclComm(ids[1], len(part.trainers), part.trainers.index(rank), device) \
            if rank in part.trainers and len(part.trainers) > 1 else None

    def send(self, trainer):
        self.bcast.send_weights(trainer)

    def wait(self) -> float:
        return self.bcast.wait()

    def recv_begin(self, engine, version: int) -> bool:
        return self.bcast.recv_weights_begin(self.root, engine, version)

    def recv_finish(self, engine, version: int):
        return self.bcast.recv_weights_finish(engine, version)

    def allreduce(self, trainer):
        if self.train is not None:
            self.train.allreduce_gradient(trainer)

    def close(self):
        for c in (self.bcast, self.train):
            if c is not None:
                c.close()


class TorchTransport:
    """torch.distributed on host tensors (the CPU tests): the same collective
    pattern as NcclTransport.  Engines expose stage(version) -> tensor or None
    and commit(version) -> (applied, pause_ms); trainers weights_tensor() and
    gradient_tensor()."""

    def __init__(self, part, rank: int):
        import torch.distributed as dist

        self.dist = dist
        self.root = part.trainers[0]
        self.bcast_ranks = [part.trainers[0], *part.generators]
        self.bcast_group = dist.new_group(self.bcast_ranks)
        self.train_group = dist.new_group(list(part.trainers))
        self.n_trainers = len(part.trainers)
        self._staged = None
        self._t0 = 0.0

    def send(self, trainer):
        self._t0 = time.perf_counter()
        self.dist.broadcast(trainer.weights_tensor(), src=self.root, group=self.bcast_group)

    def wait(self) -> float:
        return 1e3 * (time.perf_counter() - self._t0)

    def recv_begin(self, engine, version: int) -> bool:
        import torch

        from ._lib import SrlError

        try:
            view = engine.stage(version)
        except (ValueError, SrlError):  # version_conflict / busy: keep serving, still join the broadcast
            view = None
        self._staged = view is not None
        buf = view if view is not None else torch.empty(engine.standby_bytes(), dtype=torch.uint8)
        self._t0 = time.perf_counter()
        self.dist.broadcast(buf, src=self.root, group=self.bcast_group)
        return self._staged

    def recv_finish(self, engine, version: int):
        t = 1e3 * (time.perf_counter() - self._t0)
        if not self._staged:
            return False, engine.weight_version(), t, 0.0
        applied, pause = engine.commit(version)
        return applied, engine.weight_version(), t, pause

    def allreduce(self, trainer):
        if self.n_trainers > 1:
            self.dist.all_reduce(trainer.gradient_tensor(), group=self.train_group)


# ------------------------------------------------------------------ loop ---
@dataclass
class DistStep:
    step: int
    period: int
    version_before: int
    reward_mean: float
    objective: float
    ess: float
    lag: dict
    transfer_ms: float = 0.0
    train_ms: float = 0.0


@dataclass
class DistReport:
    steps: list = field(default_factory=list)
    periods: int = 0
    generated_tokens: int = 0       # over every generator rank
    generated_sequences: int = 0
    evicted: int = 0
    stalls: int = 0
    wall_s: float = 0.0
    pauses_ms: list = field(default_factory=list)
    transfers_ms: list = field(default_factory=list)
    rejected_updates: int = 0


class DistributedPipelineRL:
    """The partitioned loop.  engine / trainer are this rank's (None where the
    role does not apply); every rank runs the same period sequence."""

    def __init__(self, part, rank: int, *, engine=None, trainer=None, transport=None, control_group=None,
                 vocab_size: int, bos_token: int, batch: int, prompt_len: int, max_tokens: int,
                 train_batch: int, queue_capacity: int, rounds_per_period: int,
                 preprocessor_delay: int = 0, n_prompts: int = 8, clamp: float = 5.0,
                 granularity: str = "sequence", lr: float = 1e-5, reward_fn=None, seed: int = 0):
        self.part, self.rank = part, rank
        self.role = part.role(rank)
        self.engine, self.trainer, self.transport = engine, trainer, transport
        self.control_group = control_group
        self.V, self.bos = vocab_size, bos_token
        self.B, self.prompt_len, self.max_tokens = batch, prompt_len, max_tokens
        self.train_batch, self.R = train_batch, rounds_per_period
        self.clamp, self.granularity, self.lr = clamp, granularity, lr
        self.reward_fn = reward_fn or target_fraction_reward()
        prng = np.random.default_rng(seed)  # identical on every rank: shared prompt pool
        self.prompts = {f"p{i}": prng.integers(0, vocab_size, size=prompt_len).tolist()
                        for i in range(n_prompts)}
        # per generator (its index in the partition, not its global rank)
        gi = part.generators.index(rank) if rank in part.generators else -1
        self.rng = np.random.default_rng(seed + 1000 + gi)
        self.queue = ActorQueue(queue_capacity, preprocessor_delay)
        self.version = 0          # trainer weight version (every rank tracks it)
        self.publish = False      # the trainer stepped last period: broadcast this period
        self.consumed = 0
        self.period = 0
        self.step_no = 0
        self.live = {}
        self.next_id = 0

    # ---------------------------------------------------------- generator ---
    def _open(self, staggered: int = 0):
        pid = f"p{int(self.rng.integers(0, len(self.prompts)))}"
        n = self.max_tokens if not staggered else max(4, self.max_tokens - staggered)
        sid = self.engine.open_stream(pid, n, int(self.rng.integers(0, 2**63)), -1, self.prompts[pid])
        self.live[sid] = QueuedSequence(self.part.generators.index(self.rank) * 10**9 + self.next_id, pid, self.prompts[pid],
                                        [], [], [], [])
        self.next_id += 1

    def _generate(self, report: DistReport):
        finished = []
        update = None
        if self.publish:
            staged = self.transport.recv_begin(self.engine, self.version)
            update = staged
        self.engine.advance(self.R)
        if update is not None:
            applied, _, tms, pause = self.transport.recv_finish(self.engine, self.version)
            if applied:
                report.pauses_ms.append(pause)
            else:
                report.rejected_updates += 1
            report.transfers_ms.append(tms)
        drained = self.engine.wait_events_many(list(self.live))
        for sid, seq in list(self.live.items()):
            evs, reason, more = drained[sid]
            for e in evs:
                seq.tokens.append(int(e.token))
                seq.behavior_logprobs.append(float(e.logprob))
                seq.versions.append(int(e.weight_version))
                seq.consumed_at_emit.append(self.consumed)
            if not more or reason != "running":
                finished.append(sid)
        out = []
        for sid in finished:
            seq = self.live.pop(sid)
            seq.reward = self.reward_fn(seq.prompt, seq.tokens)
            out.append(seq)
            self._open()
        return out

    # ------------------------------------------------------------ trainer ---
    def _train(self, batch):
        trajs = [Trajectory(s.prompt_id, s.tokens, s.behavior_logprobs, s.versions, s.reward)
                 for s in batch]
        base = fit_baseline(trajs)  # rl_math.cpp:165-179, over the whole consumed batch
        packed = []
        for s in batch:
            P = 1 + len(s.prompt)
            packed.append(dict(tokens=[self.bos] + s.prompt + s.tokens, loss_begin=P,
                               behavior_logprobs=[0.0] * P + list(s.behavior_logprobs),
                               advantages=[0.0] * P + [s.reward - base.at(s.prompt_id, p)
                                                       for p in range(len(s.tokens))]))
        mine = shard(packed, self.part.trainers.index(self.rank), len(self.part.trainers))
        t0 = time.perf_counter()
        res = self.trainer.step(mine, n_trajectories=len(batch), clamp=self.clamp,
                                granularity=self.granularity) if mine else None
        self.transport.allreduce(self.trainer)
        self.trainer.apply_adam(self.lr)
        return res, 1e3 * (time.perf_counter() - t0)

    # --------------------------------------------------------------- loop ---
    def _exchange(self, mine):
        import torch.distributed as dist

        payload = [(s.id, s.prompt_id, s.prompt, s.tokens, s.behavior_logprobs, s.versions,
                    s.consumed_at_emit, s.reward) for s in mine]
        gathered = [None] * self.part.world
        dist.all_gather_object(gathered, payload, group=self.control_group)
        out = []
        for r in self.part.generators:
            for (i, pid, pr, tk, lp, vs, cae, rw) in gathered[r]:
                out.append(QueuedSequence(i, pid, list(pr), list(tk), list(lp), list(vs), list(cae), rw))
        return out

    def run(self, optimizer_steps: int, max_periods: int = 100_000) -> DistReport:
        rep = DistReport()
        t0 = time.perf_counter()
        if self.role in ("generator", "both") and not self.live:
            for i in range(self.B):
                self._open(staggered=(i * self.max_tokens) // self.B)
        target = self.step_no + optimizer_steps
        while self.step_no < target and self.period < max_periods:
            now = self.period * self.R
            self.queue.advance(now)
            batch = self.queue.pop_batch(self.train_batch)
            consumed_before = self.consumed
            if batch is not None:
                self.consumed += len(batch)
            else:
                rep.stalls += 1  # the trainer waits for a full batch (sim.cpp:350-353)
            transfer = 0.0
            mine = []
            if self.role in ("trainer", "both"):
                if self.publish and self.rank == self.part.trainers[0]:
                    self.transport.send(self.trainer)
                res, train_ms = self._train(batch) if batch is not None else (None, 0.0)
                if self.publish and self.rank == self.part.trainers[0]:
                    transfer = self.transport.wait()
            if self.role in ("generator", "both"):
                mine = self._generate(rep)
            if batch is not None and self.rank == self.part.trainers[0]:
                lag = step_record(self.version, [s.versions for s in batch],
                                  [s.consumed_at_emit for s in batch], consumed_before)
                rep.steps.append(DistStep(self.step_no, self.period, self.version,
                                          float(np.mean([s.reward for s in batch])),
                                          res.objective if res else 0.0, res.ess if res else 0.0,
                                          lag, transfer, train_ms))
            finished = self._exchange(mine)
            self.period += 1
            for s in finished:
                self.queue.push(s, (self.period) * self.R)
            rep.generated_sequences += len(finished)
            rep.generated_tokens += sum(len(s.tokens) for s in finished)
            self.publish = batch is not None
            if batch is not None:
                self.version += 1
                self.step_no += 1
        # the last step's weights still go out (every rank takes part)
        if self.publish:
            if self.role in ("trainer", "both") and self.rank == self.part.trainers[0]:
                self.transport.send(self.trainer)
                self.transport.wait()
            if self.role == "generator":
                self.transport.recv_begin(self.engine, self.version)
                applied, _, tms, pause = self.transport.recv_finish(self.engine, self.version)
                rep.transfers_ms.append(tms)
                if applied:
                    rep.pauses_ms.append(pause)
                else:
                    rep.rejected_updates += 1
            self.publish = False
        rep.periods = self.period
        rep.evicted = len(self.queue.evicted)
        rep.wall_s = time.perf_counter() - t0
        return rep


# ------------------------------------------------------------ the bench ---
def bench_partitioned(args, cfg):
    """bench.py at N > 1: the partitioned loop on the box's GPUs (one rank
    per GPU), weak scaling in the generator count.  Returns rank 0's JSON
    line: tokens/s over every generator, the update pause and broadcast
    GB/s, the lag of every consumed batch."""
    import os

    import torch
    import torch.distributed as dist

    from .engine import Engine
    from .policy import DecoderPolicy
    from .trainer import Trainer

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    part = partition(world, args.trainers)
    pol = DecoderPolicy.random(cfg, seed=0, scale=0.02, device=local)
    B, R = args.batch, args.rounds
    gen = args.train_gen
    engine = trainer = None
    if part.role(rank) == "generator":
        engine = Engine(pol, start_paused=True, max_streams=B, max_seq_len=args.prompt + gen + 2,
                        rounds_per_sync=R, event_ring=max(64, R), device=local,
                        prefill_budget=B * (args.prompt + 1))
    else:
        n_tr = len(part.trainers)
        trainer = Trainer(pol, max_tokens=((B + n_tr - 1) // n_tr) * (args.prompt + gen + 1), device=local)
    transport = NcclTransport(part, rank, local)
    loop = DistributedPipelineRL(part, rank, engine=engine, trainer=trainer, transport=transport,
                                 vocab_size=cfg.vocab_size, bos_token=cfg.bos_token, batch=B,
                                 prompt_len=args.prompt, max_tokens=gen, train_batch=B * len(part.generators),
                                 queue_capacity=8 * B * len(part.generators), rounds_per_period=R)
    loop.run(optimizer_steps=max(1, args.warmup))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = loop.run(optimizer_steps=args.steps)
    torch.cuda.synchronize()
    dist.barrier()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    payload = pol.weights()[1]
    stats = [None] * world
    dist.all_gather_object(stats, {"pauses": rep.pauses_ms, "transfers": rep.transfers_ms})
    pauses = [p for s in stats for p in s["pauses"]]
    transfers = [x for s in stats for x in s["transfers"]]
    line = None
    if rank == 0:
        lags = [st.lag for st in rep.steps]
        tms = float(np.median(transfers)) if transfers else None
        line = {
            "metric": "generated tokens/sec with in-flight updates", "value": rep.generated_tokens / dt,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / max(1, len(rep.steps)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic prompts, random-init weights",
            "config": {"workload": f"{cfg.name} PipelineRL, {len(part.generators)} generator + "
                                   f"{len(part.trainers)} trainer GPUs, batch {B} per generator, "
                                   f"rollouts of {gen} tokens, {R} rounds per period",
                       "model": cfg.name, "global_batch": B * len(part.generators),
                       "seq_len": args.prompt + gen + 1,
                       "parallelism": f"{len(part.generators)}g+{len(part.trainers)}t"},
            "e2e": {"value": rep.generated_tokens / rep.wall_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None},
            "pause_ms": {"median": float(np.median(pauses)) if pauses else None,
                         "max": float(np.max(pauses)) if pauses else None},
            "broadcast": {"payload_bytes": payload, "transfer_ms_median": tms,
                          "gbs": payload / (tms * 1e-3) / 1e9 if tms else None,
                          "nvlink_peak_gbs": 900.0},
            "lag": {"max_lag_steps": max((l["max_lag_steps"] for l in lags), default=None),
                    "mean_lag_steps": float(np.mean([l["mean_lag_steps"] for l in lags])) if lags else None,
                    "max_lag_samples": max((l["max_lag_samples"] for l in lags), default=None),
                    "consumed_batches": len(lags)},
            "stalls": rep.stalls, "evicted": rep.evicted,
        }
    transport.close()
    if engine is not None:
        engine.close()
    if trainer is not None:
        trainer.close()
    dist.destroy_process_group()
    return line
