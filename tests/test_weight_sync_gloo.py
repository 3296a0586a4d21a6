"""N>1 host logic on CPU: world-size-2 gloo process groups exercise the weight
channel (one broadcast per optimizer step into the generators' standby
buffers, strictly sequential versions, rejection without side effects) and
the generator/trainer partitioning.  The device path is the same code with
backend "nccl" and device buffers (bench.py --gpus N)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_19128_b200.weight_sync import WeightChannel, max_over_ranks, partition


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeEngine:
    """Stands in for Engine.begin/commit_weight_update: standby + active buffers."""

    def __init__(self, n):
        self.version = 0
        self.active = torch.zeros(n, dtype=torch.uint8)
        self.standby = torch.zeros(n, dtype=torch.uint8)
        self.staged = None

    def stage(self, v):
        if v != self.version + 1:  # as EngineStandby.stage / begin_weight_update
            raise ValueError("version_conflict")
        self.staged = v
        return self.standby

    def commit(self, v):
        if self.staged != v:
            return False, 0.0
        self.active, self.standby = self.standby, self.active  # pointer swap
        self.version = v
        self.staged = None
        return True, 0.0


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = partition(world, 1)
        n = 4096
        eng = FakeEngine(n)
        ch = WeightChannel(src=part.trainers[0])
        results = []
        for step in range(3):
            payload = None
            if part.role(rank) == "trainer":
                payload = torch.full((n,), (step * 7 + 3) % 251, dtype=torch.uint8)
            applied, v, _ = ch.publish(rank, torch.empty(n, dtype=torch.uint8) if rank == 0
                                       else eng.standby, payload,
                                       engine=eng if part.role(rank) == "generator" else None)
            results.append((applied, v, int(eng.active[0]), int(eng.active[-1])))
        t = max_over_ranks(float(rank + 1))
        q.put((rank, part.role(rank), results, eng.version, t))
    finally:
        dist.destroy_process_group()


def test_weight_channel_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, role, results, version, t = q.get(timeout=120)
        out[rank] = (role, results, version, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == "trainer" and out[1][0] == "generator"
    # the generator received every payload in order and swapped it in
    gen = out[1][1]
    assert [r[1] for r in gen] == [1, 2, 3]
    assert [r[2] for r in gen] == [(s * 7 + 3) % 251 for s in range(3)]
    assert all(r[2] == r[3] for r in gen)
    assert out[1][2] == 3
    assert out[0][3] == out[1][3] == 2.0  # max over ranks


def test_partitions_of_the_box():
    assert partition(1).role(0) == "both"
    p = partition(8, 4)
    assert p.trainers == (0, 1, 2, 3) and p.generators == (4, 5, 6, 7)
    p = partition(8, 2)  # 6 generators + 2 trainers (BASELINE.json config 4)
    assert len(p.generators) == 6 and p.role(1) == "trainer" and p.role(7) == "generator"
    p = partition(8, 1)  # 7 + 1
    assert len(p.generators) == 7
    with pytest.raises(ValueError):
        partition(2, 2)


def test_stale_version_is_rejected_without_side_effects():
    eng = FakeEngine(8)
    before = eng.active.clone()
    with pytest.raises(ValueError):
        eng.stage(2)  # version_conflict: not staged
    ok, _ = eng.commit(2)
    assert not ok and torch.equal(eng.active, before) and eng.version == 0


def _conflict_worker(rank, world, port, q):
    """The generator is one version ahead of the channel: it rejects the first
    update (version_conflict) but still joins the broadcast -- the trainer
    does not hang -- keeps its weights, and accepts the next one."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1024
        eng = FakeEngine(n)
        eng.version = 1
        eng.active.fill_(42)
        ch = WeightChannel(src=0)
        out = []
        for step in range(2):
            payload = torch.full((n,), 10 + step, dtype=torch.uint8) if rank == 0 else None
            if rank == 1 and step == 1:
                ch.version = 1  # the generator's channel catches up with its engine
            applied, v, _ = ch.publish(rank, torch.empty(n, dtype=torch.uint8) if rank == 0 else eng.standby,
                                       payload, engine=eng if rank == 1 else None)
            out.append((applied, v, int(eng.active[0])))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_rejecting_generator_still_joins_the_broadcast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_conflict_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[1][0] == (False, 0, 42)      # rejected: weights untouched, version unchanged
    assert out[1][1] == (True, 2, 11)       # the next update lands


def _dp_worker(rank, world, port, q):
    """Each rank: the reference-semantics tabular IS-REINFORCE gradient of its
    shard (global baseline, shard normalised by the global m), then the
    trainer's gradient all-reduce; the result must equal the full-batch
    gradient (rl_math.cpp:211-276)."""
    import numpy as np

    from oracle.oracle import Oracle
    from paper_2509_19128_b200.weight_sync import GradientSync, shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        rng = np.random.default_rng(3)
        V = 5
        doc = {"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": V, "context_order": 1,
               "rows": [{"prompt_id": "p", "context": [], "logits": [0.1, -0.2, 0.3, 0.0, 0.5]},
                        {"prompt_id": "p", "context": [1], "logits": [0.0, 0.4, -0.1, 0.2, 0.1]}]}
        trajs = []
        for i in range(7):
            toks = rng.integers(0, V, size=int(rng.integers(2, 6))).tolist()
            trajs.append(dict(prompt_id="p", tokens=toks,
                              behavior_logprobs=(-np.log(V) + 0.3 * rng.standard_normal(len(toks))).tolist(),
                              reward=float(rng.standard_normal())))
        full, _, base = orc.reinforce_gradient_tab(doc, trajs)
        mine = shard(trajs, rank, world)
        g, _, _ = orc.reinforce_gradient_tab(doc, mine, baseline=base)
        g = torch.tensor(g * (len(mine) / len(trajs)))
        GradientSync().allreduce_(g)
        q.put((rank, float(np.abs(g.numpy() - full).max()), float(np.abs(full).max())))
    finally:
        dist.destroy_process_group()


def test_trainer_data_parallel_gradient_allreduce_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, scale in res:
        assert scale > 0 and err <= 1e-12 * scale, (rank, err, scale)
