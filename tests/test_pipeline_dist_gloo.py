"""The partitioned PipelineRL loop (paper_2509_19128_b200/pipeline_dist.py) run
as real processes over gloo on CPU, with host stand-ins for the engine and the
trainer (tests/dist_fakes.py) and the torch.distributed transport -- the same
loop code the box runs with the device engine, the device trainer and the
C-ABI NCCL channel.  Checks, per partition (1+1, 2+1, 1+2):

* every consumed batch's lag record equals the C oracle's make_step_record /
  fill_sample_lags (sim.cpp:63-104) on the same token versions;
* after every broadcast each generator serves exactly the trainers' weights
  (bitwise), and the data-parallel trainers agree bitwise with each other;
* the data-parallel gradient equals the single-trainer full-batch gradient;
* the steady-state max lag is within one step of the analytic
  g_max = ceil(H I L / (mean L B)) (throughput.cpp:260-269; test_sim.cpp:233-242);
* a generator whose engine rejects the version keeps serving and nobody hangs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_19128_b200.pipeline_dist import DistributedPipelineRL, TorchTransport, step_record
from paper_2509_19128_b200.weight_sync import partition

N_PARAMS = 257
V = 97


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, trainers, port, q, kw):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from dist_fakes import FakeEngine, FakeTrainer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = partition(world, trainers)
        role = part.role(rank)
        offset = kw.pop("reject_rank_offset", {}).get(rank, 0)
        eng = FakeEngine(N_PARAMS, V, offset) if role == "generator" else None
        tr = FakeTrainer(N_PARAMS) if role == "trainer" else None
        loop = DistributedPipelineRL(part, rank, engine=eng, trainer=tr,
                                     transport=TorchTransport(part, rank), vocab_size=V,
                                     bos_token=0, **kw)
        rep = loop.run(optimizer_steps=6)
        out = dict(rank=rank, role=role, version=loop.version,
                   weights=(eng.active if eng is not None else tr.w).numpy().copy(),
                   grad=tr.g.numpy().copy() if tr is not None else None,
                   steps=[(s.version_before, s.lag) for s in rep.steps],
                   rejected=rep.rejected_updates, pauses=len(rep.pauses_ms),
                   engine_version=eng.version if eng is not None else None)
        q.put(out)
    finally:
        dist.destroy_process_group()


def run_partition(world, trainers, **kw):
    base = dict(batch=6, prompt_len=3, max_tokens=8, train_batch=6 * (world - trainers),
                queue_capacity=64, rounds_per_period=2, n_prompts=3, lr=0.5, seed=11)
    base.update(kw)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, trainers, port, q, dict(base)))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r["rank"]), base


@pytest.mark.parametrize("world,trainers", [(2, 1), (3, 1), (3, 2)])
def test_partitioned_loop(world, trainers):
    res, kw = run_partition(world, trainers)
    trs = [r for r in res if r["role"] == "trainer"]
    gens = [r for r in res if r["role"] == "generator"]
    assert len(trs) == trainers and len(gens) == world - trainers
    # six optimizer steps, every generator at the trainers' version, same weights bitwise
    for r in res:
        assert r["version"] == 6
    for g in gens:
        assert g["engine_version"] == 6 and g["rejected"] == 0
        assert np.array_equal(g["weights"], trs[0]["weights"])
    for t in trs[1:]:
        assert np.array_equal(t["weights"], trs[0]["weights"])
        assert np.array_equal(t["grad"], trs[0]["grad"])
    # lag: versions before are 0..5, lags non-negative; the analytic bound
    steps = trs[0]["steps"]
    assert [vb for vb, _ in steps] == list(range(6))
    n_gen = world - trainers
    g_max = int(np.ceil(kw["batch"] * n_gen * kw["max_tokens"] / (kw["max_tokens"] * kw["train_batch"])))
    for vb, lag in steps:
        assert min(lag["histogram"]) >= 0
        assert lag["max_lag_steps"] <= g_max + 1


def test_dp_gradient_equals_full_batch():
    one, _ = run_partition(2, 1)
    two, _ = run_partition(3, 2)
    # same generator (seeded by its index in the partition), one vs two trainer shards
    g1 = next(r for r in one if r["role"] == "trainer")
    g2 = next(r for r in two if r["role"] == "trainer")
    np.testing.assert_allclose(g2["grad"], g1["grad"], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(g2["weights"], g1["weights"], rtol=1e-6, atol=1e-6)


def test_rejecting_generator_keeps_serving():
    # rank 2's engine starts at version 10: every update conflicts (version_conflict)
    res, _ = run_partition(3, 1, reject_rank_offset={2: 10})
    bad = res[2]
    good = res[1]
    assert good["engine_version"] == 6 and good["rejected"] == 0
    assert bad["engine_version"] == 10 and bad["rejected"] == 6 and bad["pauses"] == 0


def test_step_record_matches_oracle():
    from oracle.oracle import Oracle

    rng = np.random.default_rng(3)
    orc = Oracle()
    for _ in range(20):
        vb = int(rng.integers(1, 9))
        vers = [np.sort(rng.integers(0, vb + 1, size=int(rng.integers(1, 12)))).astype(np.int32)
                for _ in range(int(rng.integers(1, 6)))]
        cae = [np.sort(rng.integers(0, 30, size=len(v))) for v in vers]
        cb = int(rng.integers(30, 40))
        mine = step_record(vb, vers, cae, cb)
        exp = orc.lag_stats(vb, vers, cae, cb)
        assert mine["histogram"] == exp["histogram"]
        assert mine["max_lag_steps"] == exp["max_lag_steps"]
        assert mine["mean_lag_steps"] == exp["mean_lag_steps"]
        assert mine["sequence_lag_sums"] == exp["sequence_lag_sums"]
        assert mine["max_lag_samples"] == exp["max_lag_samples"]
        assert mine["mean_lag_samples"] == exp["mean_lag_samples"]
        assert mine["post_warmup"] == exp["post_warmup"]
