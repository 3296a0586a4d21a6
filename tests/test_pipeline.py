"""PipelineRL loop: the host actor queue against the reference simulator's
queue semantics (sim.cpp:265-369), and (GPU) a short generator -> queue ->
trainer -> in-flight update loop on the tiny decoder whose lag bookkeeping is
checked against the C oracle (make_step_record, sim.cpp:63-87)."""
import numpy as np
import pytest

from paper_2509_19128_b200.pipeline import ActorQueue, QueuedSequence


def seq(i):
    return QueuedSequence(i, "p", [], [], [], [], [])


def test_queue_delay_capacity_and_oldest_first_eviction():
    q = ActorQueue(capacity=3, preprocessor_delay=2)
    for i in range(5):
        q.push(seq(i), now=i)
    q.advance(3)                      # ready: 0 (t=2), 1 (t=3)
    assert [s.id for s in q.ring] == [0, 1] and not q.evicted
    q.advance(10)                     # 2, 3, 4 arrive; the ring holds 3: evict the oldest (0, 1)
    assert [s.id for s in q.ring] == [2, 3, 4]
    assert [s.id for s in q.evicted] == [0, 1]
    assert q.pop_batch(4) is None     # a starved trainer stalls
    assert [s.id for s in q.pop_batch(2)] == [2, 3]
    assert [s.id for s in q.ring] == [4]


def test_queue_rejects_zero_capacity():
    with pytest.raises(ValueError):
        ActorQueue(0)


@pytest.mark.gpu
def test_pipeline_loop_tiny(cuda):
    from oracle.oracle import Oracle
    from paper_2509_19128_b200.pipeline import PipelineRL
    from paper_2509_19128_b200.policy import TINY, DecoderPolicy

    pol = DecoderPolicy.random(TINY, seed=2, scale=0.05)
    pl = PipelineRL(pol, batch=8, prompt_len=6, max_tokens=12, train_batch=6, queue_capacity=16,
                    rounds_per_poll=4, n_prompts=3, lr=3e-3, seed=1)
    rep = pl.run(optimizer_steps=6)
    orc = Oracle()
    assert len(rep.steps) == 6 and rep.generated_sequences >= 36
    assert pl.engine.weight_version() == 6 == pl.channel.version
    for k, st in enumerate(rep.steps):
        assert st.version_before == k and np.isfinite(st.objective)
        assert st.pause_ms >= 0.0
    # lag bookkeeping of every consumed batch == the oracle's make_step_record
    q2 = PipelineRL(pol, batch=8, prompt_len=6, max_tokens=12, train_batch=6, queue_capacity=16,
                    rounds_per_poll=4, n_prompts=3, lr=3e-3, seed=1)
    batches = []
    orig = q2._train

    def spy(batch, report, step):
        batches.append(([list(s.versions) for s in batch], q2.channel.version))
        return orig(batch, report, step)
    q2._train = spy
    rep2 = q2.run(optimizer_steps=4)
    for (vers, vb), st in zip(batches, rep2.steps):
        exp = orc.lag_stats(vb, [np.asarray(v, dtype=np.int32) for v in vers])
        assert st.lag_histogram == exp["histogram"]
        assert st.max_lag_steps == exp["max_lag_steps"]
        assert st.mean_lag_steps == exp["mean_lag_steps"]
    # in-flight updates land mid-sequence: some consumed sequence spans two versions
    assert any(len(set(v)) > 1 for vers, _ in batches for v in vers)
    pl.close()
    q2.close()
