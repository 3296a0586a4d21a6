"""Device engine vs the reference semantics for the reference's own policy
types (tabular, recurrent), in lockstep.  Bar: tokens, version stamps,
positions and finish reasons bit-exact; log-probs within 1e-12 relative
(device libm exp/log/tanh may differ from glibc by an ulp).

Mirrors tests/test_protocol.cpp and acceptance criteria 9/10 of the
reference (in-process, no HTTP)."""
import json

import numpy as np
import pytest

from oracle.oracle import Oracle, drift_checkpoints, random_recurrent_policy
from paper_2509_19128_b200.engine import Engine
from paper_2509_19128_b200.policy import policy_from_dict

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(__file__.replace("test_engine_gpu.py", "golden/reference_vectors.json")))
# device libm (exp/log/tanh) vs glibc differ by <= 1 ulp; through the recurrent
# state this compounds to ~1e-11 relative after 48 steps.
LP_REL = 1e-9


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def run_engine(docs, update_after, recompute, streams, total_rounds, **kw):
    """Lockstep engine run: updates to docs[j+1] land after update_after[j] rounds."""
    eng = Engine(policy_from_dict(docs[0]), recompute, start_paused=True,
                 max_streams=kw.pop("max_streams", 16), max_seq_len=kw.pop("max_seq_len", 256), **kw)
    ids = []
    opened = set()
    done = 0
    boundaries = sorted(set(update_after) | {s.get("open_after", 0) for s in streams} | {total_rounds})
    v = 0
    for b in boundaries:
        if b > done:
            eng.advance(b - done)
            done = b
        for j, ua in enumerate(update_after):
            if ua == b and v == j:
                res = eng.apply_weight_update(j + 1, policy_from_dict(docs[j + 1]))
                assert res.applied, res
                v += 1
        for i, s in enumerate(streams):
            if i not in opened and s.get("open_after", 0) == b:
                ids.append((i, eng.open_stream(s["prompt_id"], s["max_tokens"], s["seed"],
                                               s.get("terminator", -1))))
                opened.add(i)
    eng.stop()
    out = {}
    for i, sid in ids:
        evs, reason = eng.collect(sid)
        out[i] = dict(tokens=[e.token for e in evs], logprobs=[e.logprob for e in evs],
                      versions=[e.weight_version for e in evs],
                      positions=[e.position for e in evs], finish=reason)
    eng.close()
    return [out[i] for i in range(len(streams))]


def assert_same(got, exp):
    assert got["tokens"] == exp["tokens"]
    assert got["versions"] == exp["versions"]
    assert got["positions"] == list(range(len(exp["tokens"])))
    a, b = np.array(got["logprobs"]), np.array(exp["logprobs"])
    assert np.all(np.abs(a - b) <= LP_REL * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("recompute", [False, True])
def test_cross_module_recurrent_matches_reference_mixed_sample(cuda, orc, recompute):
    """acceptance.cpp:405-457 / test_protocol.cpp:231-269: engine with updates at
    the schedule's switch points == mixed_policy_sample, seed for seed."""
    g = GOLDEN["cross_module"]
    docs = g["checkpoints"]
    streams = [dict(prompt_id="p", seed=s, max_tokens=16) for s in g["seeds"]]
    got = run_engine(docs, g["switch_points"], recompute, streams, 16)
    exp = g["stale" if not recompute else "recompute"]
    for gi, ei in zip(got, exp):
        assert_same(gi, dict(tokens=ei["tokens"], logprobs=ei["behavior_logprobs"],
                             versions=ei["behavior_versions"]))
        assert gi["finish"] == "length"


def test_demo_scenario_matches_reference_transcript(cuda):
    """drive_scenario demo_two_streams (test_protocol.cpp:271-287): version split at 5."""
    g = GOLDEN["demo_scenario"]
    streams = [dict(prompt_id="demo", seed=5, max_tokens=12), dict(prompt_id="demo", seed=6, max_tokens=12)]
    got = run_engine([g["v0"], g["v1"]], [5], False, streams, 12)
    for gi, ref in zip(got, g["streams"]):
        assert_same(gi, dict(tokens=[e[1] for e in ref["events"]], logprobs=[e[2] for e in ref["events"]],
                             versions=[e[3] for e in ref["events"]]))
        assert all(v == (0 if p < 5 else 1) for p, v in enumerate(gi["versions"]))


def test_three_versions_in_order(cuda):
    """test_protocol.cpp:210-229: one stream overlapping two updates."""
    g = GOLDEN["demo_scenario"]
    got = run_engine([g["v0"], g["v1"], g["v0"]], [3, 7], False,
                     [dict(prompt_id="demo", seed=8, max_tokens=12)], 12)[0]
    bounds = []
    for v in got["versions"]:
        if not bounds or bounds[-1] != v:
            bounds.append(v)
    assert bounds == [0, 1, 2]


@pytest.mark.parametrize("recompute", [False, True])
def test_large_recurrent_engine_matches_oracle(cuda, orc, recompute):
    """64 streams x 48 tokens, V=256 D=64, three in-flight updates, staggered opens."""
    base = random_recurrent_policy(orc, 256, 64, 0.3, 11)
    docs = drift_checkpoints(orc, base, 4, 0.05, 12)
    streams = [dict(prompt_id="p", seed=1000 + i, max_tokens=48 - (i % 5),
                    open_after=(i % 3) * 2) for i in range(64)]
    ua = [7, 15, 30]
    got = run_engine(docs, ua, recompute, streams, 60, max_streams=64)
    exp = orc.engine_lockstep(docs, ua, recompute, streams, 60, max_events=64)
    for gi, ei in zip(got, exp):
        assert_same(gi, ei)
        assert gi["finish"] == ei["finish"]


def test_tabular_engine_terminator_and_rejections(cuda, orc):
    g = GOLDEN["demo_scenario"]
    # terminator-first policy yields a single-event stream (test_protocol.cpp:111-122)
    term = {"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": 2, "context_order": 0,
            "default_logits": [-2000.0, 0.0], "rows": []}
    eng = Engine(policy_from_dict(term), start_paused=False, max_streams=4, max_seq_len=64)
    sid = eng.open_stream("x", 50, 3, 1)
    evs, reason = eng.collect(sid)
    assert [e.token for e in evs] == [1] and reason == "terminator"
    eng.close()
    # out-of-order updates rejected without side effects (test_protocol.cpp:161-185)
    eng = Engine(policy_from_dict(g["v0"]), max_streams=4, max_seq_len=64)
    r = eng.apply_weight_update(2, policy_from_dict(g["v1"]))
    assert not r.applied and r.error == "version_conflict" and eng.weight_version() == 0
    r = eng.apply_weight_update(0, policy_from_dict(g["v1"]))
    assert not r.applied and eng.weight_version() == 0
    bad = dict(g["v1"], vocab_size=7, default_logits=[0.0] * 7,
               rows=[dict(r, logits=r["logits"] + [0.0]) for r in g["v1"]["rows"]])
    r = eng.apply_weight_update(1, policy_from_dict(bad))
    assert not r.applied and r.error == "policy_mismatch"
    tainted, _ = eng.collect(eng.open_stream("demo", 12, 4))
    eng.close()
    clean = run_engine([g["v0"]], [], False, [dict(prompt_id="demo", seed=4, max_tokens=12)], 12)[0]
    assert [e.token for e in tainted] == clean["tokens"]
    assert [e.weight_version for e in tainted] == [0] * 12


def test_free_running_updates_are_token_atomic(cuda, orc):
    """acceptance criterion 9: 8 free-running streams, 4 updates; every event's
    log-prob equals its stamped version's policy on the emitted prefix."""
    g = GOLDEN["demo_scenario"]
    v0, v1 = g["v0"], g["v1"]
    eng = Engine(policy_from_dict(v0), max_streams=8, max_seq_len=64, rounds_per_sync=1)
    sids = [eng.open_stream("demo", 48, 100 + i) for i in range(8)]
    versions = {0: v0}
    for v in range(1, 5):
        nxt = v1 if v % 2 else v0
        versions[v] = nxt
        assert eng.apply_weight_update(v, policy_from_dict(nxt)).applied
    for sid in sids:
        evs, reason = eng.collect(sid)
        assert len(evs) == 48 and reason == "length"
        prefix = []
        prev = 0
        for t, e in enumerate(evs):
            assert e.position == t and e.weight_version >= prev
            prev = e.weight_version
            lp = orc.policy_logprobs(versions[e.weight_version], "demo", prefix + [e.token])[-1]
            assert abs(e.logprob - lp) <= LP_REL * max(1.0, abs(lp))
            prefix.append(e.token)
    assert eng.active_streams() == 0
    eng.close()


def test_policy_logprobs_toy(cuda, orc):
    from paper_2509_19128_b200 import rlmath

    base = random_recurrent_policy(orc, 9, 5, 0.8, 123)
    toks = [0, 3, 8, 1, 1, 7]
    got = rlmath.policy_logprobs(policy_from_dict(base), "p", toks)
    exp = orc.policy_logprobs(base, "p", toks)
    assert np.allclose(got, exp, rtol=LP_REL, atol=0)
    g = GOLDEN["demo_scenario"]
    got = rlmath.policy_logprobs(policy_from_dict(g["v0"]), "demo", [0, 3, 3, 1])
    exp = orc.policy_logprobs(g["v0"], "demo", [0, 3, 3, 1])
    assert np.allclose(got, exp, rtol=LP_REL, atol=0)
    with pytest.raises(ValueError):
        rlmath.policy_logprobs(policy_from_dict(g["v0"]), "demo", [6])


def test_wait_events_many_matches_per_stream_drain(cuda):
    """The batched drain (one native call for many streams) returns what
    per-stream wait_events returns on an identical engine, including a stream
    that finished and one whose events stay behind for the next call."""
    g = GOLDEN["demo_scenario"]

    def run(batched):
        eng = Engine(policy_from_dict(g["v0"]), start_paused=True, max_streams=4, max_seq_len=64)
        sids = [eng.open_stream("demo", n, 7 + i) for i, n in enumerate([3, 9, 9])]
        got = []
        for _ in range(3):
            eng.advance(4)
            if batched:
                d = eng.wait_events_many(sids)
                got.append([(d[s][0], d[s][1], d[s][2]) for s in sids])
            else:
                got.append([eng.wait_events(s) for s in sids])
        eng.close()
        return got

    a, b = run(True), run(False)
    assert [[(evs, r, m) for evs, r, m in step] for step in a] == [[tuple(x) for x in step] for step in b]
    assert a[0][0][1] == "length" and len(a[0][1][0]) == 4
    # the columnar form carries the same fields
    eng = Engine(policy_from_dict(g["v0"]), start_paused=True, max_streams=4, max_seq_len=64)
    sids = [eng.open_stream("demo", n, 7 + i) for i, n in enumerate([3, 9, 9])]
    eng.advance(4)
    cols = eng.wait_events_many(sids, columns=True)
    for s, (evs, r, m) in zip(sids, a[0]):
        c, rc, mc = cols[s]
        assert (rc, mc) == (r, m) and c.token.tolist() == [e.token for e in evs]
        assert c.logprob.tolist() == [e.logprob for e in evs] and c.position.tolist() == [e.position for e in evs]
        assert c.weight_version.tolist() == [e.weight_version for e in evs]
    eng.close()


def test_poll_events_does_not_block(cuda):
    """srl_engine_poll_events_many: a paused engine's fresh stream has nothing
    queued -- polling returns at once (no events, still running) where
    wait_events would block; after advance() the events arrive in order."""
    g = GOLDEN["demo_scenario"]
    eng = Engine(policy_from_dict(g["v0"]), start_paused=True, max_streams=4, max_seq_len=64)
    sid = eng.open_stream("demo", 5, 7)
    got = eng.wait_events_many([sid], columns=True, block=False)[sid]
    assert len(got[0]) == 0 and got[1] == "running" and got[2]
    eng.advance(5)
    evs, reason, more = eng.wait_events_many([sid], columns=True, block=False)[sid]
    assert evs.position.tolist() == [0, 1, 2, 3, 4]
    eng.close()
