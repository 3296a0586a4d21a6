"""The reference wire protocol (docs/protocol.md) over the device engine:
paper_2509_19128_b200/server.py driven by a plain HTTP client, mirroring
tests/test_protocol.cpp of the reference (version split at the pause
boundary, three versions in order, rejection safety, checksum and group
id), on the reference's own demo policies (tests/golden)."""
import http.client
import json
import threading
import time

import pytest

from oracle.oracle import Oracle
from paper_2509_19128_b200.engine import Engine, crc32
from paper_2509_19128_b200.policy import policy_from_dict
from paper_2509_19128_b200.server import EngineServer, compact_json

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(__file__.replace("test_server_gpu.py", "golden/reference_vectors.json")))
V0, V1 = GOLDEN["demo_scenario"]["v0"], GOLDEN["demo_scenario"]["v1"]


class Client:
    def __init__(self, port):
        self.port = port

    def _req(self, method, path, body=None):
        c = http.client.HTTPConnection("127.0.0.1", self.port, timeout=60)
        data = None if body is None else json.dumps(body)
        c.request(method, path, body=data, headers={"Content-Type": "application/json"})
        r = c.getresponse()
        raw = r.read()
        c.close()
        return r.status, raw

    def post(self, path, body=None):
        st, raw = self._req("POST", path, body or {})
        return st, json.loads(raw) if raw else {}

    def get(self, path):
        st, raw = self._req("GET", path)
        return st, json.loads(raw)

    def generate(self, prompt_id, max_tokens, seed, terminator=-1):
        st, raw = self._req("POST", "/v1/chat/completions",
                            dict(prompt_id=prompt_id, max_tokens=max_tokens, seed=seed, terminator=terminator))
        assert st == 200
        lines = [json.loads(l) for l in raw.decode().splitlines() if l.strip()]
        assert lines[-1]["done"] is True
        return lines[:-1], lines[-1]["finish_reason"]

    def update(self, version, doc, checksum=None):
        return self.post("/request_weight_update",
                         dict(new_version=version, policy=doc,
                              checksum=crc32(compact_json(doc)) if checksum is None else checksum))


@pytest.fixture
def live(cuda):
    def make(start_paused):
        eng = Engine(policy_from_dict(V0), start_paused=start_paused, max_streams=8, max_seq_len=64)
        srv = EngineServer(eng).start()
        made.append((eng, srv))
        return eng, Client(srv.port)
    made = []
    yield make
    for eng, srv in made:
        eng.stop()
        srv.stop()
        eng.close()


def stream_async(client, *args):
    out = {}
    t = threading.Thread(target=lambda: out.update(res=client.generate(*args)))
    t.start()
    return t, out


def wait_streams(eng, n):
    t0 = time.time()
    while eng.total_streams() < n:
        assert time.time() - t0 < 30
        time.sleep(0.001)


def test_mid_stream_update_splits_versions_at_the_pause_boundary(live):
    eng, c = live(True)
    t, out = stream_async(c, "demo", 9, 11)
    wait_streams(eng, 1)
    assert c.post("/admin/advance", {"rounds": 4})[0] == 200
    st, body = c.update(1, V1)
    assert st == 200 and body == {"applied_version": 1}
    c.post("/admin/advance", {"rounds": 5})
    t.join(60)
    evs, reason = out["res"]
    assert reason == "length" and [e["position"] for e in evs] == list(range(9))
    assert [e["weight_version"] for e in evs] == [0] * 4 + [1] * 5
    # every event log-prob recomputed offline under its version (recompute_and_check)
    orc = Oracle()
    docs = {0: V0, 1: V1}
    toks = []
    for e in evs:
        lp = orc.policy_logprobs(docs[e["weight_version"]], "demo", toks + [e["token"]])[-1]
        assert abs(lp - e["logprob"]) <= 1e-9 * max(1.0, abs(lp))
        toks.append(e["token"])


def recompute_and_check(docs, evs, prompt="demo"):
    """Every event's log-prob recomputed offline under the version it carries
    (test_protocol.cpp recompute_and_check), positions contiguous."""
    orc = Oracle()
    toks = []
    assert [e["position"] for e in evs] == list(range(len(evs)))
    for e in evs:
        lp = orc.policy_logprobs(docs[e["weight_version"]], prompt, toks + [e["token"]])[-1]
        assert abs(lp - e["logprob"]) <= 1e-9 * max(1.0, abs(lp))
        toks.append(e["token"])


def test_two_concurrent_streams_complete_with_contiguous_positions(live):
    """test_protocol.cpp:93-104: two HTTP streams at once on a free-running
    engine (the per-thread event buffers of Engine.wait_events)."""
    eng, c = live(False)
    runs = [stream_async(c, "demo", 16, s) for s in (1, 2)]
    for t, out in runs:
        t.join(60)
        evs, reason = out["res"]
        assert len(evs) == 16 and reason == "length"
        assert [e["position"] for e in evs] == list(range(16))


def test_eight_concurrent_streams_with_four_free_running_updates(live):
    """test_protocol.cpp:314-336: eight streams while four updates land on the
    free-running engine; every event's log-prob matches its version."""
    eng, c = live(False)
    runs = [stream_async(c, "demo", 48, 1000 + i) for i in range(8)]
    docs = {0: V0}
    for v in range(1, 5):
        nxt = V1 if v % 2 == 1 else V0
        docs[v] = nxt
        st, body = c.update(v, nxt)
        assert st == 200 and body == {"applied_version": v}
    for t, out in runs:
        t.join(120)
        evs, reason = out["res"]
        assert len(evs) == 48
        recompute_and_check(docs, evs)
    assert c.get("/admin/state")[1]["active_streams"] == 0


def test_three_versions_in_order(live):
    eng, c = live(True)
    t, out = stream_async(c, "demo", 12, 8)
    wait_streams(eng, 1)
    c.post("/admin/advance", {"rounds": 3})
    assert c.update(1, V1)[0] == 200
    c.post("/admin/advance", {"rounds": 4})
    assert c.update(2, V0)[0] == 200
    c.post("/admin/advance", {"rounds": 5})
    t.join(60)
    evs, _ = out["res"]
    seen = []
    for e in evs:
        if not seen or seen[-1] != e["weight_version"]:
            seen.append(e["weight_version"])
    assert len(evs) == 12 and seen == [0, 1, 2]


def test_rejections_leave_the_engine_untouched(live):
    eng, c = live(False)
    st, body = c.update(2, V1)
    assert st == 409 and body["error"] == "version_conflict" and body["current_version"] == 0
    st, body = c.update(0, V1)
    assert st == 409 and body["error"] == "version_conflict"
    st, body = c.update(1, V1, checksum=12345)
    assert st == 400 and body["error"] == "checksum_mismatch"
    st, body = c.update(1, dict(V1, vocab_size=V1["vocab_size"] + 1))  # invalid / mismatched policy
    assert st == 400 and body["error"].split(":")[0] in ("invalid_policy", "policy_mismatch")
    st, body = c.post("/request_weight_update", {"new_version": 1})
    assert st == 400 and body["error"].startswith("bad_request")
    assert c.get("/healthz")[1]["weight_version"] == 0
    tainted, _ = c.generate("demo", 12, 4)
    _, control = live(False)
    clean, _ = control.generate("demo", 12, 4)
    assert [e["token"] for e in tainted] == [e["token"] for e in clean]
    assert [e["logprob"] for e in tainted] == [e["logprob"] for e in clean]
    assert all(e["weight_version"] == 0 for e in tainted)
    st, body = c.update(1, V1)
    assert st == 200 and c.get("/admin/state")[1]["weight_version"] == 1


def test_process_group_id_is_order_free_and_checksum_known_answer(live):
    eng, c = live(False)
    st, a = c.post("/init_process_group", {"members": ["127.0.0.1:8317", "127.0.0.1:8318"]})
    st2, b = c.post("/init_process_group", {"members": ["127.0.0.1:8318", "127.0.0.1:8317"]})
    assert st == st2 == 200 and a == b and a["size"] == 2 and a["group_id"].startswith("pg-")
    assert c.get("/admin/state")[1]["group_id"] == a["group_id"]
    assert crc32(b"123456789") == 0xCBF43926  # test_protocol.cpp:76-79
