"""The /request_weight_update checksum interop: server.py's compact_json of a
policy document must be byte-identical to what the reference client
checksums -- json::parse(policy_to_json(policy)).dump() (protocol.cpp:340-356,
nlohmann 3.11.3) -- and srl_crc32 of it equal to the reference crc32, for
the reference's demo policies and random tabular / recurrent documents
(awkward doubles: tiny, huge, negative zero, many digits)."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2509_19128_b200.engine import crc32
from paper_2509_19128_b200.policy import policy_from_dict, policy_to_dict
from paper_2509_19128_b200.server import compact_json

G = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import REF_SO, Ref

    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Ref()


def docs():
    out = [G["demo_scenario"]["v0"], G["demo_scenario"]["v1"]] + list(G["cross_module"]["checkpoints"])
    rng = np.random.default_rng(11)
    vals = [0.0, -0.0, 1.0, -2.5, 1e-300, 1e300, 5e-324, 123456789.123456789, 0.1, 1 / 3, 2.0 ** 60]
    for k in range(6):
        V = int(rng.integers(2, 7))
        rows = [{"prompt_id": "p", "context": [], "logits": [float(x) for x in rng.standard_normal(V) * 10 ** k]},
                {"prompt_id": "q", "context": [1], "logits": [vals[(i + k) % len(vals)] for i in range(V)]}]
        out.append({"schema": "streamrl.policy/1", "type": "tabular", "vocab_size": V, "context_order": 1,
                    "default_logits": [float(x) for x in rng.standard_normal(V)], "rows": rows})
    return out


def test_compact_json_matches_reference_dump(ref):
    for doc in docs():
        # what our client sends: the document of the policy as the package holds it
        ours = compact_json(policy_to_dict(policy_from_dict(doc)))
        exp = ref.policy_wire(doc)
        assert ours.decode() == exp["bytes"]
        assert crc32(ours) == exp["crc32"]
