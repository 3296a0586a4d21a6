"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU, exports every symbol include/streamrl_b200.h declares, the ctypes
signature table covers them, host-only helpers match the reference, and
compute entry points fail loudly (no CPU fallback) when no device is visible."""
import ctypes as C
import json
from pathlib import Path

import pytest

from paper_2509_19128_b200 import _lib
from paper_2509_19128_b200.policy import (QWEN25_05B, QWEN25_15B, QWEN25_7B, TINY, TabularPolicy,
                                          policy_from_json, policy_to_json)

G = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 40
    missing = [n for n in declared if not hasattr(lib, n)]
    assert missing == []
    assert sorted(_lib.SIGNATURES) == declared


def test_status_strings_map_reference_errors():
    lib = _lib.lib()
    assert lib.srl_status_string(1) == b"version_conflict"
    assert lib.srl_status_string(2) == b"invalid_policy"
    assert lib.srl_status_string(3) == b"policy_mismatch"
    assert lib.srl_status_string(4) == b"checksum_mismatch"


def test_crc32_and_process_group_id_match_reference():
    from paper_2509_19128_b200.engine import crc32, process_group_id

    for text, v in G["protocol"]["crc32"]:
        assert crc32(text.encode()) == v
    for members, gid in G["protocol"]["group_ids"]:
        assert process_group_id(members) == gid
    with pytest.raises(ValueError):
        process_group_id([])


def test_host_trainer_helpers_match_reference():
    from paper_2509_19128_b200 import rlmath

    for pi, mu, c, w in G["is_ess"]["truncated"]:
        assert rlmath.truncated_is_weight(pi, mu, c) == w
    for w, e in G["is_ess"]["ess"]:
        assert rlmath.ess(w) == e
    with pytest.raises(rlmath.EssUndefinedError):
        rlmath.ess([0.0, 0.0])
    with pytest.raises(ValueError):
        rlmath.truncated_is_weight(0.0, 0.0, 0.0)


def test_decoder_weight_bytes_and_presets():
    for cfg, params in ((QWEN25_05B, 494e6), (QWEN25_15B, 1544e6), (QWEN25_7B, 7616e6)):
        nbytes = _lib.lib().srl_decoder_weight_bytes(C.byref(cfg.native()))
        assert abs(nbytes / 2 - cfg.params()) / cfg.params() < 1e-3
        assert abs(cfg.params() - params) / params < 0.01
    assert _lib.lib().srl_decoder_weight_bytes(C.byref(TINY.native())) > 0


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    st = _lib.lib().srl_policy_decoder_create(C.byref(TINY.native()), 0, 0.02, 0, C.byref(h))
    assert st == 10  # SRL_NO_DEVICE
    from paper_2509_19128_b200.engine import Engine

    with pytest.raises(_lib.SrlError):
        Engine(policy_from_json(json.dumps(G["demo_scenario"]["v0"])))


def test_policy_documents_round_trip():
    for doc in (G["demo_scenario"]["v0"], G["cross_module"]["checkpoints"][1]):
        p = policy_from_json(json.dumps(doc))
        again = json.loads(policy_to_json(p))
        for k, v in doc.items():
            if isinstance(v, list) and v and isinstance(v[0], dict):
                assert [dict(r, logits=[float(x) for x in r["logits"]]) for r in v] == again[k]
            else:
                assert again[k] == v
    t = TabularPolicy(3, 1, {("b", (1,)): [0, 0, 0], ("a", ()): [1, 2, 3], ("a", (0,)): [0, 1, 0]})
    assert [k for k, _ in t.rows()] == [("a", ()), ("a", (0,)), ("b", (1,))]
