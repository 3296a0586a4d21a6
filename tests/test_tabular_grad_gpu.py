"""Device is_reinforce_gradient / reinforce_gradient for the reference's
TabularPolicy (srl_tabular_is_reinforce_gradient, csrc/tabular_grad.cu)
against the 16 gradient cases the unmodified reference produced
(tests/golden/reference_vectors.json, rl_math.cpp:211-276), and the
reference's own gradient unit tests restated (test_rl_math.cpp:200-287).

Bar: 1e-12 relative -- the device accumulates every row in the reference's
order with separately rounded mul / add; only its exp / log differ from
glibc's by at most an ulp."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2509_19128_b200 import rlmath
from paper_2509_19128_b200.policy import TabularPolicy, policy_from_dict

pytestmark = pytest.mark.gpu

G = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def trajs_of(case):
    return [rlmath.Trajectory(t["prompt_id"], t["tokens"], t["behavior_logprobs"],
                              t.get("behavior_versions", [0] * len(t["tokens"])), t["reward"])
            for t in case["trajectories"]]


def close(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("i", range(len(G["gradients"]["cases"])))
def test_tabular_gradient_matches_reference_vectors(cuda, i):
    case = G["gradients"]["cases"][i]
    pol = policy_from_dict(case["policy"])
    trajs = trajs_of(case)
    base = rlmath.fit_baseline(trajs)
    gran = "per_token" if case["granularity"] == 1 else "sequence"
    if case["use_is"]:
        g = rlmath.is_reinforce_gradient(pol, trajs, base, case["clamp"], gran)
    else:
        g = rlmath.reinforce_gradient(pol, trajs, base)
    exp_rows = {(r["prompt_id"], tuple(r["context"])): r["grad"] for r in case["grad"]["rows"]}
    assert set(g.rows) == set(exp_rows)  # rows created exactly where the reference created them
    for k, row in exp_rows.items():
        close(g.rows[k], row)
    dr = case["grad"]["default_row"]
    if dr:
        close(g.default_row, dr)
    else:
        assert g.default_row is None


def single_row(logits):
    return TabularPolicy(len(logits), 0, {("p", ()): np.array(logits, dtype=np.float64)}, None)


def test_hand_value_and_missing_cell(cuda):
    """test_rl_math.cpp:225-243."""
    p = single_row([0.0, 0.0])
    t = rlmath.Trajectory("p", [1], [math.log(0.5)], [0], 1.0)
    g = rlmath.reinforce_gradient(p, [t], rlmath.BaselineTable({("p", 0): 0.0}))
    close(g.rows[("p", ())], [-0.5, 0.5])
    t2 = rlmath.Trajectory("p", [1, 0], [math.log(0.5)] * 2, [0, 0], 1.0)
    with pytest.raises(ValueError):
        rlmath.reinforce_gradient(p, [t2], rlmath.BaselineTable({("p", 0): 0.0}))


def test_single_sample_baseline_gives_zero_gradient(cuda):
    """test_rl_math.cpp:217-223: a one-sample baseline zeroes every advantage,
    so no row is touched."""
    p = TabularPolicy(3, 0, {}, None)
    t = rlmath.Trajectory("p", [1, 2], [math.log(1 / 3)] * 2, [0, 0], 1.0)
    g = rlmath.reinforce_gradient(p, [t], rlmath.fit_baseline([t]))
    assert g.max_abs() == 0.0


def test_clamp_is_exactly_five_x(cuda):
    """test_rl_math.cpp:273-287."""
    p = single_row([0.0, 0.0])
    t = rlmath.Trajectory("p", [1], [math.log(0.5) - math.log(64.0)], [0], 1.0)
    b = rlmath.BaselineTable({("p", 0): 0.0})
    plain = rlmath.reinforce_gradient(p, [t], b)
    clamped = rlmath.is_reinforce_gradient(p, [t], b, 5.0)
    assert clamped.rows[("p", ())][1] == pytest.approx(5.0 * plain.rows[("p", ())][1], rel=1e-12)
    tiny = rlmath.is_reinforce_gradient(p, [t], b, 1e-300)
    assert tiny.max_abs() < 1e-290
    with pytest.raises(ValueError):
        rlmath.is_reinforce_gradient(p, [t], b, 0.0)


def test_on_policy_is_equals_plain(cuda):
    """test_rl_math.cpp:258-271: behaviour = current policy -> every IS weight
    is exactly 1 in both granularities."""
    keys = [("p", ())] + [("p", (k,)) for k in range(4)]
    rng = np.random.default_rng(3)
    pol = TabularPolicy(4, 1, {k: rng.normal(0, 0.7, 4) for k in keys}, None)
    trajs = []
    for i in range(8):
        toks = rng.integers(0, 4, size=6).tolist()
        lp = rlmath.policy_logprobs(pol, "p", toks).tolist()
        trajs.append(rlmath.Trajectory("p", toks, lp, [0] * 6, float(rng.random())))
    base = rlmath.fit_baseline(trajs)
    plain = rlmath.reinforce_gradient(pol, trajs, base)
    for gran in ("sequence", "per_token"):
        w = rlmath.is_reinforce_gradient(pol, trajs, base, 5.0, gran)
        assert set(w.rows) == set(plain.rows)
        for k in plain.rows:
            close(w.rows[k], plain.rows[k])
