"""Host-side trainer math against the reference: fit_baseline on the golden
gradient trajectories (rl_math.cpp:165-179, bit for bit) and the analytic lag
bound pipeline_max_lag_steps (throughput.cpp:260-269) against the reference
itself (oracle/_ref) and the C oracle."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2509_19128_b200.rlmath import Trajectory, fit_baseline, pipeline_max_lag_steps

G = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def test_fit_baseline_matches_reference_golden():
    trajs = [Trajectory(t["prompt_id"], t["tokens"], t["behavior_logprobs"], t["behavior_versions"],
                        t["reward"]) for t in G["gradients"]["cases"][0]["trajectories"]]
    table = fit_baseline(trajs)
    exp = {(p, t): v for p, t, v in G["gradients"]["baseline_example"]}
    assert set(table.values) == set(exp)
    for k, v in exp.items():
        assert table.at(*k) == v  # bit-exact (same summation order)
    with pytest.raises(ValueError):
        table.at("p", 99)  # a missing cell throws (trajectory.cpp:35-41)
    with pytest.raises(ValueError):
        fit_baseline([])


def test_fit_baseline_every_golden_case():
    from oracle.oracle import Oracle

    orc = Oracle()
    for case in G["gradients"]["cases"]:
        trajs = [Trajectory(t["prompt_id"], t["tokens"], t["behavior_logprobs"], t["behavior_versions"],
                            t["reward"]) for t in case["trajectories"]]
        table = fit_baseline(trajs)
        _, _, base = orc.reinforce_gradient_tab(case["policy"], case["trajectories"])
        for k, v in base.items():
            assert table.at(*k) == v


CASES = [(4, 1, 8.0, 8.0, 4), (4, 2, 8.0, 8.0, 4), (4, 4, 8.0, 8.0, 4), (64, 1, 256.0, 190.5, 64),
         (64, 4, 8192.0, 4100.0, 256), (256, 6, 4096.0, 1500.25, 512), (1, 1, 1.0, 1.0, 1),
         (64, 7, 8192.0, 8192.0, 64)]


def test_pipeline_max_lag_steps_matches_c_oracle():
    from oracle.oracle import Oracle

    orc = Oracle()
    for c in CASES:
        assert pipeline_max_lag_steps(*c) == orc.pipeline_max_lag_steps(*c)
    for bad in [(0, 1, 8.0, 8.0, 4), (4, 0, 8.0, 8.0, 4), (4, 1, 0.0, 8.0, 4), (4, 1, 8.0, 8.0, 0)]:
        with pytest.raises(ValueError):
            pipeline_max_lag_steps(*bad)


def test_pipeline_max_lag_steps_matches_reference():
    from oracle.oracle import REF_SO, Ref

    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    ref = Ref()
    for c in CASES:
        assert pipeline_max_lag_steps(*c) == ref.pipeline_max_lag_steps(*c)
    rng = np.random.default_rng(0)
    for _ in range(200):
        c = (int(rng.integers(1, 300)), int(rng.integers(1, 9)), float(rng.integers(1, 9000)),
             float(rng.uniform(1, 9000)), int(rng.integers(1, 600)))
        assert pipeline_max_lag_steps(*c) == ref.pipeline_max_lag_steps(*c)
