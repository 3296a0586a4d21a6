"""paper_2509_19128_b200.partition (the generator / trainer split of one box)
against the reference's own analytical model (throughput.cpp:36-65,
123-137, 260-330), compiled from /root/reference into oracle/_ref: the
same (H, I) choice and bit-identical rates on randomised specs, including
padding and every length law."""
import numpy as np
import pytest

from paper_2509_19128_b200.partition import (LengthDistribution, UtilizationCurve, curve_from_measurement,
                                             search_configs)


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import REF_SO, Ref

    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Ref()


def random_spec(rng):
    n = int(rng.integers(2, 9))
    hs = np.unique(rng.integers(1, 300, size=int(rng.integers(1, 8)))).astype(float)
    us = np.sort(rng.uniform(0.01, 1.0, size=len(hs)))
    kind = ["uniform", "constant", "empirical"][int(rng.integers(0, 3))]
    max_len = int(rng.integers(1, 9000))
    values = rng.integers(1, max_len + 1, size=int(rng.integers(1, 20))).tolist() if kind == "empirical" else []
    if kind == "empirical":
        max_len = max(values)
    return dict(n=n, train_batch=int(rng.integers(1, 300)), curve=[[float(h), float(u)] for h, u in zip(hs, us)],
                padding_window=int(rng.integers(0, 80)), tau=float(rng.uniform(0.5, 20.0)),
                lengths=dict(kind=kind, max_len=max_len, values=values), cap=int(rng.integers(1, 40)),
                use_padding=bool(rng.integers(0, 2)))


def ours(spec):
    curve = UtilizationCurve([tuple(p) for p in spec["curve"]], spec["padding_window"])
    L = spec["lengths"]
    return search_configs(spec["n"], spec["train_batch"], curve, spec["tau"],
                          LengthDistribution(L["kind"], L["max_len"], L["values"]), spec["cap"],
                          spec["use_padding"])


def test_search_configs_matches_reference(ref):
    rng = np.random.default_rng(2509)
    for _ in range(200):
        spec = random_spec(rng)
        exp = ref.search_configs(spec)
        got = ours(spec)
        assert got.feasible == exp["feasible"]
        if got.feasible:
            assert (got.gen_batch, got.inference_count, got.max_lag) == \
                (exp["gen_batch"], exp["inference_count"], exp["max_lag"]), spec
            assert (got.r_gen, got.r_train, got.r_total) == (exp["r_gen"], exp["r_train"], exp["r_total"])


def test_curve_from_measurement_units():
    # tokens/s x flash seconds: 2 * 1e9 flops per token at 1e15 flop/s -> 2 us per flash
    c = curve_from_measurement([(64, 50_000.0), (1, 1_000.0)], 2e9, 1e15)
    assert c.samples == [(1.0, 1000.0 * 2e-6), (64.0, 50_000.0 * 2e-6)]
    assert c.value_at(32.5) == pytest.approx(0.002 + (31.5 / 63) * (0.1 - 0.002))
