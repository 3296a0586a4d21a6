"""kl_per_position (rl_math.cpp:336-372) for the decoder policy on the device
(srl_decoder_kl_per_position, csrc/kl.cpp): the section 5.1 mixed
behaviour policy -- checkpoints switching on MixedPolicySchedule::make's
points (rl_math.cpp:286-310) with a stale (PipelineRL) or recomputed KV
cache -- against the decoder oracle walking the same prefixes
(oracle/decoder_oracle.py, fp64: stale = keep the cache, recompute =
DecoderOracle.recompute at each switch, as in tests/test_engine_gpu.py), the
reference's identities (test_rl_math.cpp:391-427) and the ordering of
acceptance.cpp:322-355 (mixed behaviour closer to the target than the first
checkpoint alone)."""
import numpy as np
import pytest
import torch

from oracle.decoder_oracle import DecoderOracle
from paper_2509_19128_b200 import rlmath
from paper_2509_19128_b200.policy import TINY, DecoderPolicy

pytestmark = pytest.mark.gpu


def host(p):
    return p.torch_weights().cpu().view(torch.int16).numpy().view(np.uint16)


def oracle_kl(cks, switch, recompute, target, prefixes):
    models = [DecoderOracle(TINY.to_dict(), host(p)) for p in cks]
    tm = DecoderOracle(TINY.to_dict(), host(target))
    n = max(len(p) for p in prefixes)
    sums, counts = np.zeros(n), np.zeros(n)
    for pre in prefixes:
        cache, tcache = models[0].new_cache(), tm.new_cache()
        cur = 0
        for t in range(len(pre)):
            g = min(sum(1 for s in switch if t >= s), len(cks) - 1)
            if g != cur and recompute:
                models[g].recompute(cache)
            cur = g
            inp = TINY.bos_token if t == 0 else pre[t - 1]
            lp = DecoderOracle.log_softmax(models[g].step([cache], [inp], [t])[0])
            lq = DecoderOracle.log_softmax(tm.step([tcache], [inp], [t])[0])
            p = np.exp(lp)
            sums[t] += max(float(np.sum(np.where(p > 0, p * (lp - lq), 0.0))), 0.0)
            counts[t] += 1
    return sums / np.maximum(counts, 1)


@pytest.fixture(scope="module")
def chain(cuda):
    base = DecoderPolicy.random(TINY, seed=31, scale=0.05)
    cks = [base]
    for i in range(4):  # drift_checkpoints analogue: each one a perturbation of the last
        cks.append(cks[-1].clone().perturb(100 + i, 0.01))
    rng = np.random.default_rng(3)
    prefixes = [rng.integers(0, TINY.vocab_size, size=n).tolist() for n in (24, 20, 9, 24)]
    return cks, prefixes


@pytest.mark.parametrize("recompute", [False, True])
def test_mixed_kl_matches_oracle(chain, recompute):
    cks, prefixes = chain
    switch = rlmath.mixed_schedule(24, 4)
    assert switch == [12, 18]  # 2L/g, then every L/g (test_rl_math.cpp:322-343)
    target = cks[-1]
    got = rlmath.kl_per_position(cks[:3], switch, recompute, target, prefixes)
    exp = oracle_kl(cks[:3], switch, recompute, target, prefixes)
    assert got.shape == exp.shape == (24,)
    # the KLs are O(1e-3); device logits agree with the oracle's to bf16
    # rounding flips, so the KL agrees to a few percent of itself
    np.testing.assert_allclose(got, exp, rtol=5e-2, atol=2e-6)


def test_kl_identities_and_ordering(chain):
    cks, prefixes = chain
    target = cks[-1]
    # identical behaviour and target: identically zero (test_rl_math.cpp:416-427)
    z = rlmath.kl_per_position([target], [], False, target, prefixes)
    assert np.all(z == 0.0)
    # acceptance.cpp:322-355: the mixed behaviour (stale or recomputed) sits
    # closer to the final checkpoint than the first checkpoint alone
    switch = rlmath.mixed_schedule(24, 4)
    conv = rlmath.kl_per_position([cks[0]], [], False, target, prefixes).mean()
    stale = rlmath.kl_per_position(cks[:3], switch, False, target, prefixes).mean()
    rec = rlmath.kl_per_position(cks[:3], switch, True, target, prefixes).mean()
    assert stale < conv and rec < conv
    # the two modes differ exactly after the first switch, agree before it
    a = rlmath.kl_per_position(cks[:3], switch, False, target, prefixes)
    b = rlmath.kl_per_position(cks[:3], switch, True, target, prefixes)
    assert np.array_equal(a[:12], b[:12]) and not np.array_equal(a[12:], b[12:])
