"""Decoder policy on the device vs the CPU oracle (oracle/decoder_oracle.py,
oracle/streamrl_oracle.c).

Tolerances (north star): sampled token ids and version tags bit-exact given
the same logits; log-probs within 1e-3 relative (fp32 accumulation of bf16
GEMMs vs the oracle's fp64 accumulation), with a 2e-3 absolute floor.

The achievable agreement is bounded by bf16 rounding-boundary flips: a value
that lands within an fp32 ulp of a bf16 rounding boundary rounds differently
under different accumulation orders, and a flipped K/V entry persists in the
cache.  Measured: the oracle at fp32 vs fp64 accumulation disagrees with
itself by up to 7e-3 at init scale 0.1 and by <3e-4 at the realistic 0.02;
tests use scale 0.03 (test_oracle_self_consistency records the spread)."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle.decoder_oracle import DecoderOracle
from oracle.oracle import Oracle
from paper_2509_19128_b200 import _lib, rlmath
from paper_2509_19128_b200.engine import Engine
from paper_2509_19128_b200.policy import QWEN25_05B, TINY, DecoderPolicy

pytestmark = pytest.mark.gpu
LP_REL, LP_ABS = 1e-3, 2e-3


def lp_close(got, exp):
    got, exp = np.asarray(got), np.asarray(exp)
    err = np.abs(got - exp)
    assert np.all(err <= np.maximum(LP_ABS, LP_REL * np.abs(exp))), f"max err {err.max()}"


def host_weights(policy):
    return policy.torch_weights().cpu().view(torch.int16).numpy().view(np.uint16)


def oracle_for(policy, dtype=np.float64):
    return DecoderOracle(policy.config.to_dict(), host_weights(policy), dtype)


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def tiny(cuda):
    return DecoderPolicy.random(TINY, seed=3, scale=0.03)


def gpu_sample(logits, seeds, draws, greedy):
    rows, V = logits.shape
    tok = torch.empty(rows, dtype=torch.int32, device=logits.device)
    lp = torch.empty(rows, dtype=torch.float64, device=logits.device)
    _lib.call("srl_kernel_sample_logits", logits.data_ptr(), V, rows, seeds.data_ptr(),
              draws.data_ptr(), int(greedy), tok.data_ptr(), lp.data_ptr(), None)
    torch.cuda.synchronize()
    return tok.cpu().numpy(), lp.cpu().numpy()


@pytest.mark.parametrize("V,temp", [(256, 1.0), (256, 6.0), (151936, 1.0), (151936, 8.0), (7, 3.0)])
def test_sampler_bit_exact_on_dumped_logits(cuda, orc, V, temp):
    rows = 64
    g = torch.Generator(device=cuda).manual_seed(V)
    logits = (torch.randn(rows, V, device=cuda, generator=g) * temp).float()
    seeds = torch.tensor([(v if v < 2**63 else v - 2**64) for v in
                          (orc.derive_stream(99, i) for i in range(rows))], dtype=torch.int64,
                         device=cuda)
    draws = torch.arange(rows, dtype=torch.int32, device=cuda) % 17
    tok, lp = gpu_sample(logits, seeds, draws, False)
    host = logits.double().cpu().numpy()
    for r in range(rows):
        u = orc.uniforms(int(seeds[r].item()) & (2**64 - 1), int(draws[r]) + 1)[-1]
        t, l = orc.sample_from_logits(host[r], u)
        assert tok[r] == t
        assert abs(lp[r] - l) <= 1e-12 * max(1.0, abs(l))
    gt, glp = gpu_sample(logits, seeds, draws, True)
    for r in range(rows):
        assert gt[r] == orc.argmax(host[r])


def test_sampler_ties_and_fallback(cuda, orc):
    V = 1000
    logits = torch.zeros(3, V, device=cuda)
    logits[1, 500] = 5.0
    logits[1, 700] = 5.0          # tie: lowest index wins under greedy
    logits[2, :] = -1e30
    logits[2, 3] = 0.0            # one-hot row
    seeds = torch.tensor([1, 2, 3], dtype=torch.int64, device=cuda)
    draws = torch.zeros(3, dtype=torch.int32, device=cuda)
    gt, _ = gpu_sample(logits, seeds, draws, True)
    assert gt.tolist() == [0, 500, 3]
    st, lp = gpu_sample(logits, seeds, draws, False)
    assert st[2] == 3 and abs(lp[2]) < 1e-12


def test_policy_logprobs_tiny_matches_oracle(cuda, tiny):
    rng = np.random.default_rng(0)
    toks = rng.integers(0, TINY.vocab_size, size=40).tolist()
    got = rlmath.policy_logprobs(tiny, "p", toks)
    exp = oracle_for(tiny).sequence_logprobs(toks)
    lp_close(got, exp)


def run_decoder_engine(policy, prompts, max_tokens, greedy, seeds, updates=(), recompute=False,
                       staged=False, **kw):
    eng = Engine(policy, recompute, start_paused=True, greedy=greedy, max_streams=8,
                 max_seq_len=128, **kw)
    sids = [eng.open_stream("p", max_tokens, s, -1, pr) for pr, s in zip(prompts, seeds)]
    done = 0
    for v, (after, pol) in enumerate(updates, start=1):
        eng.advance(after - done)
        done = after
        if staged:
            ptr, nbytes = eng.begin_weight_update(v)
            src, n = pol.weights()
            assert n == nbytes
            torch.cuda.synchronize()
            # the device copy below stands in for the trainer's ncclBroadcast
            dst = torch.as_tensor(_Raw(ptr, nbytes), device="cuda")
            dst.copy_(torch.as_tensor(_Raw(src, nbytes), device="cuda"))
            torch.cuda.synchronize()
            res, pause = eng.commit_weight_update(v)
            assert res.applied and pause >= 0.0
        else:
            assert eng.apply_weight_update(v, pol).applied
    eng.advance(max_tokens - done + 2)
    out = []
    for sid in sids:
        evs, reason = eng.collect(sid)
        out.append((evs, reason, eng.stream_tokens(sid)))
    eng.close()
    return out


class _Raw:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


@pytest.mark.parametrize("greedy", [True, False])
def test_decoder_engine_teacher_forced(cuda, tiny, greedy):
    rng = np.random.default_rng(1)
    prompts = [rng.integers(0, 256, size=n).tolist() for n in (0, 1, 5, 17, 3, 30)]
    seeds = [11 + i for i in range(len(prompts))]
    res = run_decoder_engine(tiny, prompts, 20, greedy, seeds)
    orc_model = oracle_for(tiny)
    for (evs, reason, hist), pr in zip(res, prompts):
        assert reason == "length" and len(evs) == 20
        assert [e.position for e in evs] == list(range(20))
        assert all(e.weight_version == 0 for e in evs)
        assert hist == [TINY.bos_token] + pr + [e.token for e in evs]
        cache = orc_model.new_cache()
        logits = orc_model.prefill(cache, [TINY.bos_token] + pr)[-1]
        for e in evs:
            lp = DecoderOracle.log_softmax(logits)
            lp_close([e.logprob], [lp[e.token]])
            if greedy:
                top = np.sort(logits)[-2:]
                if top[1] - top[0] > 0.05:
                    assert e.token == int(np.argmax(logits))
            logits = orc_model.step([cache], [e.token], [len(cache["tokens"])])[0]


@pytest.mark.parametrize("recompute,staged", [(False, False), (True, False), (False, True)])
def test_decoder_inflight_update(cuda, tiny, recompute, staged):
    v1 = tiny.clone().perturb(77, 0.01)
    v2 = v1.clone().perturb(78, 0.01)
    rng = np.random.default_rng(2)
    prompts = [rng.integers(0, 256, size=n).tolist() for n in (4, 9, 2)]
    res = run_decoder_engine(tiny, prompts, 16, True, [1, 2, 3], updates=[(5, v1), (11, v2)],
                             recompute=recompute, staged=staged)
    models = [oracle_for(p) for p in (tiny, v1, v2)]
    for (evs, reason, _), pr in zip(res, prompts):
        vers = [e.weight_version for e in evs]
        assert vers == [0] * 5 + [1] * 6 + [2] * 5
        cache = models[0].new_cache()
        logits = models[0].prefill(cache, [TINY.bos_token] + pr)[-1]
        wrong = []
        for t, e in enumerate(evs):
            lp_close([e.logprob], [DecoderOracle.log_softmax(logits)[e.token]])
            if t == 5:  # the first token under v1, scored as if v0 were still live
                c0 = models[0].new_cache()
                l0 = models[0].prefill(c0, [TINY.bos_token] + pr + [x.token for x in evs[:5]])[-1]
                wrong.append(abs(DecoderOracle.log_softmax(l0)[e.token] - e.logprob))
            nv = vers[t + 1] if t + 1 < len(evs) else vers[t]
            m = models[nv]
            if nv != vers[t] and recompute:
                # recompute mode: the whole prefix is re-encoded under the new weights
                cache["tokens"].append(e.token)
                toks = list(cache["tokens"])
                cache.update(m.new_cache())
                logits = m.prefill(cache, toks)[-1]
            else:
                logits = m.step([cache], [e.token], [len(cache["tokens"])])[0]
        assert max(wrong) > 10 * LP_ABS  # the version split is observable at this tolerance


def test_qwen05b_shape_engine(cuda):
    """Qwen2.5-0.5B shape, constant batch 64: all slots stream, one stream
    checked teacher-forced against the fp32 oracle."""
    pol = DecoderPolicy.random(QWEN25_05B, seed=5, scale=0.02)
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, QWEN25_05B.vocab_size, size=8).tolist() for _ in range(64)]
    eng = Engine(pol, start_paused=True, max_streams=64, max_seq_len=64)
    sids = [eng.open_stream("p", 6, 100 + i, -1, pr) for i, pr in enumerate(prompts)]
    assert eng.advance(6) == 64 * 6
    evs, reason = eng.collect(sids[7])
    eng.close()
    assert reason == "length" and len(evs) == 6
    m = oracle_for(pol, np.float32)
    cache = m.new_cache()
    logits = m.prefill(cache, [QWEN25_05B.bos_token] + prompts[7])[-1].astype(np.float64)
    for e in evs:
        lp_close([e.logprob], [DecoderOracle.log_softmax(logits)[e.token]])
        logits = m.step([cache], [e.token], [len(cache["tokens"])])[0].astype(np.float64)


def test_lag_stats_kernel_matches_oracle(cuda, orc):
    rng = np.random.default_rng(4)
    for _ in range(5):
        n_seq = int(rng.integers(1, 40))
        vb = int(rng.integers(5, 60))
        seqs = []
        for _ in range(n_seq):
            L = int(rng.integers(1, 300))
            start = int(rng.integers(max(0, vb - 30), vb + 1))
            seqs.append(np.sort(rng.integers(start, vb + 1, size=L)).astype(np.int32))
        exp = orc.lag_stats(vb, seqs)
        vers = torch.tensor(np.concatenate(seqs), device=cuda)
        offs = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64,
                            device=cuda)
        hist = torch.zeros(128, dtype=torch.int64, device=cuda)
        sums = torch.zeros(n_seq, dtype=torch.int64, device=cuda)
        tot = torch.zeros(4, dtype=torch.int64, device=cuda)
        _lib.call("srl_lag_stats", vers.data_ptr(), offs.data_ptr(), n_seq, vb, hist.data_ptr(), 128,
                  sums.data_ptr(), tot.data_ptr(), None)
        torch.cuda.synchronize()
        h = {i: int(c) for i, c in enumerate(hist.cpu().tolist()) if c}
        assert h == exp["histogram"]
        assert sums.cpu().tolist() == exp["sequence_lag_sums"]
        t = tot.cpu().tolist()
        assert t[0] == exp["tokens"] and t[2] == exp["max_lag_steps"] and t[3] == 0
        assert t[1] / t[0] == exp["mean_lag_steps"]


def test_oracle_self_consistency(cuda, tiny):
    """The bound above: oracle(fp32 accumulate) vs oracle(fp64) vs device."""
    rng = np.random.default_rng(9)
    seq = rng.integers(0, 256, size=48).tolist()
    a = oracle_for(tiny).sequence_logprobs(seq)
    b = oracle_for(tiny, np.float32).sequence_logprobs(seq)
    g = rlmath.policy_logprobs(tiny, "p", seq)
    assert np.abs(a - b).max() < 1e-3
    lp_close(g, a)
