"""The precise engine (srl_engine_options.precise): the activations between
the GEMMs travel as bf16 hi + lo pairs through the multi-kernel round, so
only q / k / v and the K/V cache are bf16.  Against the fp64 oracle with
those rounding points (DecoderOracle(rounding="kv")) the sampled tokens'
log-probs must sit within north_star's 1e-3 relative at every shape -- the
same shapes whose default (bf16-activation) round sits at the bf16-flip
floor in test_megakernel_gpu.py: 0.5B (24 layers), 1.5B (28 layers, hd 128,
contexts past 2048 keys), the 7B widths at batch 256."""
import numpy as np
import pytest

from oracle.decoder_oracle import DecoderOracle
from paper_2509_19128_b200.engine import Engine
from paper_2509_19128_b200.policy import QWEN25_05B, QWEN25_15B, DecoderConfig, DecoderPolicy

from .test_decoder_gpu import host_weights

pytestmark = pytest.mark.gpu

CFG7B2L = DecoderConfig("qwen2.5-7b-2l", 152064, 3584, 2, 28, 4, 128, 18944, False, 151643, 4096)


@pytest.mark.parametrize("cfg,batch,lens,check", [
    (QWEN25_05B, 64, [0, 1, 33, 200, 700], (0, 1, 2, 3, 4, 30)),
    (QWEN25_15B, 16, [0, 5, 60, 2100], (0, 1, 2, 3, 9)),
    (CFG7B2L, 256, [0, 3, 40], (0, 1, 2, 100, 255)),
])
def test_precise_engine_logprobs_within_1e3(cuda, cfg, batch, lens, check):
    pol = DecoderPolicy.random(cfg, seed=31, scale=0.02)
    rng = np.random.default_rng(17)
    lens = list(lens) + list(rng.integers(1, 30, size=batch - len(lens)))
    prompts = [rng.integers(0, cfg.vocab_size, size=int(n)).tolist() for n in lens]
    steps = 4
    eng = Engine(pol, start_paused=True, precise=True, max_streams=batch,
                 max_seq_len=max(lens) + steps + 8, prefill_budget=max(4096, sum(lens) + batch))
    sids = [eng.open_stream("p", steps, 500 + i, -1, pr) for i, pr in enumerate(prompts)]
    eng.profile_next_round()
    eng.advance(steps + 4)
    assert "decode_megakernel" not in eng.kernel_profile()
    out = {i: eng.collect(sids[i])[0] for i in check}
    eng.close()
    m = DecoderOracle(cfg.to_dict(), host_weights(pol), np.float64, rounding="kv")
    worst = 0.0
    for i, evs in out.items():
        assert [e.position for e in evs] == list(range(steps))
        cache = m.new_cache()
        logits = m.prefill_fast(cache, [cfg.bos_token] + prompts[i])
        for e in evs:
            exp = DecoderOracle.log_softmax(logits)[e.token]
            worst = max(worst, abs(e.logprob - exp) / abs(exp))
            assert abs(e.logprob - exp) <= 1e-3 * abs(exp), (i, e.position, e.logprob, exp)
            logits = m.step([cache], [e.token], [len(cache["tokens"])])[0]
    print(f"{cfg.name} precise engine: max relative log-prob error {worst:.2e}")
