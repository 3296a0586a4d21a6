import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle.decoder_oracle import DecoderOracle
from paper_2509_19128_b200.policy import QWEN25_05B, QWEN25_15B, DecoderPolicy
from tests.test_decoder_gpu import oracle_for
for cfg in (QWEN25_05B, QWEN25_15B):
    pol = DecoderPolicy.random(cfg, seed=9, scale=0.02)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, cfg.vocab_size, size=40).tolist()
    res = []
    for dt in (np.float32, np.float64):
        t = time.time()
        m = oracle_for(pol, dt)
        c = m.new_cache()
        lg = m.prefill(c, [cfg.bos_token] + toks[:30])[-1].astype(np.float64)
        lps = []
        for tk in toks[30:]:
            lps.append(DecoderOracle.log_softmax(lg)[tk])
            lg = m.step([c], [tk], [len(c["tokens"])])[0].astype(np.float64)
        res.append(np.array(lps)); del m
        print(cfg.name, dt.__name__, time.time() - t, flush=True)
    print(cfg.name, "fp32 vs fp64 oracle |dlp|:", np.abs(res[0] - res[1]))
