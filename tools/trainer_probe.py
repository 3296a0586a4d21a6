#!/usr/bin/env python
"""One trainer step (IS-REINFORCE fwd + bwd + Adam) at a Qwen2.5 shape, for
profiling: python tools/trainer_probe.py [--config qwen2.5-0.5b] [--seqs 64]
[--len 321] [--steps 2] [--fast]"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200.policy import PRESETS, DecoderPolicy  # noqa: E402
from paper_2509_19128_b200.trainer import Trainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen2.5-0.5b")
ap.add_argument("--seqs", type=int, default=64)
ap.add_argument("--len", type=int, default=321)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--fast", action="store_true", help="single bf16 operands instead of the precise mode")
a = ap.parse_args()
cfg = PRESETS[a.config]
pol = DecoderPolicy.random(cfg, seed=0, scale=0.02)
rng = np.random.default_rng(0)
trajs = []
for i in range(a.seqs):
    toks = [cfg.bos_token] + rng.integers(0, cfg.vocab_size, size=a.len - 1).tolist()
    trajs.append(dict(tokens=toks, loss_begin=65, behavior_logprobs=[-12.0] * a.len,
                      advantages=[float(rng.standard_normal())] * a.len))
tr = Trainer(pol, max_tokens=a.seqs * a.len, precise=not a.fast)
for s in range(a.steps):
    r = tr.step(trajs)
    tr.apply_adam(1e-6)
    torch.cuda.synchronize()
    g = tr.gradient()
    print(f"step {s}: {r.step_ms:.1f} ms (forward {r.forward_ms:.1f}), {r.tokens} tokens, J={r.objective:.3e} ess={r.ess:.3f} |g|={g.norm().item():.3e} finite={bool(torch.isfinite(g).all())}", flush=True)
