#!/usr/bin/env python
"""PipelineRL loop on one GPU (generator and trainer time-shared): constant
generation batch, host actor queue, IS-REINFORCE trainer, in-flight weight
update every optimizer step.  Prints one JSON line per run.

  python tools/pipeline_demo.py --config tiny --steps 30
  python tools/pipeline_demo.py --config qwen2.5-0.5b --batch 64 --max-tokens 256 --steps 6
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200.pipeline import PipelineRL  # noqa: E402
from paper_2509_19128_b200.policy import PRESETS, DecoderPolicy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="tiny")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--prompt", type=int, default=16)
ap.add_argument("--max-tokens", type=int, default=32)
ap.add_argument("--train-batch", type=int, default=32)
ap.add_argument("--rounds-per-poll", type=int, default=8)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--lr", type=float, default=3e-3)
ap.add_argument("--scale", type=float, default=0.05)
a = ap.parse_args()

cfg = PRESETS[a.config]
pol = DecoderPolicy.random(cfg, seed=0, scale=a.scale)
pl = PipelineRL(pol, batch=a.batch, prompt_len=a.prompt, max_tokens=a.max_tokens,
                train_batch=a.train_batch, queue_capacity=4 * a.train_batch,
                rounds_per_poll=a.rounds_per_poll, n_prompts=8, lr=a.lr, seed=0)
pl.run(optimizer_steps=1)  # warm-up: allocations, first launches, CUDA graphs
rep = pl.run(optimizer_steps=a.steps)
r = [s.reward_mean for s in rep.steps]
out = {
    "config": a.config, "batch": a.batch, "train_batch": a.train_batch, "max_tokens": a.max_tokens,
    "optimizer_steps": len(rep.steps), "rounds": rep.rounds, "generated_tokens": rep.generated_tokens,
    "wall_s": rep.wall_s, "generate_s": rep.generate_s, "train_s": rep.train_s,
    "tokens_per_s_wall": rep.generated_tokens / rep.wall_s,
    "tokens_per_s_generating": rep.generated_tokens / rep.generate_s,
    "trainer_ms_per_step": 1e3 * rep.train_s / max(1, len(rep.steps)),
    "reward_first_last": [float(np.mean(r[:3])), float(np.mean(r[-3:]))],
    "max_lag_steps": max(s.max_lag_steps for s in rep.steps),
    "mean_lag_steps": float(np.mean([s.mean_lag_steps for s in rep.steps])),
    "max_sample_lag": max(s.sample_max_lag for s in rep.steps),
    "pause_ms_max": max(s.pause_ms for s in rep.steps), "stalls": rep.stalls, "evicted": rep.evicted,
}
print(json.dumps(out))
pl.close()
