#!/usr/bin/env python
"""Measured B200 utilization curve U(h) of the decode engine, in the format of
the reference's analytical model (/root/reference/proj/assets/curves/
default_utilization.csv: "h,utilization"; throughput.hpp UtilizationCurve):
U(h) = (generated tokens/s at constant generation batch h) x flops per token
/ peak bf16 flops.  The reference's `streamrl search` / speedup-vs-lag tools
take this file in place of their default curve.

  python tools/utilization_curve.py --config qwen2.5-0.5b --out profiles/r1_utilization_qwen2.5-0.5b.csv
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200.engine import Engine  # noqa: E402
from paper_2509_19128_b200.policy import PRESETS, DecoderPolicy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen2.5-0.5b")
ap.add_argument("--batches", default="1,2,4,8,16,32,48,64,96,128,192,256")
ap.add_argument("--prompt", type=int, default=128)
ap.add_argument("--rounds", type=int, default=64)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = PRESETS[a.config]
H, I, L, V = cfg.hidden, cfg.intermediate, cfg.layers, cfg.vocab_size
qd, qkv = cfg.q_heads * cfg.head_dim, (cfg.q_heads + 2 * cfg.kv_heads) * cfg.head_dim
matmul = L * (qkv * H + H * qd + 2 * I * H + H * I) + V * H
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
peak = peaks.get("bf16_tflops", 1590.0) * 1e12
pol = DecoderPolicy.random(cfg, seed=0, scale=0.02)
rows = []
for h in [int(x) for x in a.batches.split(",")]:
    eng = Engine(pol, start_paused=True, max_streams=h, max_seq_len=a.prompt + 3 * a.rounds + 8,
                 rounds_per_sync=a.rounds, event_ring=a.rounds, prefill_budget=h * (a.prompt + 1))
    rng = np.random.default_rng(h)
    for i in range(h):
        eng.open_stream("p", 3 * a.rounds, i, -1, rng.integers(0, V, size=a.prompt).tolist())
    eng.advance(a.rounds)  # prefill + warm-up (graphs / megakernel state)
    s0 = eng.stats()
    eng.advance(a.rounds)
    s1 = eng.stats()
    ms = (s1["decode_ms"] - s0["decode_ms"]) / a.rounds
    ctx = a.prompt + 1 + 1.5 * a.rounds
    attn = 4 * ctx * qd * L  # QK^T + PV per generated token
    tps = h / (ms * 1e-3)
    util = tps * (2 * matmul + attn) / peak
    rows.append((h, util, tps, ms))
    print(f"h={h:4d} round {ms:7.3f} ms  {tps:9.0f} tok/s  U={util:.5f}", flush=True)
    eng.close()
if a.out:
    with open(a.out, "w") as f:
        f.write("h,utilization\n")
        for h, u, _, _ in rows:
            f.write(f"{h},{u:.6f}\n")
    Path(a.out).with_suffix(".json").write_text(json.dumps(
        {"config": a.config, "peak_bf16_tflops": peak / 1e12, "flops_per_token": 2 * matmul,
         "rows": [{"h": h, "utilization": u, "tokens_per_s": t, "round_ms": m} for h, u, t, m in rows]}, indent=1))
