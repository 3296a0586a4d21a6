#!/usr/bin/env python
"""Generator / trainer split of one 8 x B200 box from measured curves
(SURVEY 8f rank 3): the reference's search_configs (throughput.cpp:288-330,
restated in paper_2509_19128_b200/partition.py and checked against the
reference in tests/test_partition_cpu.py) over the B200 U(h) curve measured
by tools/utilization_curve.py and the trainer throughput measured by
bench.py, for a set of lag caps.

  python tools/partition_plan.py --curve profiles/r2_utilization_qwen2.5-1.5b.json \
      --trainer-tok-s 41000 --out profiles/r2_partition_plan_qwen2.5-1.5b.json
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_19128_b200.partition import (LengthDistribution, curve_from_measurement,  # noqa: E402
                                             search_configs)

ap = argparse.ArgumentParser()
ap.add_argument("--curve", required=True, help="utilization_curve.py JSON (rows of h, tokens_per_s)")
ap.add_argument("--trainer-tok-s", type=float, required=True, help="trained tokens/s of ONE trainer GPU")
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--train-batch", type=int, default=256, help="sequences per optimizer step")
ap.add_argument("--max-len", type=int, default=8192)
ap.add_argument("--lengths", default="uniform", choices=["uniform", "constant"])
ap.add_argument("--caps", default="1,2,4,8,16,32")
ap.add_argument("--out", default=None)
a = ap.parse_args()

doc = json.loads(Path(a.curve).read_text())
fpt, peak = doc["flops_per_token"], doc["peak_bf16_tflops"] * 1e12
curve = curve_from_measurement([(r["h"], r["tokens_per_s"]) for r in doc["rows"]], fpt, peak)
flash = fpt / peak
tau = (1.0 / a.trainer_tok_s) / flash  # flashes per trained token on one trainer GPU
lengths = LengthDistribution(a.lengths, a.max_len)
plans = []
for cap in [int(c) for c in a.caps.split(",")]:
    r = search_configs(a.n, a.train_batch, curve, tau, lengths, cap, use_padding=False)
    plan = {"lag_cap_steps": cap, "feasible": r.feasible}
    if r.feasible:
        plan.update(generators=r.inference_count, trainers=a.n - r.inference_count, gen_batch=r.gen_batch,
                    max_lag_steps=r.max_lag, tokens_per_s=r.r_total / flash,
                    gen_tokens_per_s=r.r_gen / flash, train_tokens_per_s=r.r_train / flash,
                    bound="generation" if r.r_gen < r.r_train else "training")
    plans.append(plan)
    print(json.dumps(plan), flush=True)
out = {"config": doc.get("config"), "n_gpus": a.n, "train_batch": a.train_batch,
       "lengths": f"{a.lengths}({a.max_len})", "flash_s": flash, "tau_flashes_per_trained_token": tau,
       "trainer_tokens_per_s_per_gpu": a.trainer_tok_s,
       "curve": [(h, u) for h, u in curve.samples], "plans": plans,
       "model": "throughput.cpp:288-330 search_configs (paper_2509_19128_b200/partition.py)"}
if a.out:
    Path(a.out).write_text(json.dumps(out, indent=1))
