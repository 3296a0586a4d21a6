#!/usr/bin/env python
"""Probe + timeline analysis of the persistent decode megakernel.

Runs the bench workload (Qwen2.5-0.5B shape, batch 64) for a few rounds,
profiles one decode round with SRL_MK_TRACE (per-CTA, per-phase globaltimer
stamps written by decode_megakernel) and prints, per phase kind, where the
time goes: barrier propagation (last arrival of the previous phase -> median
CTA start), the activation dependency seen by the TMA producer, the first
accumulator, split-K exchange, epilogue, and the phase period.

  python tools/mk_trace.py [--config qwen2.5-0.5b] [--batch 64] [--rounds 40]
"""
import argparse
import os
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
KINDS = ["embed", "qkv", "attn", "o", "gu", "down", "lm", "sample"]


def load(path):
    b = Path(path).read_bytes()
    n, grid = struct.unpack_from("ii", b, 0)
    meta = np.frombuffer(b, dtype=np.int32, count=4 * n, offset=8).reshape(n, 4)
    tr = np.frombuffer(b, dtype=np.uint64, offset=8 + 16 * n).reshape(n, grid, 16).astype(np.int64)
    return meta, tr


GHZ = 1.965  # SM clock under load (bench clocks: 1965 MHz)
# per-CTA stamps inside a phase, SM cycles since the phase start (tr[8]);
# attention items use 10-14 as cycles since the item start
GEMM_FIELDS = [(4, "dep"), (14, "full0"), (15, "committed"), (1, "acc"), (11, "stored"), (12, "arrived"), (2, "xchg"), (5, "red"),
               (13, "xready"), (6, "epi"), (9, "end")]
ATTN_FIELDS = [(4, "bulk"), (6, "loads"), (1, "issued"), (2, "partials"), (5, "reduced"), (11, "operands"), (12, "keys"), (13, "sync"), (14, "merged"), (10, "item")]


def analyse(meta, tr):
    n, grid, _ = tr.shape
    t0 = tr[:, :, 0]
    base = t0[0].min()
    rows = []
    prev_last = None
    for p in range(n):
        kind = KINDS[meta[p, 0]]
        active = tr[p, :, 7] > 0
        st = t0[p][active] - base
        arr = tr[p, :, 7][active] - base
        last = arr.max()
        r = dict(p=p, kind=kind, cs=int(meta[p, 1]), items=int(meta[p, 2]),
                 start_med=np.median(st), last=last)
        r["bar"] = (np.median(st) - prev_last) if prev_last is not None else 0.0
        r["period"] = last - prev_last if prev_last is not None else last
        r["arrive"] = float(np.median(tr[p, :, 7][active] - tr[p, :, 3][active]))
        r["spans"] = (tr[p, :, 7][active] - t0[p][active]).astype(np.float64)
        r["items_per_cta"] = tr[p, :, 15][active] if kind == "attn" else np.zeros(0)
        fields = ATTN_FIELDS if kind == "attn" else GEMM_FIELDS
        for k, name in fields:
            v = tr[p, :, k].copy()
            if k in (4, 14, 15) and kind != "attn":  # raw clock64 of the producer / MMA warps
                v = np.where(v > 0, v - tr[p, :, 8], 0)
            ok = (v > 0) & active
            r[name] = float(np.median(v[ok])) / GHZ if ok.any() else float("nan")
            r[name + "_max"] = float(v[ok].max()) / GHZ if ok.any() else float("nan")
        rows.append(r)
        prev_last = last
    return rows


def report(rows):
    total = rows[-1]["last"]
    print(f"round {total / 1e3:.1f} us over {len(rows)} phases (ns medians over layers; "
          f"inner stamps = median over CTAs, ns since the CTA's phase start)")
    by = {}
    for r in rows:
        by.setdefault(r["kind"], []).append(r)
    for k in KINDS:
        if k not in by:
            continue
        rs = by[k]
        med = lambda key: np.nanmedian([x.get(key, np.nan) for x in rs])
        fields = ATTN_FIELDS if k == "attn" else GEMM_FIELDS
        inner = " ".join(f"{name}={med(name):.0f}/{med(name + '_max'):.0f}" for _, name in fields
                         if not np.isnan(med(name)))
        if k == "attn":  # per-CTA busy time in the phase: the work balance across SMs
            spans = np.concatenate([x["spans"] for x in rs]) / 1e3
            print(f"attn   per-CTA phase span (us): min {spans.min():.1f} median {np.median(spans):.1f} "
                  f"p90 {np.percentile(spans, 90):.1f} max {spans.max():.1f}")
            items = np.concatenate([x["items_per_cta"] for x in rs])
            print(f"attn   items per CTA: mean {items.mean():.2f} max {items.max()} "
                  f"(stamps below: item #{os.environ.get('SRL_MK_TRACE_ITEM', '0')} of each CTA)")
        print(f"{k:6s} n={len(rs):2d} cs={rs[0]['cs']:2d} items={rs[0]['items']:4d} "
              f"period={med('period'):6.0f} barrier={med('bar'):5.0f} arrive={med('arrive'):4.0f} | {inner}"
              f"  [sum period {sum(x['period'] for x in rs) / 1e3:.1f} us]")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen2.5-0.5b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=40)
    ap.add_argument("--steady-gen", type=int, default=0,
                    help="bench-like steady state: stream i already (i + 0.5)/B through a rollout of this length")
    ap.add_argument("--trace", default="gpurun_out/mk_trace.bin")
    ap.add_argument("--file", help="analyse an existing trace instead of running")
    a = ap.parse_args()
    if a.file:
        report(analyse(*load(a.file)))
        return
    os.environ["SRL_MK_TRACE"] = str(Path(a.trace).resolve())
    Path(a.trace).parent.mkdir(parents=True, exist_ok=True)
    from paper_2509_19128_b200.engine import Engine
    from paper_2509_19128_b200.policy import PRESETS, DecoderPolicy

    cfg = PRESETS[a.config]
    pol = DecoderPolicy.random(cfg, seed=0, scale=0.02)
    extra = [int((i + 0.5) * a.steady_gen / a.batch) for i in range(a.batch)] if a.steady_gen else [0] * a.batch
    max_seq = a.prompt + max(extra) + a.rounds + 8
    eng = Engine(pol, start_paused=True, max_streams=a.batch, max_seq_len=max_seq,
                 rounds_per_sync=8, event_ring=64, prefill_budget=max(a.batch * (a.prompt + 1), max_seq))
    rng = np.random.default_rng(0)
    for i in range(a.batch):
        eng.open_stream("p", a.rounds + 4, i, -1, rng.integers(0, cfg.vocab_size, a.prompt + extra[i]).tolist())
    eng.advance(a.rounds)
    eng.profile_next_round()
    eng.advance(1)
    prof = eng.kernel_profile()
    print({k: round(v[0], 4) for k, v in prof.items()})
    eng.close()
    report(analyse(*load(a.trace)))


if __name__ == "__main__":
    main()
