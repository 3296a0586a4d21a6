#!/usr/bin/env python
"""PipelineRL generator hot path on B200: generated tokens/s with in-flight
weight updates, weight-update pause, token lag.

Workload (BASELINE.json configs[1], the config the metric is quoted on; its
generator side fits one GPU): Qwen2.5-0.5B-shaped random-init bf16 policy,
constant generation batch 64 (Algorithm 2: finished streams are refilled with
new synthetic prompts at once), one in-flight weight update per optimizer
step.  One bench step = one optimizer-step period: R decode rounds of the
whole batch, then the update (the trainer's fresh weights land in the standby
buffer -- ncclBroadcast from rank 0 for N > 1, a device copy at N = 1 -- and
are swapped in at the next token boundary; streams continue on their stale
KV cache).

  value         tokens / device time (CUDA events on the engine stream + the
                update copy/broadcast + the swap pause), max over ranks
  e2e           the same through the public API (Engine.advance / wait_events
                / open_stream / begin/commit_weight_update), wall clock: every
                step includes the H2D prompts of refilled streams and the D2H
                token events, plus the host-side event collection
  roofline      the dominant kernel class of a decode round, timed with CUDA
                events around each launch of a profiled round
  cpu_baseline  the CPU oracle port of the same decoder (oracle/, numpy fp32,
                all host cores) on a bounded sample of the workload

Inputs: weights (0.99 GB) are larger than L2 (126 MB) and stream every round.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "generated tokens/sec with in-flight updates"
UNIT = "tokens/s"
KERNEL_CLASSES = ["plan", "embed", "qkv_gemm", "rope_kv_append", "attention", "o_gemm",
                  "gate_up_gemm", "down_gemm", "lm_head_gemm", "sample"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen2.5-0.5b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--gen", type=int, default=256, help="max_tokens per stream")
    ap.add_argument("--rounds", type=int, default=32, help="decode rounds per optimizer step")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=4)
    ap.add_argument("--no-trainer", action="store_true", help="skip the trainer-step measurement")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the one-GPU PipelineRL loop")
    ap.add_argument("--train-seqs", type=int, default=64, help="trajectories per trainer step")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- clocks ---
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(s[1]) for s in self.samples if len(s) > 8 and s[1].replace(".", "").isdigit()]
        smax = [float(s[2]) for s in self.samples if len(s) > 8 and s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples if len(s) > 8
                          for n, v in zip(names, s[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(sm)}


# ------------------------------------------------------------ roofline ---
def algorithmic_bytes(cfg, rows, ctx_sum):
    """Minimum HBM bytes per kernel class of one decode round over `rows`
    streams whose contexts sum to ctx_sum tokens (bf16 weights/KV, fp32
    logits).  SURVEY.md section 8(d)."""
    H, V, L, I = cfg.hidden, cfg.vocab_size, cfg.layers, cfg.intermediate
    nq, nkv, hd = cfg.q_heads, cfg.kv_heads, cfg.head_dim
    qkv = (nq + 2 * nkv) * hd
    b = {}
    b["embed"] = rows * H * (2 + 4 + 2)
    # QKV GEMM with the fused bias + RoPE + paged K/V append epilogue
    b["qkv_gemm"] = L * (qkv * H * 2 + rows * H * 2 + rows * qkv * 2)
    b["rope_kv_append"] = 0
    b["attention"] = L * (ctx_sum * 2 * nkv * hd * 2 + rows * nq * hd * 2 * 2)
    b["o_gemm"] = L * (H * nq * hd * 2 + rows * nq * hd * 2 + rows * H * (4 + 4 + 2))
    b["gate_up_gemm"] = L * (2 * I * H * 2 + rows * H * 2 + rows * I * 2)
    b["down_gemm"] = L * (H * I * 2 + rows * I * 2 + rows * H * (4 + 4 + 2))
    b["lm_head_gemm"] = V * H * 2 + rows * H * 2 + rows * V * 4
    # the sampler reads the LM-head epilogue's per-(row, 128-column tile)
    # (max, fp64 sum) statistics and walks one tile of the row
    b["sample"] = rows * (((V + 127) // 128) * 12 + 128 * 4)
    b["plan"] = rows * 16
    return b


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d.get("bf16_tflops"), "measured"
    return 6650.0, 1590.0, "fallback"


def load_traffic():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        return json.loads(p.read_text())
    return {}


# -------------------------------------------------------- CPU baseline ---
def cpu_decode_sample(cfg, batch, prompt, steps, warmup=0, seed=0):
    """The oracle port (oracle/decoder_oracle.py, numpy fp32, BLAS on all host
    cores) decoding `steps` rounds of `batch` streams after a short prefill.
    Returns (tokens/s, seconds, cores)."""
    from oracle.decoder_oracle import DecoderOracle, layout

    _, total = layout(cfg.to_dict())
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal(total, dtype=np.float32) * 0.02).view(np.uint32)
    w = (w >> 16).astype(np.uint16)
    off, _ = layout(cfg.to_dict())
    for name, (o, n) in off.items():  # unit norm gains like the device init
        if name.endswith("ln1") or name.endswith("ln2") or name == "final_norm":
            w[o:o + n] = 0x3F80
    m = DecoderOracle(cfg.to_dict(), w, np.float32)
    caches = [m.new_cache() for _ in range(batch)]
    prompts = rng.integers(0, cfg.vocab_size, size=(batch, prompt))
    toks = np.full(batch, cfg.bos_token)
    for p in range(prompt + 1):
        logits = m.step(caches, toks, np.full(batch, p))
        toks = prompts[:, p] if p < prompt else logits.argmax(-1)
    for _ in range(warmup):
        logits = m.step(caches, toks, np.full(batch, len(caches[0]["tokens"])))
        toks = logits.argmax(-1)
    t0 = time.perf_counter()
    for _ in range(steps):
        logits = m.step(caches, toks, np.full(batch, len(caches[0]["tokens"])))
        toks = logits.argmax(-1)
    dt = time.perf_counter() - t0
    return batch * steps / dt, dt, os.cpu_count()


def matmul_params(cfg):
    """Parameters that enter a GEMM per token (all projections + LM head)."""
    H, I, L, V = cfg.hidden, cfg.intermediate, cfg.layers, cfg.vocab_size
    qd, qkv = cfg.q_heads * cfg.head_dim, (cfg.q_heads + 2 * cfg.kv_heads) * cfg.head_dim
    return L * (qkv * H + H * qd + 2 * I * H + H * I) + V * H


def trainer_measure(cfg, pol, n_seq, prompt, gen, steps=3):
    """Trainer side of config 2: one optimizer step =
    current-policy log-prob recompute + truncated-IS REINFORCE objective + full
    backward + Adam over n_seq trajectories of prompt + gen tokens.  Device
    time from the trainer's own CUDA events (srl_trainer_stats.step_ms) plus
    the Adam kernel; tensor throughput counts 6 * matmul params per token plus
    causal attention (fwd 4 * T^2/2 * nq * hd per layer and sequence, x3)."""
    import torch

    from paper_2509_19128_b200.trainer import Trainer

    rng = np.random.default_rng(7)
    seq = prompt + 1 + gen
    trajs = []
    for i in range(n_seq):
        toks = [cfg.bos_token] + rng.integers(0, cfg.vocab_size, size=seq - 1).tolist()
        mu = (-np.log(cfg.vocab_size) + 0.1 * rng.standard_normal(seq)).tolist()
        a = float(rng.standard_normal())
        trajs.append(dict(tokens=toks, loss_begin=prompt + 1, behavior_logprobs=mu,
                          advantages=[a] * seq))
    tr = Trainer(pol.clone(), max_tokens=n_seq * seq)
    tr.step(trajs)  # warm-up (allocations, first launches)
    tr.apply_adam(1e-6)
    torch.cuda.synchronize()
    ms, fwd = [], []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r = tr.step(trajs)
        e0.record()
        tr.apply_adam(1e-6)
        e1.record()
        torch.cuda.synchronize()
        ms.append(r.step_ms + e0.elapsed_time(e1))
        fwd.append(r.forward_ms)
    tokens = r.tokens
    attn = cfg.layers * n_seq * 4 * (seq * seq / 2) * cfg.q_heads * cfg.head_dim * 3
    flops = 6.0 * matmul_params(cfg) * tokens + attn
    t = float(np.median(ms))
    _, bf16, kind = load_peaks()
    tf = flops / (t * 1e-3) / 1e12
    out = {"workload": f"{n_seq} trajectories x {seq} tokens ({tokens} scored rows), "
                       f"IS-REINFORCE fwd + bwd + Adam",
           "tokens_per_s": tokens / (t * 1e-3), "step_ms": t, "forward_ms": float(np.median(fwd)),
           "tflops": tf, "bound": "tensor", "peak_tflops": bf16, "peak_kind": kind,
           "frac": tf / bf16 if bf16 else None, "objective": r.objective, "ess": r.ess}
    tr.close()
    return out


def recompute_pause_measure(cfg, pol, payload_policy, args, rounds=128):
    """The same in-flight update with the engine in recompute mode
    (engine.cpp:107-113): at the swap every live stream's KV cache is rebuilt
    from its full prefix under the new weights (chunked prefill, tensor-core
    attention segments) -- the pause PipelineRL avoids by keeping the stale
    cache.  B streams of prompt + `rounds` generated tokens."""
    from paper_2509_19128_b200.engine import Engine

    eng = Engine(pol, recompute_state=True, start_paused=True, max_streams=args.batch,
                 max_seq_len=args.prompt + rounds + 8, rounds_per_sync=32,
                 prefill_budget=args.batch * (args.prompt + 1))
    rng = np.random.default_rng(5)
    for i in range(args.batch):
        eng.open_stream("p", rounds + 4, i, -1, rng.integers(0, cfg.vocab_size, size=args.prompt).tolist())
    eng.advance(rounds)
    ctx = sum(len(eng.stream_tokens(f"s{i}")) for i in range(args.batch))
    res = eng.apply_weight_update(1, payload_policy)
    assert res.applied
    pause = eng.stats()["last_pause_ms"]
    eng.close()
    return {"ms": pause, "rebuilt_tokens": ctx,
            "note": f"{args.batch} streams, recompute mode: full-prefix KV rebuild at the swap"}


HOSTPROF = os.environ.get("SRL_BENCH_HOSTPROF") == "1"
HOSTPROF_ACC = {"advance": 0.0, "publish": 0.0, "drain": 0.0, "refill": 0.0}


def pipeline_measure(cfg, args, steps=6):
    """The whole PipelineRL loop time-shared on ONE GPU (paper_2509_19128_b200/
    pipeline.py): constant-batch generator -> actor queue -> IS-REINFORCE
    trainer step on every train_batch finished sequences -> in-flight update.
    Config 2 puts generator and trainer on two GPUs; here they alternate, so
    tokens_per_s_wall is a lower bound for that configuration."""
    from paper_2509_19128_b200.pipeline import PipelineRL
    from paper_2509_19128_b200.policy import DecoderPolicy

    pol = DecoderPolicy.random(cfg, seed=1, scale=0.02)
    pl = PipelineRL(pol, batch=args.batch, prompt_len=args.prompt, max_tokens=args.gen,
                    train_batch=args.batch, queue_capacity=4 * args.batch, rounds_per_poll=args.rounds,
                    n_prompts=8, lr=1e-5, seed=0)
    pl.run(optimizer_steps=1)  # warm-up
    rep = pl.run(optimizer_steps=steps)
    pl.close()
    return {"workload": f"{cfg.name}, batch {args.batch}, train batch {args.batch} sequences of "
                        f"{args.prompt} + {args.gen} tokens, {steps} optimizer steps",
            "tokens_per_s_wall": rep.generated_tokens / rep.wall_s,
            "tokens_per_s_generating": rep.generated_tokens / rep.generate_s,
            "trainer_ms_per_step": 1e3 * rep.train_s / max(1, len(rep.steps)),
            "max_lag_steps": max(st.max_lag_steps for st in rep.steps),
            "mean_lag_steps": float(np.mean([st.mean_lag_steps for st in rep.steps])),
            "pause_ms_max": max(st.pause_ms for st in rep.steps),
            "stalls": rep.stalls, "evicted": rep.evicted}


def reference_arm(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    # each step = one decode round of the whole batch on the CPU port
    batch = args.batch
    prompt = min(args.prompt, 16)
    tps, dt, cores = cpu_decode_sample(cfg, batch, prompt, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic prompts, random-init weights",
        "config": {"workload": f"{cfg.name} decode, batch {batch}, CPU oracle port",
                   "global_batch": batch, "seq_len": prompt + 1 + args.steps,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": tps, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{batch} streams x {args.steps} decode rounds after a "
                                   f"{prompt}-token prefill (reference has no decoder; "
                                   f"oracle/decoder_oracle.py, numpy fp32)"},
        "e2e": {"value": tps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- ours ---
class _Raw:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def main():
    args = parse()
    from paper_2509_19128_b200.policy import PRESETS

    cfg = PRESETS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2509_19128_b200 import _lib
    from paper_2509_19128_b200.engine import Engine
    from paper_2509_19128_b200.policy import DecoderPolicy
    from paper_2509_19128_b200.weight_sync import EngineStandby, WeightChannel, max_over_ranks

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # policy v0 and two alternating "trainer" payloads (random init, then drift)
    pol = DecoderPolicy.random(cfg, seed=0, scale=0.02, device=local)
    payloads = [pol.clone().perturb(1000 + i, 0.002) for i in range(2)]
    B, R = args.batch, args.rounds
    max_seq = args.prompt + 1 + args.gen + 1
    eng = Engine(pol, start_paused=True, max_streams=B, max_seq_len=max_seq,
                 rounds_per_sync=R, event_ring=max(64, R), use_graphs=not args.no_graphs,
                 device=local, prefill_budget=B * (args.prompt + 1))
    rng = np.random.default_rng(1234 + rank)
    live = {}
    h2d_bytes = 0
    d2h_bytes = 0

    def open_one(i, max_tokens):
        nonlocal h2d_bytes
        pr = rng.integers(0, cfg.vocab_size, size=args.prompt).tolist()
        sid = eng.open_stream("synthetic", max_tokens, int(rng.integers(0, 2**63)), -1, pr)
        h2d_bytes += 4 * len(pr) + 24
        live[sid] = []
        return sid

    # staggered initial lengths so finishes (and refills) spread over steps
    for i in range(B):
        open_one(i, max(8, args.gen - (i * args.gen) // B))

    token_versions = []  # finished sequences (for lag stats)
    s = torch.cuda.Stream(device=dev)
    chan = WeightChannel(src=0)
    standby = EngineStandby(eng, dev)

    def step(record):
        nonlocal d2h_bytes
        st0 = eng.stats()
        t_wall = time.perf_counter()
        emitted = eng.advance(R)
        t_adv = time.perf_counter()
        # in-flight update: trainer rank 0's weights -> every standby buffer
        # (ncclBroadcast for N > 1, a device copy at N = 1) -> swap at the next
        # token boundary; the streams continue on their stale KV cache
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        src, n = payloads[(chan.version + 1) % 2].weights()
        payload = torch.as_tensor(_Raw(src, n), device=dev)
        with torch.cuda.stream(s):
            e0.record(s)
            applied, _, pause = chan.publish(rank, None, payload if rank == 0 else None,
                                                   engine=standby)
            e1.record(s)
        s.synchronize()
        t_pub = time.perf_counter()
        assert applied, "weight update rejected"
        # actor side: drain events, refill finished streams (constant batch)
        finished = []
        drained = eng.wait_events_many(list(live), columns=True)
        for sid, (evs, reason, more) in drained.items():
            d2h_bytes += 24 * len(evs)
            live[sid].extend(evs.weight_version.tolist())
            if not more or reason != "running":
                finished.append(sid)
        t_drain = time.perf_counter()
        for sid in finished:
            token_versions.append(live.pop(sid))
            open_one(0, args.gen)
        wall = time.perf_counter() - t_wall
        if HOSTPROF and record is not None:  # SRL_BENCH_HOSTPROF=1: host split of the e2e step
            hp = HOSTPROF_ACC
            hp["advance"] += t_adv - t_wall
            hp["publish"] += t_pub - t_adv
            hp["drain"] += t_drain - t_pub
            hp["refill"] += time.perf_counter() - t_drain
        st1 = eng.stats()
        upd_ms = e0.elapsed_time(e1)
        dev_ms = (st1["decode_ms"] - st0["decode_ms"]) + upd_ms + pause
        if record is not None:
            record.append(dict(tokens=emitted, dev_ms=dev_ms, wall_ms=1000 * wall, pause_ms=pause,
                               prefill_ms=st1["prefill_ms"] - st0["prefill_ms"],
                               prefill_rows=st1["prefill_rows"] - st0["prefill_rows"],
                               update_ms=upd_ms, launches=st1["launches"] - st0["launches"],
                               finished=len(finished)))

    for _ in range(args.warmup):
        step(None)
    # one profiled round (outside the timed region): per-kernel-class CUDA events
    eng.profile_next_round()
    eng.advance(2)  # a pending refill prefill may take the first round; the next decode round is profiled
    prof = eng.kernel_profile()
    fused_ms = []
    if "decode_megakernel" in prof:  # average the one-launch round over a few more rounds
        fused_ms.append(prof["decode_megakernel"][0])
        for _ in range(7):
            eng.profile_next_round()
            eng.advance(1)
            fused_ms.append(eng.kernel_profile()["decode_megakernel"][0])
    ctx_now = [len(eng.stream_tokens(sid)) for sid in live]
    # drain the profiled round's events so the actor stays consistent
    for sid in list(live):
        evs, reason, more = eng.wait_events(sid)
        live[sid].extend(e.weight_version for e in evs)

    clocks = ClockSampler(local)
    h2d0, d2h0 = h2d_bytes, d2h_bytes
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    rec = []
    for _ in range(args.steps):
        step(rec)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    tokens = sum(r["tokens"] for r in rec)
    dev_ms = sum(r["dev_ms"] for r in rec)
    wall_ms = sum(r["wall_ms"] for r in rec)
    launches = sum(r["launches"] for r in rec)
    pauses = [r["pause_ms"] for r in rec]
    upd = [r["update_ms"] for r in rec]
    dev_ms_max = max_over_ranks(dev_ms)
    wall_ms_max = max_over_ranks(wall_ms)
    total_tokens = float(tokens)
    if world > 1:
        t = torch.tensor([float(tokens)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_tokens = t.item()

    # lag bookkeeping of the sequences consumed so far (device lag kernel)
    lag = {"max_lag_steps": None}
    seqs = token_versions + [v for v in live.values() if v]
    if seqs:
        vers = torch.tensor(np.concatenate([np.asarray(v, dtype=np.int32) for v in seqs]), device=dev)
        offs = torch.tensor(np.concatenate([[0], np.cumsum([len(v) for v in seqs])]),
                            dtype=torch.int64, device=dev)
        hist = torch.zeros(4096, dtype=torch.int64, device=dev)
        sums = torch.zeros(len(seqs), dtype=torch.int64, device=dev)
        tot = torch.zeros(4, dtype=torch.int64, device=dev)
        _lib.call("srl_lag_stats", vers.data_ptr(), offs.data_ptr(), len(seqs), chan.version,
                  hist.data_ptr(), 4096, sums.data_ptr(), tot.data_ptr(), None)
        torch.cuda.synchronize()
        tt = tot.cpu().tolist()
        lag = {"max_lag_steps": int(tt[2]), "mean_lag_steps": tt[1] / max(tt[0], 1),
               "sequences": len(seqs), "finished_sequences": len(token_versions)}

    # roofline of the dominant kernel (profiled rounds)
    hbm, bf16, peak_kind = load_peaks()
    abytes = algorithmic_bytes(cfg, B, sum(ctx_now))
    step_bytes = sum(abytes.values())
    cls_ms = {k: prof[k][0] for k in KERNEL_CLASSES}
    traffic_db = load_traffic().get(args.config, {})
    if fused_ms:
        # the whole round is ONE persistent kernel: its algorithmic bytes are
        # the round's, its duration the CUDA-event time of the launch
        mk_ms = float(np.mean(fused_ms))
        roof = {"kernel": "decode_megakernel", "bound": "hbm",
                "achieved": step_bytes / (mk_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_kind": peak_kind, "traffic": traffic_db.get("decode_megakernel"),
                "launches_per_round": 1, "bytes_per_launch": step_bytes, "ms_per_launch": mk_ms,
                "ms_per_launch_samples": len(fused_ms),
                "phase_ms_per_round": {k: round(v, 4) for k, v in cls_ms.items()}}
        round_ms = mk_ms
    else:
        dom = max(cls_ms, key=cls_ms.get)
        round_ms = sum(cls_ms.values())
        nlaunch = max(prof[dom][1], 1)
        roof = {"kernel": dom, "bound": "hbm", "achieved": abytes[dom] / (cls_ms[dom] * 1e-3) / 1e9,
                "peak": hbm, "unit": "GB/s", "peak_kind": peak_kind,
                "traffic": traffic_db.get(dom), "launches_per_round": prof[dom][1],
                "bytes_per_launch": abytes[dom] / nlaunch, "ms_per_launch": cls_ms[dom] / nlaunch}
    roof["frac"] = roof["achieved"] / roof["peak"]
    round_roof = {"bound": "hbm", "achieved": step_bytes / (round_ms * 1e-3) / 1e9, "peak": hbm,
                  "unit": "GB/s", "bytes": step_bytes, "ms": round_ms,
                  "bytes_by_class": {k: int(v) for k, v in abytes.items()}}
    round_roof["frac"] = round_roof["achieved"] / hbm
    roofline_tps = B / (step_bytes / (hbm * 1e9))

    value = total_tokens / (dev_ms_max * 1e-3)
    e2e = total_tokens / (wall_ms_max * 1e-3)
    if HOSTPROF:
        print("host ms/step", {k: round(1e3 * v / args.steps, 3) for k, v in HOSTPROF_ACC.items()},
              "device ms/step", round(dev_ms / args.steps, 3), file=sys.stderr)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts, random-init weights",
        "config": {"workload": f"{cfg.name} generator, constant batch {B}, in-flight update "
                               f"every {R} decode rounds (one optimizer step)",
                   "model": cfg.name, "global_batch": B * world, "seq_len": max_seq,
                   "prompt": args.prompt, "max_tokens": args.gen, "rounds_per_step": R,
                   "parallelism": f"generator replicas x{world} (update broadcast from rank 0)"
                                  if world > 1 else "1 generator (update = device copy)",
                   "cuda_graphs": not args.no_graphs,
                   "l2": "inputs larger than L2 (0.99 GB weights streamed every round)"},
        "e2e": {"value": e2e, "unit": UNIT,
                "h2d_bytes_per_step": (h2d_bytes - h2d0) // args.steps,
                "d2h_bytes_per_step": (d2h_bytes - d2h0) // args.steps},
        "gpu_launches": launches,
        "pause_ms": {"median": float(np.median(pauses)), "max": float(np.max(pauses))},
        "update_copy_ms": {"median": float(np.median(upd)), "max": float(np.max(upd)),
                           "payload_bytes": pol.weights()[1]},
        "lag": lag,
        "roofline": roof,
        "round_roofline": round_roof,
        "roofline_tokens_per_s": roofline_tps,
        "kernel_ms_per_round": {k: round(v, 4) for k, v in cls_ms.items()},
        "update_gbs": pol.weights()[1] / (float(np.median(upd)) * 1e-3) / 1e9,
        "prefill": {"ms_per_step": sum(r["prefill_ms"] for r in rec) / args.steps,
                    "rows_per_step": sum(r["prefill_rows"] for r in rec) / args.steps,
                    "note": "refill prefill rounds of finished streams (inside value's device time)"},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_trainer:
        tclk = ClockSampler(local)
        tclk.start()
        out["trainer"] = trainer_measure(cfg, pol, args.train_seqs, args.prompt, args.gen)
        out["trainer"]["clocks"] = tclk.stop()
    if rank == 0 and world == 1 and not args.no_pipeline:
        out["pause_ms_recompute_mode"] = recompute_pause_measure(cfg, pol, payloads[0], args)
        out["pipeline_1gpu"] = pipeline_measure(cfg, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tps, dt, cores = cpu_decode_sample(cfg, B, 8, args.cpu_steps, 1)
        out["cpu_baseline"] = {"value": tps, "unit": UNIT, "cores": cores, "kind": "port",
                               "sample": f"{B} streams x {args.cpu_steps} decode rounds after an "
                                         f"8-token prefill, oracle/decoder_oracle.py numpy fp32 "
                                         f"({dt:.1f} s)"}
    eng.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
