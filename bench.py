#!/usr/bin/env python
"""PipelineRL generator hot path on B200: generated tokens/s with in-flight
weight updates, weight-update pause, token lag.

Workload (N = 1): BASELINE.json's largest single-GPU configuration -- the
1-GPU point of configs[4]'s scaling sweep on the Qwen2.5-1.5B shape, with
configs[2]'s 8k-token synthetic reasoning rollouts: random-init bf16 weights,
constant generation batch 64 (Algorithm 2: a finished stream is replaced by a
new synthetic prompt at once), rollouts of up to 8192 generated tokens.  The
batch starts in the steady state of such a generator: stream i is a rollout
already (i + 0.5)/64 of the way through (its prefix is prefilled before the
timed region), so contexts are spread uniformly over 64..8256 tokens.  One
bench step = one optimizer-step period: R decode rounds of the whole batch
while the trainer's fresh weights stream into the standby buffer on a side
stream, then the swap at the next token boundary (the streams continue on
their stale KV cache).

  value         tokens / device time (CUDA events on the engine stream, plus
                the swap pause and any transfer time not hidden under decode)
  e2e           the same through the public API (Engine.advance /
                begin/commit_weight_update / wait_events_many / open_stream),
                host wall clock: every step includes the H2D prompts of
                refilled streams and the D2H token events
  pause         swap_ms = the decode loop blocked by the pointer swap;
                decode_stall_ms = (step time with the update in flight) -
                (step time without an update): what the update costs decode
  lag           per consumed sequence (sim.cpp:63-104): version at consumption
                minus the version that emitted each token
  roofline      the decode megakernel (one launch per round), CUDA events
  cpu_baseline  the CPU port of the same decode round (oracle/decoder_cpu.py,
                numpy fp32 on all host cores) on the same streams and contexts

N > 1 (torchrun, or --gpus N which relaunches itself under torchrun): the
partitioned PipelineRL of paper_2509_19128_b200/pipeline_dist.py -- trainer
ranks (data-parallel, gradient all-reduce) and generator ranks (weight
broadcast into their standby buffers), 1+1 / 2+2 / 4+4 / 6+2 (--trainers).

Inputs: weights (3.09 GB) and KV caches (~7.6 GB) are larger than L2
(126 MB) and stream every round.
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


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen2.5-1.5b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--gen", type=int, default=8192, help="max generated tokens per rollout")
    ap.add_argument("--rounds", type=int, default=32, help="decode rounds per optimizer step")
    ap.add_argument("--no-steady", action="store_true",
                    help="start every stream at its prompt instead of the steady-state spread")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-trainer", action="store_true", help="skip the trainer-step measurement")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the one-GPU PipelineRL loop")
    ap.add_argument("--no-extra", action="store_true", help="skip the 0.5B / 7B generator lines")
    ap.add_argument("--extra", default="qwen2.5-0.5b:64:256,qwen2.5-7b:256:1024,qwen2.5-1.5b:64:8192:precise",
                    help="extra generator configs name:batch:gen[:precise] (N = 1)")
    ap.add_argument("--train-seqs", type=int, default=64, help="trajectories per trainer step")
    ap.add_argument("--train-gen", type=int, default=256, help="generated tokens per trainer trajectory")
    ap.add_argument("--trainers", type=int, default=None, help="trainer ranks of the partition (N > 1)")
    return ap.parse_args(argv)


_T0 = time.perf_counter()


def log(msg):
    """Phase progress on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: one process per GPU."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


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
        return self

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


def matmul_params(cfg):
    """Parameters that enter a GEMM per token (all projections + LM head)."""
    H, I, L, V = cfg.hidden, cfg.intermediate, cfg.layers, cfg.vocab_size
    qd, qkv = cfg.q_heads * cfg.head_dim, (cfg.q_heads + 2 * cfg.kv_heads) * cfg.head_dim
    return L * (qkv * H + H * qd + 2 * I * H + H * I) + V * H


def pipeline_max_lag_steps(gen_batch, inference_count, max_len, mean_len, train_batch):
    """g_max = ceil(H * I * L / (mean L * B)) (throughput.cpp:260-269)."""
    import math

    return int(math.ceil(gen_batch * inference_count * max_len / (mean_len * train_batch)))


def steady_contexts(B, prompt, gen):
    """Stream i of a steady-state constant-batch generator is (i + 0.5)/B of
    the way through its rollout: (prefix tokens after the prompt, tokens left)."""
    out = []
    for i in range(B):
        done = int((i + 0.5) * gen / B)
        out.append((done, gen - done))
    return out


# ---------------------------------------------------------- trainer side ---
def trainer_measure(cfg, pol, n_seq, prompt, gen, steps=3, precise=True):
    """Trainer side: one optimizer step = current-policy
    log-prob recompute + truncated-IS REINFORCE objective + full backward +
    Adam over n_seq trajectories of prompt + gen tokens.  Device time from the
    trainer's own CUDA events (srl_trainer_stats.step_ms) plus the Adam
    kernel; tensor throughput counts 6 * matmul params per token plus causal
    attention (fwd 4 * T^2/2 * nq * hd per layer and sequence, x3)."""
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
    tr = Trainer(pol.clone(), max_tokens=n_seq * seq, precise=precise)
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
    mode = ("precise: activations and backward operands as bf16 hi + lo pairs (1e-3 parity mode)"
            if precise else "fast: single bf16 operands")
    out = {"workload": f"{cfg.name}: {n_seq} trajectories x {seq} tokens ({tokens} scored rows), "
                       f"IS-REINFORCE fwd + bwd + Adam", "mode": mode,
           "flops_counted": "model flops (6 x matmul params per token + causal attention); the "
                            "precise mode's extra split-operand MMAs are not counted",
           "tokens_per_s": tokens / (t * 1e-3), "step_ms": t, "forward_ms": float(np.median(fwd)),
           "tflops": tf, "bound": "tensor", "peak_tflops": bf16, "peak_kind": kind,
           "frac": tf / bf16 if bf16 else None, "objective": r.objective, "ess": r.ess}
    tr.close()
    return out


def recompute_pause_measure(cfg, pol, payload_policy, B, prompt, rounds=128):
    """The same in-flight update with the engine in recompute mode
    (engine.cpp:107-113): at the swap every live stream's KV cache is rebuilt
    from its full prefix under the new weights (chunked prefill, tensor-core
    attention segments) -- the pause PipelineRL avoids by keeping the stale
    cache.  B streams of prompt + `rounds` generated tokens."""
    from paper_2509_19128_b200.engine import Engine

    eng = Engine(pol, recompute_state=True, start_paused=True, max_streams=B,
                 max_seq_len=prompt + rounds + 8, rounds_per_sync=32,
                 prefill_budget=B * (prompt + 1))
    rng = np.random.default_rng(5)
    for i in range(B):
        eng.open_stream("p", rounds + 4, i, -1, rng.integers(0, cfg.vocab_size, size=prompt).tolist())
    eng.advance(rounds)
    ctx = sum(len(eng.stream_tokens(f"s{i}")) for i in range(B))
    res = eng.apply_weight_update(1, payload_policy)
    assert res.applied
    pause = eng.stats()["last_pause_ms"]
    eng.close()
    return {"ms": pause, "rebuilt_tokens": ctx,
            "note": f"{B} streams, recompute mode: full-prefix KV rebuild at the swap"}


def pipeline_measure(cfg, B, prompt, gen, rounds, steps=6):
    """The whole PipelineRL loop time-shared on ONE GPU (paper_2509_19128_b200/
    pipeline.py): constant-batch generator -> actor queue -> IS-REINFORCE
    trainer step on every train_batch finished sequences -> in-flight update.
    Per consumed batch: the lag statistics of make_step_record (sim.cpp:63-104)
    and the analytic bound g_max (throughput.cpp:260-269) for this loop."""
    from paper_2509_19128_b200.pipeline import PipelineRL
    from paper_2509_19128_b200.policy import DecoderPolicy

    pol = DecoderPolicy.random(cfg, seed=1, scale=0.02)
    pl = PipelineRL(pol, batch=B, prompt_len=prompt, max_tokens=gen, train_batch=B,
                    queue_capacity=4 * B, rounds_per_poll=rounds, n_prompts=8, lr=1e-5, seed=0)
    pl.run(optimizer_steps=1)  # warm-up
    rep = pl.run(optimizer_steps=steps)
    pl.close()
    mean_len = float(np.mean([st.mean_length for st in rep.steps]))
    return {"workload": f"{cfg.name}, batch {B}, train batch {B} sequences of "
                        f"{prompt} + {gen} tokens, {steps} optimizer steps",
            "tokens_per_s_wall": rep.generated_tokens / rep.wall_s,
            "tokens_per_s_generating": rep.generated_tokens / rep.generate_s,
            "trainer_ms_per_step": 1e3 * rep.train_s / max(1, len(rep.steps)),
            "max_lag_steps": max(st.max_lag_steps for st in rep.steps),
            "mean_lag_steps": float(np.mean([st.mean_lag_steps for st in rep.steps])),
            "sample_max_lag": max(st.sample_max_lag for st in rep.steps),
            "g_max_analytic": pipeline_max_lag_steps(B, 1, gen, mean_len, B),
            "pause_ms_max": max(st.pause_ms for st in rep.steps),
            "stalls": rep.stalls, "evicted": rep.evicted}


# ------------------------------------------------------- generator side ---
class _Raw:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def generator_measure(cfg, *, B, prompt, gen, R, steps, warmup, steady=True, use_graphs=True,
                      device=0, n_payloads=2, profile=True, lag=True, precise=False):
    """One generator GPU: constant batch B, an in-flight update every R rounds
    whose transfer into the standby buffer overlaps the decode rounds (a side
    stream), swap at the token boundary after them.  Returns the measurement
    dict (value / e2e / pause / stall / lag / roofline) and the policy."""
    import torch

    from paper_2509_19128_b200 import _lib
    from paper_2509_19128_b200.engine import Engine
    from paper_2509_19128_b200.policy import DecoderPolicy

    dev = torch.device("cuda", device)
    pol = DecoderPolicy.random(cfg, seed=0, scale=0.02, device=device)
    payloads = [pol.clone().perturb(1000 + i, 0.002) for i in range(n_payloads)]
    max_seq = prompt + 1 + gen + 1
    eng = Engine(pol, start_paused=True, max_streams=B, max_seq_len=max_seq,
                 rounds_per_sync=R, event_ring=max(64, R), use_graphs=use_graphs, device=device,
                 prefill_budget=max(B * (prompt + 1), max_seq), precise=precise)
    rng = np.random.default_rng(1234 + device)
    live = {}
    h2d = [0]
    d2h = [0]

    def open_one(done=0, left=gen):
        pr = rng.integers(0, cfg.vocab_size, size=prompt + done).tolist()
        sid = eng.open_stream("synthetic", left, int(rng.integers(0, 2**63)), -1, pr)
        h2d[0] += 4 * len(pr) + 24
        live[sid] = []
        return sid

    log(f"generator {cfg.name} B={B}: opening streams")
    if steady:
        for done, left in steady_contexts(B, prompt, gen):
            open_one(done, left)
    else:  # staggered lengths so finishes (and refills) spread over steps
        for i in range(B):
            open_one(0, max(8, gen - (i * gen) // B))
    # seat every stream (prefill of the steady-state prefixes) before timing:
    # a stream has been prefilled once it emitted its first token
    waiting = set(live)
    while waiting:
        eng.advance(4)
        for sid, (evs, reason, more) in eng.wait_events_many(list(live), columns=True, block=False).items():
            live[sid].extend(evs.weight_version.tolist())
            if len(evs) or reason != "running":
                waiting.discard(sid)
    log("generator: streams seated (prefill done)")
    side = torch.cuda.Stream(device=dev)
    consumed = []       # (version at consumption, token versions) per finished sequence
    version = [0]

    def step(record, update=True):
        st0 = eng.stats()
        t_wall = time.perf_counter()
        copy_ms = 0.0
        if update:
            # the trainer's weights stream into the standby buffer on a side
            # stream while the decode rounds run; the swap waits for the copy
            nxt = version[0] + 1
            ptr, n = eng.begin_weight_update(nxt)
            src, _ = payloads[nxt % len(payloads)].weights()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(side):
                e0.record(side)
                # D2D cudaMemcpyAsync on the side stream: it advances in the gaps between the
                # megakernel's rounds (which hold every SM); decode_stall_ms is its cost
                _lib.call("srl_device_copy_async", ptr, src, n, side.cuda_stream)
                e1.record(side)
        emitted = eng.advance(R)
        pause = 0.0
        if update:
            side.synchronize()
            res, pause = eng.commit_weight_update(nxt)
            assert res.applied, "weight update rejected"
            version[0] = nxt
            copy_ms = e0.elapsed_time(e1)
        # actor side: drain events, refill finished streams (constant batch)
        finished = []
        drained = eng.wait_events_many(list(live), columns=True, block=False)
        for sid, (evs, reason, more) in drained.items():
            d2h[0] += 24 * len(evs)
            live[sid].extend(evs.weight_version.tolist())
            if not more or reason != "running":
                finished.append(sid)
        for sid in finished:
            consumed.append((version[0], live.pop(sid)))
            open_one()
        wall = time.perf_counter() - t_wall
        st1 = eng.stats()
        dec = st1["decode_ms"] - st0["decode_ms"]
        dev_ms = dec + pause + max(0.0, copy_ms - dec)
        if record is not None:
            record.append(dict(tokens=emitted, dev_ms=dev_ms, decode_ms=dec, wall_ms=1000 * wall,
                               pause_ms=pause, copy_ms=copy_ms,
                               prefill_ms=st1["prefill_ms"] - st0["prefill_ms"],
                               prefill_rows=st1["prefill_rows"] - st0["prefill_rows"],
                               launches=st1["launches"] - st0["launches"], finished=len(finished)))

    for _ in range(warmup):
        step(None)
    log("generator: warm-up done")
    prof, fused_ms = {}, []
    if profile:  # profiled rounds (outside the timed region): per-class CUDA events
        eng.profile_next_round()
        eng.advance(2)  # a pending refill prefill may take the first round
        prof = eng.kernel_profile()
        if "decode_megakernel" in prof:  # the one-launch round, averaged over 8 rounds
            fused_ms.append(prof["decode_megakernel"][0])
            for _ in range(7):
                eng.profile_next_round()
                eng.advance(1)
                fused_ms.append(eng.kernel_profile()["decode_megakernel"][0])
    ctx_now = [len(eng.stream_tokens(sid)) for sid in live]
    for sid, (evs, reason, more) in eng.wait_events_many(list(live), columns=True, block=False).items():
        live[sid].extend(evs.weight_version.tolist())

    clocks = ClockSampler(device).start()
    h2d0, d2h0 = h2d[0], d2h[0]
    torch.cuda.synchronize()
    rec = []
    # NVTX range around the timed steps: `ncu --nvtx --nvtx-push-pop-scope process
    # --nvtx-include "timed/"` lists exactly the launches of the timed region (the
    # engine launches from its own thread, hence process scope; not the setup prefill)
    torch.cuda.nvtx.range_push("timed")
    for _ in range(steps):
        step(rec)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    log("generator: timed steps done")
    # the same steps without an update in flight: the decode stall the update causes
    rec_nu = []
    for _ in range(max(3, steps // 2)):
        step(rec_nu, update=False)

    tokens = sum(r["tokens"] for r in rec)
    dev_ms = sum(r["dev_ms"] for r in rec)
    wall_ms = sum(r["wall_ms"] for r in rec)
    out = {
        "tokens": tokens, "dev_ms": dev_ms, "wall_ms": wall_ms,
        "launches": sum(r["launches"] for r in rec),
        "h2d_bytes_per_step": (h2d[0] - h2d0) // steps, "d2h_bytes_per_step": (d2h[0] - d2h0) // steps,
        "clocks": clk, "ctx_now": ctx_now, "max_seq": max_seq,
    }
    per_upd = float(np.mean([r["decode_ms"] + r["pause_ms"] + max(0.0, r["copy_ms"] - r["decode_ms"])
                             for r in rec]))
    per_nu = float(np.mean([r["decode_ms"] for r in rec_nu]))
    nbytes = pol.weights()[1]
    out["pause"] = {
        "swap_ms": {"median": float(np.median([r["pause_ms"] for r in rec])),
                    "max": float(np.max([r["pause_ms"] for r in rec]))},
        "decode_stall_ms": per_upd - per_nu,
        "step_ms_with_update": per_upd, "step_ms_without_update": per_nu,
        "transfer_ms": float(np.median([r["copy_ms"] for r in rec])),
        "transfer_gbs": nbytes / (float(np.median([r["copy_ms"] for r in rec])) * 1e-3) / 1e9,
        "payload_bytes": nbytes,
        "transfer": "D2D cudaMemcpyAsync into the standby buffer on a side stream, overlapped with "
                    "the decode rounds: it advances between rounds (the megakernel holds every SM), "
                    "so transfer_ms spans the step and decode_stall_ms is what it costs decode "
                    "(N = 1: the trainer shares the GPU; N > 1: ncclBroadcast over NVLink)",
    }
    if lag and consumed:
        # lag of every consumed sequence (sim.cpp:63-104), on the device
        mx, tot, cnt = 0, 0, 0
        for vb in sorted({vb for vb, _ in consumed}):
            idx = [i for i, (b, _) in enumerate(consumed) if b == vb]
            sub = [consumed[i][1] for i in idx]
            sv = torch.tensor(np.concatenate([np.asarray(v, np.int32) for v in sub]), device=dev)
            so = torch.tensor(np.concatenate([[0], np.cumsum([len(v) for v in sub])]),
                              dtype=torch.int64, device=dev)
            hist = torch.zeros(8192, dtype=torch.int64, device=dev)
            sums = torch.zeros(len(sub), dtype=torch.int64, device=dev)
            t4 = torch.zeros(4, dtype=torch.int64, device=dev)
            _lib.call("srl_lag_stats", sv.data_ptr(), so.data_ptr(), len(sub), vb, hist.data_ptr(),
                      8192, sums.data_ptr(), t4.data_ptr(), None)
            t = t4.cpu().tolist()
            cnt += t[0]
            tot += t[1]
            mx = max(mx, t[2])
        out["lag"] = {"consumed_sequences": len(consumed), "tokens": cnt, "max_lag_steps": mx,
                      "mean_lag_steps": tot / max(cnt, 1),
                      "updates_per_rollout": int(np.ceil(gen / R)),
                      "definition": "each finished sequence consumed at the drain that saw it "
                                    "finish; lag = version then - version that emitted the token "
                                    "(sim.cpp:74); one update every rounds_per_step rounds"}
    # roofline of the dominant kernel (profiled rounds)
    hbm, _, peak_kind = load_peaks()
    abytes = algorithmic_bytes(cfg, B, sum(ctx_now))
    step_bytes = sum(abytes.values())
    cls_ms = {k: prof[k][0] for k in KERNEL_CLASSES} if prof else {}
    traffic = load_traffic().get(f"{cfg.name}:{B}:{gen}", {})
    if fused_ms:
        mk_ms = float(np.mean(fused_ms))
        roof = {"kernel": "decode_megakernel", "bound": "hbm",
                "achieved": step_bytes / (mk_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_kind": peak_kind, "traffic": traffic.get("decode_megakernel"),
                "launches_per_round": 1, "bytes_per_launch": step_bytes, "ms_per_launch": mk_ms,
                "ms_per_launch_samples": len(fused_ms),
                "phase_ms_per_round": {k: round(v, 4) for k, v in cls_ms.items()}}
        round_ms = mk_ms
    elif cls_ms:
        dom = max(cls_ms, key=cls_ms.get)
        round_ms = sum(cls_ms.values())
        nlaunch = max(prof[dom][1], 1)
        roof = {"kernel": dom, "bound": "hbm", "achieved": abytes[dom] / (cls_ms[dom] * 1e-3) / 1e9,
                "peak": hbm, "unit": "GB/s", "peak_kind": peak_kind,
                "traffic": traffic.get(dom), "launches_per_round": prof[dom][1],
                "bytes_per_launch": abytes[dom] / nlaunch, "ms_per_launch": cls_ms[dom] / nlaunch}
    else:
        roof, round_ms = None, None
    if roof:
        roof["frac"] = roof["achieved"] / roof["peak"]
        out["roofline"] = roof
        out["round_roofline"] = {"bound": "hbm", "achieved": step_bytes / (round_ms * 1e-3) / 1e9,
                                 "peak": hbm, "unit": "GB/s", "bytes": step_bytes, "ms": round_ms,
                                 "ctx_sum": int(sum(ctx_now)),
                                 "bytes_by_class": {k: int(v) for k, v in abytes.items()},
                                 "frac": step_bytes / (round_ms * 1e-3) / 1e9 / hbm}
        out["roofline_tokens_per_s"] = B / (step_bytes / (hbm * 1e9))
        out["kernel_ms_per_round"] = {k: round(v, 4) for k, v in cls_ms.items()}
    out["prefill"] = {"ms_per_step": sum(r["prefill_ms"] for r in rec) / steps,
                      "rows_per_step": sum(r["prefill_rows"] for r in rec) / steps,
                      "note": "refill prefill rounds of finished streams (inside value's device time)"}
    eng.close()
    return out, pol


def cpu_sample(cfg, contexts, rounds=2):
    """The CPU port (oracle/decoder_cpu.py) on the same streams and contexts."""
    from oracle.decoder_cpu import time_rounds

    tps, dt, cores = time_rounds(cfg.to_dict(), contexts, rounds)
    return {"value": tps, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(contexts)} streams x {rounds} decode rounds at the measured contexts "
                      f"(mean {np.mean(contexts):.0f} tokens), oracle/decoder_cpu.py numpy fp32 "
                      f"on all host cores ({dt:.1f} s); the reference has no decoder"}


# ------------------------------------------------------ reference arm ---
def reference_arm(args, cfg):
    """The CPU path on the host cores, same config as our arm: each step is one
    decode round of the same B streams at the same steady-state contexts
    (oracle/decoder_cpu.py: the reference has no transformer, so this is the
    builder's port).  Next to it, the REFERENCE ITSELF (oracle/_ref, compiled
    from /root/reference on the build machine): its Engine on the toy
    recurrent policy, one instance per core, and its update pause
    (policy_to_json + crc32 + policy_from_json + apply_weight_update)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.decoder_cpu import CpuDecoder

    B = args.batch
    ctx = [1 + args.prompt + d for d, _ in steady_contexts(B, args.prompt, args.gen)] \
        if not args.no_steady else [1 + args.prompt] * B
    dec = CpuDecoder(cfg.to_dict())
    dec.add_streams(ctx, max(ctx) + args.steps + args.warmup + 1)
    toks = np.zeros(B, dtype=np.int64)
    for _ in range(args.warmup):
        toks = dec.round(toks)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        toks = dec.round(toks)
    dt = time.perf_counter() - t0
    tps = B * args.steps / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic prompts, random-init weights",
        "config": {"workload": f"{cfg.name} generator, constant batch {B}, rollouts of up to "
                               f"{args.gen} tokens (steady-state contexts), CPU",
                   "model": cfg.name, "global_batch": B, "seq_len": 1 + args.prompt + args.gen + 1,
                   "parallelism": "cpu", "same_config": True,
                   "sample": "each step = one decode round of the same B streams at the same "
                             "contexts as the device run (no update: the CPU time per token is "
                             "dominated by the round)"},
        "cpu_baseline": {"value": tps, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{B} streams x {args.steps} decode rounds, mean context "
                                   f"{np.mean(ctx):.0f} tokens, oracle/decoder_cpu.py numpy fp32"},
        "e2e": {"value": tps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:  # the reference itself, on the configuration it can run
        from oracle.oracle import Ref

        ref = Ref()
        doc = ref.random_recurrent_policy(256, 128, 0.6, 1)
        nxt = ref.drift_checkpoints(doc, 1, 0.05, 2)[-1]
        tok, sec = ref.engine_throughput_parallel(doc, cores, 64, 200)
        tok1, sec1 = ref.engine_throughput(doc, 64, 200)
        line["reference_engine_toy"] = {
            "value": tok / sec, "unit": UNIT, "cores": cores, "kind": "reference",
            "one_core": tok1 / sec1,
            "sample": f"{cores} x reference proto::Engine (RecurrentToyPolicy V=256 D=128), 64 "
                      f"streams x 200 tokens each, one instance per core (oracle/_ref)"}
        line["reference_pause_toy"] = {
            "stale": ref.update_pause(doc, nxt, 64, 128, False),
            "recompute": ref.update_pause(doc, nxt, 64, 128, True),
            "note": "reference update path for the toy policy (V=256, D=128): policy_to_json + "
                    "crc32 + policy_from_json + apply_weight_update with 64 live streams"}
    except Exception as e:  # noqa: BLE001 -- oracle/_ref is only built where /root/reference exists
        line["reference_engine_toy"] = {"unavailable": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- ours ---
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    from paper_2509_19128_b200.policy import PRESETS

    cfg = PRESETS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    world, rank, local = dist_env()
    if world > 1:
        from paper_2509_19128_b200.pipeline_dist import bench_partitioned

        line = bench_partitioned(args, cfg)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    B, R = args.batch, args.rounds
    g, pol = generator_measure(cfg, B=B, prompt=args.prompt, gen=args.gen, R=R, steps=args.steps,
                               warmup=args.warmup, steady=not args.no_steady,
                               use_graphs=not args.no_graphs, device=local)
    value = g["tokens"] / (g["dev_ms"] * 1e-3)
    e2e = g["tokens"] / (g["wall_ms"] * 1e-3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": g["dev_ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts, random-init weights",
        "config": {"workload": f"{cfg.name} generator, constant batch {B}, rollouts of up to "
                               f"{args.gen} tokens" + ("" if args.no_steady else
                                                       " (steady-state contexts)")
                               + f", in-flight update every {R} decode rounds",
                   "model": cfg.name, "global_batch": B, "seq_len": g["max_seq"],
                   "prompt": args.prompt, "max_tokens": args.gen, "rounds_per_step": R,
                   "parallelism": "1 GPU: generator (update = device copy into the standby buffer)",
                   "cuda_graphs": not args.no_graphs,
                   "l2": "inputs larger than L2 (weights + KV caches streamed every round)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": g["h2d_bytes_per_step"],
                "d2h_bytes_per_step": g["d2h_bytes_per_step"]},
        "gpu_launches": g["launches"],
        "pause_ms": g["pause"]["swap_ms"],
        "pause": g["pause"],
        "lag": g.get("lag"),
        "roofline": g.get("roofline"),
        "round_roofline": g.get("round_roofline"),
        "roofline_tokens_per_s": g.get("roofline_tokens_per_s"),
        "kernel_ms_per_round": g.get("kernel_ms_per_round"),
        "prefill": g["prefill"],
        "clocks": g["clocks"],
    }
    ctx_now = g["ctx_now"]
    if not args.no_trainer:
        log("trainer")
        tclk = ClockSampler(local).start()
        out["trainer"] = trainer_measure(cfg, pol, args.train_seqs, args.prompt, args.train_gen)
        out["trainer"]["clocks"] = tclk.stop()
        log("trainer (fast bf16 mode)")
        out["trainer_fast"] = trainer_measure(cfg, pol, args.train_seqs, args.prompt, args.train_gen,
                                              precise=False)
    if not args.no_pipeline:
        log("recompute-mode pause")
        payload = pol.clone().perturb(99, 0.002)
        out["pause_ms_recompute_mode"] = recompute_pause_measure(cfg, pol, payload, B, args.prompt)
        del payload
        log("pipeline_1gpu")
        out["pipeline_1gpu"] = pipeline_measure(cfg, B, args.prompt, args.train_gen, R)
    del pol
    if not args.no_extra:
        out["extra_configs"] = {}
        for spec in filter(None, args.extra.split(",")):
            name, b, gen, *mode = spec.split(":")
            precise = bool(mode) and mode[0] == "precise"
            c = PRESETS[name]
            log(f"extra config {spec}")
            try:
                e, p = generator_measure(c, B=int(b), prompt=args.prompt, gen=int(gen), R=R,
                                         steps=max(3, args.steps // 2), warmup=2, steady=True,
                                         use_graphs=not args.no_graphs, device=local, n_payloads=1,
                                         precise=precise)
                del p
                out["extra_configs"][spec] = {
                    "note": ("precise engine: activations between the GEMMs as bf16 hi + lo pairs "
                             "(multi-kernel round), log-probs within 1e-3 of the fp64 oracle")
                            if precise else None,
                    "value": e["tokens"] / (e["dev_ms"] * 1e-3), "e2e": e["tokens"] / (e["wall_ms"] * 1e-3),
                    "ms_per_step": e["dev_ms"] / max(3, args.steps // 2),
                    "pause": e["pause"], "roofline": e.get("roofline"),
                    "round_roofline": {k: v for k, v in (e.get("round_roofline") or {}).items()
                                       if k != "bytes_by_class"},
                    "roofline_tokens_per_s": e.get("roofline_tokens_per_s"),
                    "lag": e.get("lag"), "clocks": e["clocks"]}
            except Exception as ex:  # noqa: BLE001 -- an extra line must not sink the headline
                out["extra_configs"][spec] = {
                    "note": ("precise engine: activations between the GEMMs as bf16 hi + lo pairs "
                             "(multi-kernel round), log-probs within 1e-3 of the fp64 oracle")
                            if precise else None,"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
    if not args.no_cpu_baseline:
        log("cpu baseline")
        out["cpu_baseline"] = cpu_sample(cfg, ctx_now)
    log("done")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
