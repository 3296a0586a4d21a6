"""CPU decode baseline for bench.py.  TEST INFRASTRUCTURE ONLY.

The reference (/root/reference/proj) has no transformer, so the CPU arm of the
benchmark cannot run the reference's own code at the Qwen shapes.  This module
is the builder's port of the same decode round the device engine runs
(decoder_oracle.py's algorithm: RMSNorm, QKV + bias, RoPE, causal GQA
attention over the stream's KV cache, O, SwiGLU MLP, LM head, log-softmax,
one token per stream per round -- engine.cpp:119-153 semantics), written for
speed on the host rather than as a checker: fp32 numpy, every projection
batched over the streams (BLAS on all host cores), per-stream K/V kept in
preallocated [layer, kv head, position, head dim] arrays so each head's
attention is two BLAS calls (fp32, or fp16 storage when host memory is short).

Only bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm use it, on
a bounded sample (a few rounds of the same streams and contexts as the device
run); nothing in paper_2509_19128_b200/ imports it.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np


class CpuDecoder:
    def __init__(self, cfg: dict, seed: int = 0, scale: float = 0.02):
        self.cfg = cfg
        H, V, L = cfg["hidden"], cfg["vocab_size"], cfg["layers"]
        nq, nkv, hd, I = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"], cfg["intermediate"]
        qkv = (nq + 2 * nkv) * hd
        rng = np.random.default_rng(seed)
        # random-init weights; the timing does not depend on the values, so large
        # matrices repeat one 4M-element random block (host setup in seconds)
        block = rng.standard_normal(1 << 22, dtype=np.float32) * np.float32(scale)

        def mat(*shape):
            n = int(np.prod(shape))
            out = np.empty(n, dtype=np.float32)
            for o in range(0, n, block.size):
                out[o:o + block.size] = block[:min(block.size, n - o)]
            return out.reshape(shape)

        self.embed = mat(V, H)
        self.lm_head = self.embed if cfg["tie_embeddings"] else mat(V, H)
        self.layers = []
        for _ in range(L):
            self.layers.append(dict(ln1=np.ones(H, np.float32), qkv_w=mat(qkv, H),
                                    qkv_b=mat(qkv), o_w=mat(H, nq * hd), ln2=np.ones(H, np.float32),
                                    gate_w=mat(I, H), up_w=mat(I, H), down_w=mat(H, I)))
        self.final_norm = np.ones(H, np.float32)
        half = hd // 2
        self.inv_freq = (cfg["rope_theta"] ** (-2.0 * np.arange(half) / hd)).astype(np.float64)
        self.scale = np.float32(1.0 / math.sqrt(hd))
        self.kv = []  # per stream: [L, 2, nkv, cap, hd]
        self.ctx = []
        self.kv_dtype = np.float32

    def _norm(self, x, g):
        r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + np.float32(self.cfg["rms_eps"]))
        return (x * r * g).astype(np.float32)

    def _rope(self, x, pos):
        half = self.cfg["head_dim"] // 2
        ang = pos[:, None].astype(np.float64) * self.inv_freq
        c = np.cos(ang).astype(np.float32)[:, None, :]
        s = np.sin(ang).astype(np.float32)[:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    def add_streams(self, contexts, capacity, seed=1):
        """Streams whose caches already hold `contexts[i]` positions (random
        K/V contents: the timing of a round does not depend on them)."""
        L, nkv, hd = self.cfg["layers"], self.cfg["kv_heads"], self.cfg["head_dim"]
        need = len(contexts) * L * 2 * nkv * capacity * hd * 4
        try:
            import psutil

            if need > 0.6 * psutil.virtual_memory().available:
                self.kv_dtype = np.float16
        except ImportError:
            pass
        rng = np.random.default_rng(seed)
        tile = rng.standard_normal((L, 2, nkv, 256, hd), dtype=np.float32).astype(self.kv_dtype)
        for c in contexts:
            kv = np.empty((L, 2, nkv, capacity, hd), dtype=self.kv_dtype)
            for o in range(0, c, 256):
                n = min(256, c - o)
                kv[:, :, :, o:o + n] = tile[:, :, :, :n]
            self.kv.append(kv)
            self.ctx.append(int(c))

    def round(self, tokens):
        """One decode round: every stream feeds one token; returns greedy next tokens."""
        cfg = self.cfg
        nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
        G = nq // nkv
        rows = len(tokens)
        pos = np.asarray(self.ctx, dtype=np.int64)
        x = self.embed[np.asarray(tokens)]
        for l, w in enumerate(self.layers):
            xn = self._norm(x, w["ln1"])
            qkv = xn @ w["qkv_w"].T + w["qkv_b"]
            q = self._rope(qkv[:, :nq * hd].reshape(rows, nq, hd), pos)
            k = self._rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(rows, nkv, hd), pos)
            v = qkv[:, (nq + nkv) * hd:].reshape(rows, nkv, hd)
            attn = np.empty((rows, nq, hd), dtype=np.float32)
            qs = q.reshape(rows, nkv, G, hd) * self.scale
            for r in range(rows):
                kv = self.kv[r]
                t = self.ctx[r]
                kv[l, 0, :, t] = k[r]
                kv[l, 1, :, t] = v[r]
                for kh in range(nkv):
                    K = kv[l, 0, kh, :t + 1]                      # [T, hd]
                    Vv = kv[l, 1, kh, :t + 1]
                    if K.dtype != np.float32:
                        K, Vv = K.astype(np.float32), Vv.astype(np.float32)
                    s = qs[r, kh] @ K.T                           # [G, T]
                    s = np.exp(s - s.max(-1, keepdims=True))
                    s /= s.sum(-1, keepdims=True)
                    attn[r, kh * G:(kh + 1) * G] = s @ Vv
            x = x + attn.reshape(rows, nq * hd) @ w["o_w"].T
            xn = self._norm(x, w["ln2"])
            g = xn @ w["gate_w"].T
            u = xn @ w["up_w"].T
            x = x + ((g / (1.0 + np.exp(-g))) * u) @ w["down_w"].T
        logits = self._norm(x, self.final_norm) @ self.lm_head.T
        m = logits.max(-1, keepdims=True)
        lp = logits - (m + np.log(np.exp(logits - m).sum(-1, keepdims=True)))  # log-softmax
        nxt = lp.argmax(-1)
        for r in range(rows):
            self.ctx[r] += 1
        return nxt


def time_rounds(cfg: dict, contexts, rounds: int, warmup: int = 1, seed: int = 0):
    """(tokens/s, seconds, cores) of `rounds` decode rounds over streams at
    `contexts` (same streams, same context lengths as the device run)."""
    dec = CpuDecoder(cfg, seed)
    dec.add_streams(contexts, max(contexts) + warmup + rounds + 1)
    toks = np.random.default_rng(seed + 1).integers(0, cfg["vocab_size"], size=len(contexts))
    for _ in range(warmup):
        toks = dec.round(toks)
    t0 = time.perf_counter()
    for _ in range(rounds):
        toks = dec.round(toks)
    dt = time.perf_counter() - t0
    return len(contexts) * rounds / dt, dt, os.cpu_count()
