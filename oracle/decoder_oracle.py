"""CPU restatement of the decoder policy (numpy).  TEST INFRASTRUCTURE ONLY.

The reference has no transformer: its "policy model" is
a tabular or 1-layer tanh RNN policy walked by PolicyWalker
(/root/reference/proj/core/src/rl_math.cpp:27-82).  This module restates the
decoder policy this framework adds -- Qwen2.5-shaped, bf16 weights -- with the
PolicyWalker contract: per-position log-probabilities in the log domain,
state (the KV cache) carried across checkpoint switches, stale or recomputed
after a switch (rl_math.cpp:64-73, engine.cpp:103-113).

It rounds to bf16 at exactly the points the device path does (normalised
activations, q/k/v, attention output, SwiGLU output) and accumulates every
dot product in fp64, so GPU-vs-oracle differences come only from fp32
accumulation order.  The reference has no transformer to pin it against;
tests/test_decoder_oracle.py pins it to an independent implementation
instead: with the rounding points off (exact=True) it equals transformers'
Qwen2ForCausalLM (5.5.0, float64) to 1e-9 on random Qwen2-shaped weights in
this layout, and central finite differences of its IS-REINFORCE objective
equal the fp64 autograd gradient that the device trainer is checked against
(tests/torch_decoder_ref.py), the recipe of test_rl_math.cpp:57-90.
"""
from __future__ import annotations

import math

import numpy as np


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    b = a.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_bits_to_f32(u16):
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def layout(cfg):
    """Element offsets of the flat weight buffer (csrc/decoder.cu make_layout)."""
    H, V, L = cfg["hidden"], cfg["vocab_size"], cfg["layers"]
    nq, nkv, hd, I = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"], cfg["intermediate"]
    qkv = (nq + 2 * nkv) * hd
    cur = 0
    off = {}

    def take(name, n):
        nonlocal cur
        off[name] = (cur, n)
        cur += (n + 63) // 64 * 64

    take("embed", V * H)
    for l in range(L):
        take(f"{l}.ln1", H)
        take(f"{l}.qkv_w", qkv * H)
        take(f"{l}.qkv_b", qkv)
        take(f"{l}.o_w", H * nq * hd)
        take(f"{l}.ln2", H)
        take(f"{l}.gate_up_w", 2 * I * H)
        take(f"{l}.down_w", H * I)
    take("final_norm", H)
    if cfg["tie_embeddings"]:
        off["lm_head"] = off["embed"]
    else:
        take("lm_head", V * H)
    return off, cur


class DecoderOracle:
    """fp64-accumulating decoder forward with a per-stream KV cache."""

    def __init__(self, cfg: dict, weights_u16: np.ndarray, dtype=np.float64, exact: bool = False,
                 rounding: str = "device"):
        """exact=True drops the device's bf16 rounding points and fp32 storage
        of activations (every value fp64): the plain Qwen2 forward, the form
        pinned against transformers' Qwen2ForCausalLM (tests/test_decoder_oracle.py).
        rounding="kv": the precise engine's rounding points only -- q, k, v
        (the bf16 K/V cache and query operand); the normalised inputs, the
        attention output and the SwiGLU output stay fp32 (the device carries
        them as bf16 hi + lo pairs)."""
        self.cfg = cfg
        self.dtype = np.float64 if exact else dtype
        self.exact = exact
        self._f = np.float64 if exact else np.float32
        self._rnd = (lambda a: np.asarray(a, dtype=np.float64)) if exact else bf16_round
        # rounding points of the activations between the GEMMs
        self._rnd_act = (lambda a: np.asarray(a, dtype=np.float32)) if (rounding == "kv" and not exact) \
            else self._rnd
        self.off, total = layout(cfg)
        w = np.asarray(weights_u16)
        if w.size < total:
            raise ValueError("weight buffer smaller than the layout")
        self.w = {}
        H, I = cfg["hidden"], cfg["intermediate"]
        nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
        qkv = (nq + 2 * nkv) * hd
        shapes = {"embed": (cfg["vocab_size"], H), "lm_head": (cfg["vocab_size"], H),
                  "final_norm": (H,)}
        for l in range(cfg["layers"]):
            shapes.update({f"{l}.ln1": (H,), f"{l}.qkv_w": (qkv, H), f"{l}.qkv_b": (qkv,),
                           f"{l}.o_w": (H, nq * hd), f"{l}.ln2": (H,),
                           f"{l}.gate_up_w": (2 * I, H), f"{l}.down_w": (H, I)})
        for name, (o, n) in self.off.items():
            vals = w[o:o + n] if w.dtype == np.float64 else bf16_bits_to_f32(w[o:o + n])
            self.w[name] = vals.reshape(shapes[name]).astype(self.dtype)
        half = hd // 2
        self.inv_freq = cfg["rope_theta"] ** (-2.0 * np.arange(half) / hd)
        self.scale = self._f(1.0 / math.sqrt(hd))

    @classmethod
    def from_flat64(cls, cfg: dict, flat64: np.ndarray):
        """Exact-mode oracle over arbitrary fp64 weight values in the flat
        layout (finite-difference probes perturb single weights)."""
        return cls(cfg, np.asarray(flat64, dtype=np.float64), exact=True)

    # ------------------------------------------------------------ pieces
    def _rstd(self, x):
        ssq = (x.astype(np.float64) ** 2).sum(-1)
        return 1.0 / np.sqrt(ssq / self.cfg["hidden"] + self.cfg["rms_eps"])

    def _xg(self, x, gain):
        return self._rnd_act(x.astype(self._f) * gain.astype(self._f)).astype(self.dtype)

    def _rope(self, x, pos):
        """x: [..., hd] fp32 values at integer position pos (scalar or [rows])."""
        hd = self.cfg["head_dim"]
        half = hd // 2
        ang = np.asarray(pos, dtype=np.float64)[..., None] * self.inv_freq
        c = np.cos(ang).astype(self._f)
        s = np.sin(ang).astype(self._f)
        while c.ndim < x.ndim:
            c, s = c[..., None, :], s[..., None, :]
        x1, x2 = x[..., :half].astype(self._f), x[..., half:].astype(self._f)
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    def new_cache(self):
        L = self.cfg["layers"]
        return {"k": [[] for _ in range(L)], "v": [[] for _ in range(L)], "tokens": []}

    # ------------------------------------------------------------- step
    def step(self, caches, tokens, positions):
        """Feed one token per stream (rows), append K/V, return fp64 logits [rows x V]."""
        cfg, w = self.cfg, self.w
        H, I = cfg["hidden"], cfg["intermediate"]
        nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
        G = nq // nkv
        tokens = np.asarray(tokens)
        rows = len(tokens)
        x = w["embed"][tokens].astype(self._f)  # fp32 residual stream
        xg = self._xg(x, w["0.ln1"])
        rstd = self._rstd(x)
        for l in range(cfg["layers"]):
            qkv = (xg @ w[f"{l}.qkv_w"].T) * rstd[:, None] + w[f"{l}.qkv_b"]
            qkv = qkv.astype(self._f)
            q = qkv[:, :nq * hd].reshape(rows, nq, hd)
            k = qkv[:, nq * hd:(nq + nkv) * hd].reshape(rows, nkv, hd)
            v = qkv[:, (nq + nkv) * hd:].reshape(rows, nkv, hd)
            q = self._rnd(self._rope(q, positions))
            k = self._rnd(self._rope(k, positions))
            v = self._rnd(v)
            attn = np.zeros((rows, nq, hd), dtype=np.float64)
            for r in range(rows):
                c = caches[r]
                c["k"][l].append(k[r])
                c["v"][l].append(v[r])
                K = np.stack(c["k"][l]).astype(np.float64)  # [T, nkv, hd]
                Vv = np.stack(c["v"][l]).astype(np.float64)
                qs = (q[r].astype(self._f) * self.scale).astype(np.float64)  # [nq, hd]
                for h in range(nq):
                    kh = h // G
                    s = K[:, kh, :] @ qs[h]
                    p = np.exp(s - s.max())
                    attn[r, h] = (p @ Vv[:, kh, :]) / p.sum()
            attn = self._rnd_act(attn.reshape(rows, nq * hd)).astype(self.dtype)
            x = (x + attn @ w[f"{l}.o_w"].T).astype(self._f)
            xg = self._xg(x, w[f"{l}.ln2"])
            rstd = self._rstd(x)
            gu = (xg @ w[f"{l}.gate_up_w"].T) * rstd[:, None]
            gu = gu.reshape(rows, I // 64, 2, 64)
            g, u = gu[:, :, 0, :].reshape(rows, I), gu[:, :, 1, :].reshape(rows, I)
            g32, u32 = g.astype(self._f), u.astype(self._f)
            act = self._rnd_act(g32 / (self._f(1) + np.exp(-g32)) * u32).astype(self.dtype)
            x = (x + act @ w[f"{l}.down_w"].T).astype(self._f)
            nxt = w[f"{l + 1}.ln1"] if l + 1 < cfg["layers"] else w["final_norm"]
            xg = self._xg(x, nxt)
            rstd = self._rstd(x)
        for r in range(rows):
            caches[r]["tokens"].append(int(tokens[r]))
        return (xg @ w["lm_head"].T) * rstd[:, None]

    def prefill_fast(self, cache, tokens, chunk: int = 256):
        """prefill() for one stream with the rows of each chunk batched (BLAS-3
        instead of one matrix-vector product per token): the same operations,
        dtypes and rounding points as step(), causal attention over the cache;
        only the fp64 summation order of the products differs.  Returns the
        logits of the last position."""
        cfg, w = self.cfg, self.w
        I = cfg["intermediate"]
        nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
        G = nq // nkv
        last = None
        for c0 in range(0, len(tokens), chunk):
            toks = np.asarray(tokens[c0:c0 + chunk])
            rows = len(toks)
            p0 = len(cache["tokens"])
            pos = np.arange(p0, p0 + rows)
            x = w["embed"][toks].astype(self._f)
            xg = self._xg(x, w["0.ln1"])
            rstd = self._rstd(x)
            for l in range(cfg["layers"]):
                qkv = ((xg @ w[f"{l}.qkv_w"].T) * rstd[:, None] + w[f"{l}.qkv_b"]).astype(self._f)
                q = self._rnd(self._rope(qkv[:, :nq * hd].reshape(rows, nq, hd), pos))
                k = self._rnd(self._rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(rows, nkv, hd), pos))
                v = self._rnd(qkv[:, (nq + nkv) * hd:].reshape(rows, nkv, hd))
                cache["k"][l].extend(list(k))
                cache["v"][l].extend(list(v))
                K = np.stack(cache["k"][l]).astype(np.float64)  # [T, nkv, hd]
                Vv = np.stack(cache["v"][l]).astype(np.float64)
                qs = (q.astype(self._f) * self.scale).astype(np.float64)  # [rows, nq, hd]
                mask = np.arange(K.shape[0])[None, :] > pos[:, None]
                attn = np.zeros((rows, nq, hd), dtype=np.float64)
                for h in range(nq):
                    kh = h // G
                    sc = qs[:, h, :] @ K[:, kh, :].T  # [rows, T]
                    sc = np.where(mask, -np.inf, sc)
                    pr = np.exp(sc - sc.max(-1, keepdims=True))
                    attn[:, h] = (pr @ Vv[:, kh, :]) / pr.sum(-1, keepdims=True)
                attn = self._rnd_act(attn.reshape(rows, nq * hd)).astype(self.dtype)
                x = (x + attn @ w[f"{l}.o_w"].T).astype(self._f)
                xg = self._xg(x, w[f"{l}.ln2"])
                rstd = self._rstd(x)
                gu = ((xg @ w[f"{l}.gate_up_w"].T) * rstd[:, None]).reshape(rows, I // 64, 2, 64)
                g32 = gu[:, :, 0, :].reshape(rows, I).astype(self._f)
                u32 = gu[:, :, 1, :].reshape(rows, I).astype(self._f)
                act = self._rnd_act(g32 / (self._f(1) + np.exp(-g32)) * u32).astype(self.dtype)
                x = (x + act @ w[f"{l}.down_w"].T).astype(self._f)
                nxt = w[f"{l + 1}.ln1"] if l + 1 < cfg["layers"] else w["final_norm"]
                xg = self._xg(x, nxt)
                rstd = self._rstd(x)
            cache["tokens"].extend(int(t) for t in toks)
            last = (xg[-1:] @ w["lm_head"].T) * rstd[-1:, None]
        return last[0] if last is not None else None

    def prefill(self, cache, tokens):
        """Feed a whole prefix into one cache; returns logits of every position."""
        out = []
        for p, t in enumerate(tokens):
            out.append(self.step([cache], [t], [len(cache["tokens"])])[0])
        return np.stack(out) if out else np.zeros((0, self.cfg["vocab_size"]))

    def recompute(self, cache):
        """Recompute mode: rebuild the cache from its tokens under these weights."""
        fresh = self.new_cache()
        self.prefill(fresh, list(cache["tokens"]))
        cache.update(fresh)

    @staticmethod
    def log_softmax(logits):
        m = logits.max(-1, keepdims=True)
        return logits - (m + np.log(np.exp(logits - m).sum(-1, keepdims=True)))

    def sequence_logprobs(self, tokens):
        """policy_logprobs (rl_math.cpp:128-142) of tokens after bos."""
        cache = self.new_cache()
        inputs = [self.cfg["bos_token"]] + list(tokens[:-1])
        logits = self.prefill(cache, inputs)
        lp = self.log_softmax(logits)
        return lp[np.arange(len(tokens)), tokens]
