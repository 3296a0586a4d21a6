"""float64 torch-autograd restatement of the decoder policy and the
IS-REINFORCE objective, used only as the reference for the device trainer's
gradient (a floating-point kernel: the one place tests use torch as the
reference).  bf16 rounding points of the device forward are mimicked with a
straight-through estimator so forward values match the device to fp32
accumulation order.
"""
import math

import numpy as np
import torch

from oracle.decoder_oracle import bf16_bits_to_f32, layout


def bf16_st(x):
    return x + (x.to(torch.float32).to(torch.bfloat16).to(x.dtype) - x).detach()


class TorchDecoder:
    def __init__(self, cfg: dict, flat_u16: np.ndarray, exact: bool = False, rounding: str = "device",
                 dtype=torch.float64):
        """exact=True: no bf16 rounding points, fp64 RoPE tables and scale
        (pinned against transformers' Qwen2 in tests/test_decoder_oracle.py).
        rounding (exact=False): "device" = every bf16 rounding point of the
        generator / fast trainer (normalised inputs, q/k/v, attention output,
        SwiGLU output); "kv" = the precise trainer's, which carries every
        activation as a bf16 hi + lo pair and rounds only q, k, v (the paged
        K/V cache and the query operand are bf16)."""
        self.cfg = cfg
        self.exact = exact
        self.rounding = rounding
        self.dtype = dtype  # float32: the same restatement at fp32 accumulation (self-spread)
        self.off, self.total = layout(cfg)
        H, I = cfg["hidden"], cfg["intermediate"]
        nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
        qkv = (nq + 2 * nkv) * hd
        shapes = {"embed": (cfg["vocab_size"], H), "final_norm": (H,)}
        for l in range(cfg["layers"]):
            shapes.update({f"{l}.ln1": (H,), f"{l}.qkv_w": (qkv, H), f"{l}.qkv_b": (qkv,),
                           f"{l}.o_w": (H, nq * hd), f"{l}.ln2": (H,),
                           f"{l}.gate_up_w": (2 * I, H), f"{l}.down_w": (H, I)})
        if not cfg["tie_embeddings"]:
            shapes["lm_head"] = (cfg["vocab_size"], H)
        self.p = {}
        for name, shape in shapes.items():
            o, n = self.off[name]
            t = torch.tensor(bf16_bits_to_f32(flat_u16[o:o + n]).astype(np.float64)).reshape(shape)
            self.p[name] = t.to(dtype).requires_grad_(True)

    def flat_grad(self):
        g = np.zeros(self.total)
        for name, t in self.p.items():
            o, n = self.off[name]
            if t.grad is not None:
                g[o:o + n] += t.grad.detach().cpu().numpy().ravel()
        return g

    def logprobs(self, tokens):
        """log pi(tokens[p+1] | tokens[:p+1]) for p = 0..n-2 (tokens[0] = bos)."""
        c, p = self.cfg, self.p
        H, I = c["hidden"], c["intermediate"]
        nq, nkv, hd = c["q_heads"], c["kv_heads"], c["head_dim"]
        G, half = nq // nkv, hd // 2
        inp = torch.tensor(tokens[:-1])
        tgt = torch.tensor(tokens[1:])
        T = len(inp)
        x = p["embed"][inp]
        pos = torch.arange(T, dtype=torch.float64)
        inv = c["rope_theta"] ** (-2.0 * torch.arange(half, dtype=torch.float64) / hd)
        ang = pos[:, None] * inv
        if self.exact:
            cos, sin = ang.cos(), ang.sin()
        else:
            cos = ang.cos().to(torch.float32).to(torch.float64)
            sin = ang.sin().to(torch.float32).to(torch.float64)
        cos, sin = cos.to(self.dtype), sin.to(self.dtype)
        bf16 = (lambda z: z) if (self.exact or self.rounding == "kv") else bf16_st
        bf16_qkv = (lambda z: z) if self.exact else bf16_st

        def rope(z):  # [T, heads, hd]
            z1, z2 = z[..., :half], z[..., half:]
            return torch.cat([z1 * cos[:, None] - z2 * sin[:, None],
                              z2 * cos[:, None] + z1 * sin[:, None]], -1)

        def rstd(z):
            return 1.0 / torch.sqrt((z * z).mean(-1) + c["rms_eps"])

        mask = torch.ones(T, T, dtype=torch.bool).tril()
        scale = 1.0 / math.sqrt(hd) if self.exact else float(np.float32(1.0 / math.sqrt(hd)))
        for l in range(c["layers"]):
            u = bf16(x * p[f"{l}.ln1"])
            qkv = rstd(x)[:, None] * (u @ p[f"{l}.qkv_w"].T) + p[f"{l}.qkv_b"]
            q = bf16_qkv(rope(qkv[:, :nq * hd].reshape(T, nq, hd)))
            k = bf16_qkv(rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(T, nkv, hd)))
            v = bf16_qkv(qkv[:, (nq + nkv) * hd:].reshape(T, nkv, hd))
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            s = torch.einsum("thd,shd->hts", q * scale, k)
            s = s.masked_fill(~mask, float("-inf"))
            a = torch.softmax(s, -1)
            o = bf16(torch.einsum("hts,shd->thd", a, v).reshape(T, nq * hd))
            x = x + o @ p[f"{l}.o_w"].T
            u2 = bf16(x * p[f"{l}.ln2"])
            gu = rstd(x)[:, None] * (u2 @ p[f"{l}.gate_up_w"].T)
            gu = gu.reshape(T, I // 64, 2, 64)
            g, up = gu[:, :, 0, :].reshape(T, I), gu[:, :, 1, :].reshape(T, I)
            act = bf16(torch.nn.functional.silu(g) * up)
            x = x + act @ p[f"{l}.down_w"].T
        uF = bf16(x * p["final_norm"])
        W = p["embed"] if c["tie_embeddings"] else p["lm_head"]
        logits = rstd(x)[:, None] * (uF @ W.T)
        return torch.log_softmax(logits, -1)[torch.arange(T), tgt]

    def is_reinforce(self, trajs, m, clamp, granularity):
        """J and its gradient (into .grad); weights stop-gradient."""
        J = torch.zeros((), dtype=self.dtype)
        lps = []
        for t in trajs:
            lp = self.logprobs(t["tokens"])
            lps.append(lp.detach().cpu().numpy())
            lb = t["loss_begin"] - 1
            mu = torch.tensor(t["behavior_logprobs"][1:], dtype=self.dtype)
            adv = torch.tensor(t["advantages"][1:], dtype=self.dtype)
            sl = slice(lb, None)
            if granularity == "sequence":
                w = torch.clamp(torch.exp(lp[sl].sum() - mu[sl].sum()), max=clamp).detach()
            else:
                w = torch.clamp(torch.exp(lp[sl] - mu[sl]), max=clamp).detach()
            J = J + (w * adv[sl] * lp[sl]).sum() / m
        J.backward()
        return float(J.detach()), lps
