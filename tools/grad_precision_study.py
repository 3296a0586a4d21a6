"""Which bf16 rounding point of the device backward dominates the gradient
error?  CPU study (float64 torch): the reference gradient of
tests/torch_decoder_ref.py against the same model with the device backward's
rounding points switched on one at a time (custom autograd functions that
round what the device rounds).  Prints rel-L2 and the worst per-tensor
relative error for each switch.

  python tools/grad_precision_study.py [--layers 2] [--hidden 128] ...
"""
from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.decoder_oracle import bf16_bits_to_f32, layout  # noqa: E402

torch.set_default_dtype(torch.float64)


def bf(x):
    return x.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def split(x):
    """hi + lo bf16 pair, as the device would carry it."""
    h = bf(x)
    return h + bf(x - h)


class Opts:
    dy = "exact"       # dY of the linear layers: exact | bf16 | split
    xn = "exact"       # rstd * xg operand of dW: exact | bf16 | fold (rstd folded into dY)
    gu = "exact"       # saved gate/up for the SwiGLU backward: exact | bf16
    dgu = "exact"      # SwiGLU backward output: exact | bf16 | split
    dlogits = "exact"  # exact | bf16 | split
    attn = "exact"     # dO, P, dS in the attention backward: exact | bf16 | split


O = Opts()


def rnd(x, mode):
    if mode == "bf16":
        return bf(x)
    if mode == "split":
        return split(x)
    return x


def st(x):  # straight-through bf16 rounding of forward values (device rounding points)
    return x + (bf(x) - x).detach()


class NormLinear(torch.autograd.Function):
    """y = rstd[:, None] * (u @ W^T) (+ b); u = bf16(x * gain) is exact bf16."""

    @staticmethod
    def forward(ctx, u, W, rstd):
        ctx.save_for_backward(u, W, rstd)
        return rstd[:, None] * (u @ W.T)

    @staticmethod
    def backward(ctx, g):
        u, W, rstd = ctx.saved_tensors
        dy = rnd(g, O.dy)
        du = rstd[:, None] * (dy @ W)        # dzw (device: fp32 out of the GEMM, then rmsnorm bwd)
        if O.xn == "bf16":
            dW = dy.T @ bf(rstd[:, None] * u)
        elif O.xn == "fold":
            dW = rnd(g * rstd[:, None], O.dy).T @ u
        else:
            dW = dy.T @ (rstd[:, None] * u)
        drstd = ((dy @ W) * u).sum(-1)
        return du, dW, drstd


class Linear(torch.autograd.Function):
    """y = a @ W^T, a exact bf16 (attention output, SwiGLU activation)."""

    @staticmethod
    def forward(ctx, a, W):
        ctx.save_for_backward(a, W)
        return a @ W.T

    @staticmethod
    def backward(ctx, g):
        a, W = ctx.saved_tensors
        dy = rnd(g, O.dy)
        return dy @ W, dy.T @ a


class SwiGLU(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, up):
        ctx.save_for_backward(g, up)
        return torch.nn.functional.silu(g) * up

    @staticmethod
    def backward(ctx, d):
        g, up = ctx.saved_tensors
        if O.gu == "bf16":
            g, up = bf(g), bf(up)
        s = torch.sigmoid(g)
        dg = d * up * s * (1 + g * (1 - s))
        dup = d * g * s
        return rnd(dg, O.dgu), rnd(dup, O.dgu)


class Attn(torch.autograd.Function):
    """softmax(q k^T * scale, causal) v per head; q, k, v exact bf16."""

    @staticmethod
    def forward(ctx, q, k, v, scale):
        T = q.shape[0]
        mask = torch.ones(T, T, dtype=torch.bool).tril()
        s = torch.einsum("thd,shd->hts", q * scale, k).masked_fill(~mask, float("-inf"))
        p = torch.softmax(s, -1)
        o = torch.einsum("hts,shd->thd", p, v)
        ctx.save_for_backward(q, k, v, p, o)
        ctx.scale = scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, p, o = ctx.saved_tensors
        m = O.attn
        do_ = rnd(do, m)
        D = (do * o).sum(-1)                              # [t, h]
        dv = torch.einsum("hts,thd->shd", rnd(p, m), do_)
        dp = torch.einsum("thd,shd->hts", do_, v)
        ds = p * (dp - D.T[:, :, None])
        dsr = rnd(ds, m)
        dq = ctx.scale * torch.einsum("hts,shd->thd", dsr, k)
        dk = ctx.scale * torch.einsum("hts,thd->shd", dsr, q)
        return dq, dk, dv, None


class Logits(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z):
        return z

    @staticmethod
    def backward(ctx, g):
        return rnd(g, O.dlogits)


def make_weights(cfg, seed, scale):
    off, total = layout(cfg)
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal(total) * scale).astype(np.float32)
    for name, (o, n) in off.items():
        if name.endswith("ln1") or name.endswith("ln2") or name == "final_norm":
            w[o:o + n] = 1.0 + 0.1 * rng.standard_normal(n)
    u = (w.view(np.uint32) >> 16).astype(np.uint16)
    return off, total, u


def grads(cfg, u16, trajs, clamp=5.0):
    off, total = layout(cfg)
    H, I, V = cfg["hidden"], cfg["intermediate"], cfg["vocab_size"]
    nq, nkv, hd = cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
    G, half = nq // nkv, hd // 2
    shapes = {"embed": (V, H), "final_norm": (H,)}
    for l in range(cfg["layers"]):
        qkv = (nq + 2 * nkv) * hd
        shapes.update({f"{l}.ln1": (H,), f"{l}.qkv_w": (qkv, H), f"{l}.qkv_b": (qkv,),
                       f"{l}.o_w": (H, nq * hd), f"{l}.ln2": (H,),
                       f"{l}.gate_up_w": (2 * I, H), f"{l}.down_w": (H, I)})
    p = {}
    for name, shape in shapes.items():
        o, n = off[name]
        p[name] = torch.tensor(bf16_bits_to_f32(u16[o:o + n]).astype(np.float64)).reshape(shape).requires_grad_(True)
    J = torch.zeros(())
    for t in trajs:
        tokens = t["tokens"]
        inp, tgt = torch.tensor(tokens[:-1]), torch.tensor(tokens[1:])
        T = len(inp)
        x = p["embed"][inp]
        pos = torch.arange(T, dtype=torch.float64)
        inv = cfg["rope_theta"] ** (-2.0 * torch.arange(half, dtype=torch.float64) / hd)
        ang = pos[:, None] * inv
        cos = ang.cos().float().double()
        sin = ang.sin().float().double()

        def rope(z):
            z1, z2 = z[..., :half], z[..., half:]
            return torch.cat([z1 * cos[:, None] - z2 * sin[:, None], z2 * cos[:, None] + z1 * sin[:, None]], -1)

        def rstd(z):
            return 1.0 / torch.sqrt((z * z).mean(-1) + cfg["rms_eps"])

        scale = float(np.float32(1.0 / math.sqrt(hd)))
        for l in range(cfg["layers"]):
            u = st(x * p[f"{l}.ln1"])
            qkv = NormLinear.apply(u, p[f"{l}.qkv_w"], rstd(x)) + p[f"{l}.qkv_b"]
            q = st(rope(qkv[:, :nq * hd].reshape(T, nq, hd)))
            k = st(rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(T, nkv, hd)))
            v = st(qkv[:, (nq + nkv) * hd:].reshape(T, nkv, hd))
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            o = st(Attn.apply(q, k, v, scale).reshape(T, nq * hd))
            x = x + Linear.apply(o, p[f"{l}.o_w"])
            u2 = st(x * p[f"{l}.ln2"])
            gu = NormLinear.apply(u2, p[f"{l}.gate_up_w"], rstd(x)).reshape(T, I // 64, 2, 64)
            g, up = gu[:, :, 0, :].reshape(T, I), gu[:, :, 1, :].reshape(T, I)
            act = st(SwiGLU.apply(g, up))
            x = x + Linear.apply(act, p[f"{l}.down_w"])
        uF = st(x * p["final_norm"])
        W = p["embed"] if cfg["tie_embeddings"] else p["lm_head"]
        logits = Logits.apply(NormLinear.apply(uF, W, rstd(x)))
        lp = torch.log_softmax(logits, -1)[torch.arange(T), tgt]
        lb = t["loss_begin"] - 1
        w = min(clamp, 1.0)
        J = J + (w * torch.tensor(t["advantages"][1:])[lb:] * lp[lb:]).sum() / len(trajs)
    J.backward()
    g = np.zeros(total)
    for name, t in p.items():
        o, n = off[name]
        g[o:o + n] += t.grad.numpy().ravel()
    return g, off


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--hidden", type=int, default=128)
    ap.add_argument("--inter", type=int, default=512)
    ap.add_argument("--vocab", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--kv", type=int, default=1)
    ap.add_argument("--hd", type=int, default=64)
    ap.add_argument("--scale", type=float, default=0.03)
    ap.add_argument("--seqs", type=int, default=4)
    ap.add_argument("--len", type=int, default=48)
    a = ap.parse_args()
    cfg = dict(hidden=a.hidden, intermediate=a.inter, vocab_size=a.vocab, layers=a.layers, q_heads=a.heads,
               kv_heads=a.kv, head_dim=a.hd, tie_embeddings=True, rope_theta=10000.0, rms_eps=1e-6)
    off, total, u16 = make_weights(cfg, 1, a.scale)
    rng = np.random.default_rng(2)
    trajs = []
    for i in range(a.seqs):
        toks = rng.integers(0, a.vocab, size=a.len).tolist()
        trajs.append(dict(tokens=toks, loss_begin=2, advantages=[float(rng.standard_normal())] * a.len))
    ref, _ = grads(cfg, u16, trajs)

    def run(label, **kw):
        for k, v in vars(Opts).items():
            if not k.startswith("_"):
                setattr(O, k, v)
        for k, v in kw.items():
            setattr(O, k, v)
        g, _ = grads(cfg, u16, trajs)
        rel = np.linalg.norm(g - ref) / np.linalg.norm(ref)
        worst = 0.0
        wname = ""
        for name, (o, n) in off.items():
            b = ref[o:o + n]
            if np.linalg.norm(b) > 0:
                e = np.linalg.norm(g[o:o + n] - b) / np.linalg.norm(b)
                if e > worst:
                    worst, wname = e, name
        print(f"{label:40s} relL2 {rel:.2e}  worst {worst:.2e} ({wname})", flush=True)

    run("device today (all bf16)", dy="bf16", xn="bf16", gu="bf16", dgu="bf16", dlogits="bf16", attn="bf16")
    run("dy bf16 only", dy="bf16")
    run("xn bf16 only", xn="bf16")
    run("gu bf16 only", gu="bf16")
    run("dgu bf16 only", dgu="bf16")
    run("dlogits bf16 only", dlogits="bf16")
    run("attn bf16 only", attn="bf16")
    run("all split, xn fold, gu exact", dy="split", xn="fold", dgu="split", dlogits="split", attn="split")
    run("all split, xn fold, gu bf16", dy="split", xn="fold", gu="bf16", dgu="split", dlogits="split",
        attn="split")
    run("split except dlogits bf16", dy="split", xn="fold", dgu="split", dlogits="bf16", attn="split")
    run("split except attn bf16", dy="split", xn="fold", dgu="split", dlogits="split", attn="bf16")


if __name__ == "__main__":
    main()
