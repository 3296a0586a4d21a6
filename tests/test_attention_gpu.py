"""The multi-kernel round's single-query paged GQA attention
(decoder.cu attention_kernel, srl_kernel_attention_decode) against a plain
PyTorch fp32 reference of the same op on random bf16 q / K / V: contexts
inside one 32-key tile, across tiles, across the 512-key splits (the merged
split partials), page boundaries, GQA group sizes of the 0.5B (7), 1.5B (6)
and 7B (7, hd 128) shapes.  Bar: 5e-3 relative to the output scale -- the
output is bf16 (half an ulp is 2^-9 of the value); P enters the P.V product
as hi + lo bf16 halves, so the fp32 result itself is far closer."""
import math

import numpy as np
import pytest
import torch

from paper_2509_19128_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nq,nkv,hd", [(14, 2, 64), (12, 2, 128), (28, 4, 128)])
def test_attention_decode_matches_torch(cuda, nq, nkv, hd):
    g = torch.Generator(device="cuda").manual_seed(nq * hd)
    ctxs = [1, 5, 31, 32, 33, 64, 65, 511, 512, 513, 1100, 2047, 4100]
    rows = len(ctxs)
    pps = (max(ctxs) + 63) // 64
    # pages of slot r are a permutation (paged, not contiguous)
    perm = torch.randperm(rows * pps, generator=g, device="cuda").to(torch.int32)
    bt = perm.view(rows, pps).contiguous()
    kc = (torch.randn(rows * pps, nkv, 64, hd, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    vc = torch.randn(rows * pps, nkv, 64, hd, generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn(rows, nq, hd, generator=g, device="cuda").to(torch.bfloat16)
    slot = torch.arange(rows, dtype=torch.int32, device="cuda")
    pos = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32, device="cuda")
    out = torch.empty(rows, nq, hd, dtype=torch.bfloat16, device="cuda")
    _lib.call("srl_kernel_attention_decode", q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(), pps,
              slot.data_ptr(), pos.data_ptr(), rows, nq, nkv, hd, max(ctxs), out.data_ptr(), None)
    torch.cuda.synchronize()
    G = nq // nkv
    scale = 1.0 / math.sqrt(hd)
    for r, c in enumerate(ctxs):
        pages = bt[r, :(c + 63) // 64].long()
        K = kc[pages].float().permute(1, 0, 2, 3).reshape(nkv, -1, hd)[:, :c]  # [nkv, c, hd]
        V = vc[pages].float().permute(1, 0, 2, 3).reshape(nkv, -1, hd)[:, :c]
        qh = q[r].float().view(nkv, G, hd)
        s = torch.einsum("kgd,kcd->kgc", qh, K) * scale
        p = torch.softmax(s, -1)
        ref = torch.einsum("kgc,kcd->kgd", p, V).reshape(nq, hd)
        err = (out[r].float() - ref).abs().max().item()
        # the output is bf16: half an ulp is 2^-9 relative, up to 3.9e-3 for values in [1, 2)
        assert err <= 5e-3 * max(1.0, ref.abs().max().item()), (c, err)


@pytest.mark.parametrize("nq,nkv,hd", [(14, 2, 64), (12, 2, 128), (28, 4, 128)])
def test_attention_prefill_matches_torch(cuda, nq, nkv, hd):
    """attn_fwd_mma (srl_kernel_attention_prefill): the trainer's forward and a
    prefill round's prompt rows.  Ragged packed segments (1 .. 321 rows, inside
    one 64-key block, on and across block / page boundaries), segments that
    start mid-context (seg_pos0: recompute chunks, continued prompts), paged
    caches, GQA groups of 7 / 6 / 7.  O against fp32 at the bf16 output bar,
    the split output (hi + lo, the trainer's precise mode) at 1e-4, lse 1e-4."""
    g = torch.Generator(device="cuda").manual_seed(7 * nq + hd)
    lens = [1, 5, 63, 64, 65, 200, 321, 130]
    pos0 = [0, 0, 0, 10, 64, 0, 0, 700]
    n = len(lens)
    pps = (max(p + l for p, l in zip(pos0, lens)) + 63) // 64
    slots = [(3 * y + 1) % n for y in range(n)]  # segments read other slots' pages
    perm = torch.randperm(n * pps, generator=g, device="cuda").to(torch.int32)
    bt = perm.view(n, pps).contiguous()
    kc = (torch.randn(n * pps, nkv, 64, hd, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    vc = torch.randn(n * pps, nkv, 64, hd, generator=g, device="cuda").to(torch.bfloat16)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int32)
    T = int(sum(lens))
    q = torch.randn(T, nq, hd, generator=g, device="cuda").to(torch.bfloat16)
    d_start = torch.tensor(starts, dtype=torch.int32, device="cuda")
    d_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    d_pos0 = torch.tensor(pos0, dtype=torch.int32, device="cuda")
    d_slot = torch.tensor(slots, dtype=torch.int32, device="cuda")
    W = nq * hd
    out = torch.full((T, 2 * W), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((T, nq), float("nan"), dtype=torch.float32, device="cuda")
    _lib.call("srl_kernel_attention_prefill", q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(), pps,
              d_start.data_ptr(), d_len.data_ptr(), d_pos0.data_ptr(), d_slot.data_ptr(), n, max(lens), nq, nkv, hd,
              out.data_ptr(), lse.data_ptr(), W, None)
    torch.cuda.synchronize()
    G = nq // nkv
    scale = 1.0 / math.sqrt(hd)
    for y in range(n):
        L, p0, s0 = lens[y], pos0[y], int(starts[y])
        ctx = p0 + L
        pages = bt[slots[y], :(ctx + 63) // 64].long()
        K = kc[pages].float().permute(1, 0, 2, 3).reshape(nkv, -1, hd)[:, :ctx]  # [nkv, ctx, hd]
        V = vc[pages].float().permute(1, 0, 2, 3).reshape(nkv, -1, hd)[:, :ctx]
        qh = q[s0:s0 + L].float().view(L, nkv, G, hd)
        s = torch.einsum("tkgd,kcd->tkgc", qh, K) * scale
        keypos = torch.arange(ctx, device="cuda")
        qpos = p0 + torch.arange(L, device="cuda")
        s = s.masked_fill((keypos[None, :] > qpos[:, None])[:, None, None, :], float("-inf"))
        ref_lse = torch.logsumexp(s, -1).reshape(L, nq)
        ref = torch.einsum("tkgc,kcd->tkgd", torch.softmax(s, -1), V).reshape(L, W)
        hi = out[s0:s0 + L, :W].float()
        lo = out[s0:s0 + L, W:].float()
        sc = max(1.0, ref.abs().max().item())
        assert (hi - ref).abs().max().item() <= 5e-3 * sc, y
        assert (hi + lo - ref).abs().max().item() <= 1e-4 * sc, y
        assert torch.allclose(lse[s0:s0 + L], ref_lse, rtol=1e-4, atol=1e-4), y
