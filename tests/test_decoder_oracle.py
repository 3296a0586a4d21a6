"""Pins the decoder restatements to an independent implementation.

The reference has no transformer, so the builder's CPU
decoder oracle (oracle/decoder_oracle.py) and the fp64 autograd restatement
used for trainer gradients (tests/torch_decoder_ref.py) are pinned here:

* forward: with the device's bf16 rounding points switched off (exact=True)
  both equal transformers' Qwen2ForCausalLM (5.5.0, in float64, sdpa
  attention: eager softmaxes in fp32) on random Qwen2-shaped weights in our flat layout -- RoPE
  convention, GQA head mapping, the 64-row gate/up interleave, QKV bias, RMSNorm
  placement, tied / untied LM head;
* backward: the autograd gradient of the IS-REINFORCE objective equals central
  finite differences of the same objective computed by the oracle, on 60
  random parameters (the recipe of test_rl_math.cpp:57-90: step 1e-5,
  relative tolerance 1e-4);
* the device rounding points are a small, documented perturbation of the
  exact forward (bf16 activations: within 2e-2 absolute log-prob here).
"""
import math

import numpy as np
import pytest
import torch

from oracle.decoder_oracle import DecoderOracle, bf16_bits_to_f32, layout

CFGS = [
    dict(name="g2", vocab_size=100, hidden=64, layers=2, q_heads=4, kv_heads=2, head_dim=16,
         intermediate=128, tie_embeddings=True, bos_token=0, max_positions=64, rope_theta=10000.0,
         rms_eps=1e-6),
    dict(name="g3-untied", vocab_size=70, hidden=96, layers=3, q_heads=6, kv_heads=2, head_dim=16,
         intermediate=192, tie_embeddings=False, bos_token=1, max_positions=64,
         rope_theta=1000000.0, rms_eps=1e-5),
]


def random_flat(cfg, seed, scale=0.08):
    off, total = layout(cfg)
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal(total).astype(np.float32) * scale).view(np.uint32)
    w = ((w + 0x7FFF + ((w >> 16) & 1)) >> 16).astype(np.uint16)  # round to bf16
    for name, (o, n) in off.items():  # gains near 1
        if name.endswith("ln1") or name.endswith("ln2") or name == "final_norm":
            g = (1.0 + 0.1 * rng.standard_normal(n)).astype(np.float32).view(np.uint32)
            w[o:o + n] = (g >> 16).astype(np.uint16)
    return w


def hf_model(cfg, flat_u16):
    from transformers import Qwen2Config, Qwen2ForCausalLM

    H, I, nq, nkv, hd = cfg["hidden"], cfg["intermediate"], cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"]
    c = Qwen2Config(vocab_size=cfg["vocab_size"], hidden_size=H, intermediate_size=I,
                    num_hidden_layers=cfg["layers"], num_attention_heads=nq, num_key_value_heads=nkv,
                    rms_norm_eps=cfg["rms_eps"], max_position_embeddings=cfg["max_positions"],
                    tie_word_embeddings=cfg["tie_embeddings"], rope_theta=cfg["rope_theta"],
                    attn_implementation="sdpa")
    assert H // nq == hd
    m = Qwen2ForCausalLM(c).to(torch.float64).eval()
    off, _ = layout(cfg)

    def t(name, shape):
        o, n = off[name]
        return torch.tensor(bf16_bits_to_f32(flat_u16[o:o + n]).astype(np.float64)).reshape(shape)

    sd = {"model.embed_tokens.weight": t("embed", (cfg["vocab_size"], H)),
          "model.norm.weight": t("final_norm", (H,))}
    for l in range(cfg["layers"]):
        qkv_w = t(f"{l}.qkv_w", ((nq + 2 * nkv) * hd, H))
        qkv_b = t(f"{l}.qkv_b", ((nq + 2 * nkv) * hd,))
        a, b = nq * hd, (nq + nkv) * hd
        gu = t(f"{l}.gate_up_w", (2 * I, H)).reshape(I // 64, 2, 64, H)  # 64-row interleave
        p = f"model.layers.{l}."
        sd.update({p + "self_attn.q_proj.weight": qkv_w[:a], p + "self_attn.q_proj.bias": qkv_b[:a],
                   p + "self_attn.k_proj.weight": qkv_w[a:b], p + "self_attn.k_proj.bias": qkv_b[a:b],
                   p + "self_attn.v_proj.weight": qkv_w[b:], p + "self_attn.v_proj.bias": qkv_b[b:],
                   p + "self_attn.o_proj.weight": t(f"{l}.o_w", (H, nq * hd)),
                   p + "mlp.gate_proj.weight": gu[:, 0].reshape(I, H),
                   p + "mlp.up_proj.weight": gu[:, 1].reshape(I, H),
                   p + "mlp.down_proj.weight": t(f"{l}.down_w", (H, I)),
                   p + "input_layernorm.weight": t(f"{l}.ln1", (H,)),
                   p + "post_attention_layernorm.weight": t(f"{l}.ln2", (H,))})
    if not cfg["tie_embeddings"]:
        sd["lm_head.weight"] = t("lm_head", (cfg["vocab_size"], H))
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    assert all(k == "lm_head.weight" for k in missing) and (cfg["tie_embeddings"] or not missing)
    if cfg["tie_embeddings"]:
        assert torch.equal(m.lm_head.weight, sd["model.embed_tokens.weight"])
    _lift_to_fp64(m, cfg)
    return m


def _lift_to_fp64(m, cfg):
    """transformers computes RMSNorm and the RoPE tables in fp32 even inside a
    float64 model (Qwen2RMSNorm.forward, Qwen2RotaryEmbedding.forward); lift
    those two to fp64 (same formulas) so the comparison is exact to fp64."""
    import types

    from transformers.models.qwen2.modeling_qwen2 import Qwen2RMSNorm

    def norm_fwd(self, x):
        return self.weight * (x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.variance_epsilon))

    for mod in m.modules():
        if isinstance(mod, Qwen2RMSNorm):
            mod.forward = types.MethodType(norm_fwd, mod)
    hd = cfg["head_dim"]
    inv = cfg["rope_theta"] ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)

    def rope_fwd(self, x, position_ids):
        freqs = position_ids[..., None].to(torch.float64) * inv
        emb = torch.cat((freqs, freqs), dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)

    m.model.rotary_emb.forward = types.MethodType(rope_fwd, m.model.rotary_emb)


def hf_logits(m, tokens):
    with torch.no_grad():
        return m(torch.tensor([tokens])).logits[0].numpy()


@pytest.mark.parametrize("cfg", CFGS, ids=[c["name"] for c in CFGS])
def test_oracle_exact_equals_transformers_qwen2(cfg):
    w = random_flat(cfg, 7)
    m = hf_model(cfg, w)
    rng = np.random.default_rng(1)
    tokens = [cfg["bos_token"]] + rng.integers(0, cfg["vocab_size"], size=23).tolist()
    ref = hf_logits(m, tokens)
    orc = DecoderOracle(cfg, w, exact=True)
    got = orc.prefill(orc.new_cache(), tokens)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-10)
    # incremental decode over a prefilled cache == the full forward
    c2 = orc.new_cache()
    orc.prefill(c2, tokens[:10])
    steps = [orc.step([c2], [t], [len(c2["tokens"])])[0] for t in tokens[10:]]
    np.testing.assert_allclose(np.stack(steps), ref[10:], rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("cfg", CFGS, ids=[c["name"] for c in CFGS])
def test_device_rounding_is_a_small_perturbation(cfg):
    w = random_flat(cfg, 8)
    rng = np.random.default_rng(2)
    tokens = [cfg["bos_token"]] + rng.integers(0, cfg["vocab_size"], size=15).tolist()
    exact = DecoderOracle(cfg, w, exact=True)
    dev = DecoderOracle(cfg, w)
    le = DecoderOracle.log_softmax(exact.prefill(exact.new_cache(), tokens))
    ld = DecoderOracle.log_softmax(dev.prefill(dev.new_cache(), tokens))
    assert np.max(np.abs(le - ld)) < 2e-2
    assert np.max(np.abs(le - ld)) > 0  # the rounding points are really there


@pytest.mark.parametrize("cfg", CFGS, ids=[c["name"] for c in CFGS])
def test_torch_reference_exact_equals_transformers(cfg):
    from tests.torch_decoder_ref import TorchDecoder

    w = random_flat(cfg, 9)
    m = hf_model(cfg, w)
    rng = np.random.default_rng(3)
    tokens = [cfg["bos_token"]] + rng.integers(0, cfg["vocab_size"], size=17).tolist()
    lp_hf = torch.log_softmax(torch.tensor(hf_logits(m, tokens)), -1).numpy()
    lp_hf = lp_hf[np.arange(len(tokens) - 1), tokens[1:]]
    td = TorchDecoder(cfg, w, exact=True)
    np.testing.assert_allclose(td.logprobs(tokens).detach().numpy(), lp_hf, rtol=1e-10, atol=1e-11)


def _objective(lps, trajs, m, clamp, granularity, weights_from=None):
    """J of rl_math.cpp:211-276 (stop-gradient IS weight) from per-token log-probs."""
    J = 0.0
    for lp, t, wf in zip(lps, trajs, weights_from if weights_from is not None else lps):
        lb = t["loss_begin"] - 1
        mu = np.asarray(t["behavior_logprobs"][1:])[lb:]
        adv = np.asarray(t["advantages"][1:])[lb:]
        if granularity == "sequence":
            w = min(clamp, math.exp(wf[lb:].sum() - mu.sum()))
        else:
            w = np.minimum(clamp, np.exp(wf[lb:] - mu))
        J += float((w * adv * lp[lb:]).sum()) / m
    return J


@pytest.mark.parametrize("granularity", ["sequence", "per_token"])
def test_autograd_gradient_equals_finite_differences(granularity):
    """test_rl_math.cpp:57-90 recipe on the decoder: the fp64 autograd gradient
    (the reference for the device trainer's gradient) against central finite
    differences of the oracle's objective, 60 random parameters."""
    from tests.torch_decoder_ref import TorchDecoder

    cfg = CFGS[0]
    w = random_flat(cfg, 10)
    rng = np.random.default_rng(4)
    trajs = []
    for i in range(3):
        n = int(rng.integers(8, 14))
        toks = [cfg["bos_token"]] + rng.integers(0, cfg["vocab_size"], size=n - 1).tolist()
        trajs.append(dict(tokens=toks, loss_begin=3,
                          behavior_logprobs=(-math.log(cfg["vocab_size"]) + 0.3 * rng.standard_normal(n)).tolist(),
                          advantages=rng.standard_normal(n).tolist()))
    m, clamp = 3, 5.0
    td = TorchDecoder(cfg, w, exact=True)
    J, _ = td.is_reinforce(trajs, m, clamp, granularity)
    grad = td.flat_grad()

    off, total = layout(cfg)
    flat = bf16_bits_to_f32(w).astype(np.float64)
    base_lps = None

    def oracle_lps(flat64):
        orc = DecoderOracle.from_flat64(cfg, flat64)
        return [orc.sequence_logprobs(t["tokens"][1:]) for t in trajs]

    base_lps = oracle_lps(flat)
    assert abs(_objective(base_lps, trajs, m, clamp, granularity) - J) < 1e-10
    idx = rng.choice(total, size=60, replace=False)
    idx = [i for i in idx if any(o <= i < o + n for o, n in off.values())]
    h = 1e-5
    for i in idx:
        fp, fm = flat.copy(), flat.copy()
        fp[i] += h
        fm[i] -= h
        # stop-gradient on the IS weight: the weight stays at its base value
        jp = _objective(oracle_lps(fp), trajs, m, clamp, granularity, weights_from=base_lps)
        jm = _objective(oracle_lps(fm), trajs, m, clamp, granularity, weights_from=base_lps)
        fd = (jp - jm) / (2 * h)
        assert abs(fd - grad[i]) <= 1e-4 * max(1e-3, abs(fd), abs(grad[i])), (i, fd, grad[i])
