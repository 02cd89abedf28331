"""Pins for oracle/vit.py (the MLLM ViT encoder + merger):
  * LayerNorm, erf-GELU: torch's library routines (F.layer_norm, F.gelu) with
    autograd in fp64, forward and backward;
  * bidirectional attention: torch SDPA (is_causal=False) with autograd, fp64;
  * QuickGELU: closed-form values (0 at 0, slope 1/2 at 0, x for large x,
    0 for very negative x) and central finite differences;
  * the whole encoder + merger and the MLLM step: central finite
    differences on micro shapes (every parameter tensor probed);
  * ViT-600M shape: 0.63B parameters + merger;
  * HuggingFace Qwen2-VL's vision tower in fp64 (its fp32 RoPE evaluated in
    fp64): output and parameter gradients.
"""
import dataclasses

import numpy as np
import pytest
import torch

import stp_inputs as si
from oracle import model as om
from oracle import vit as ov

MICRO_V = ov.VitCfg(hidden=8, n_layers=2, n_heads=2, head_dim=4, mlp=12, patch_dim=6, merge=4, out_hidden=8)
MICRO_LM = si.ModelCfg(vocab=16, hidden=8, n_layers=2, n_q_heads=2, n_kv_heads=1, head_dim=4, ffn=16, seq=6)


def _vparams(c, seed=0, std=0.3):
    rng = np.random.default_rng(seed)
    out = {}
    for k, sh in ov.vit_param_shapes(c).items():
        if k.endswith("_g"):
            out[k] = 1.0 + 0.1 * rng.standard_normal(sh)
        else:
            out[k] = std * rng.standard_normal(sh)
    return out


def test_layernorm_matches_torch():
    rng = np.random.default_rng(1)
    x, g, b, dy = rng.standard_normal((7, 13)), rng.standard_normal(13), rng.standard_normal(13), \
        rng.standard_normal((7, 13))
    y, xh, r = ov.layernorm_fwd(x, g, b, 1e-6)
    tx, tg, tb = (torch.tensor(a, requires_grad=True) for a in (x, g, b))
    ty = torch.nn.functional.layer_norm(tx, (13,), tg, tb, eps=1e-6)
    ty.backward(torch.tensor(dy))
    assert np.allclose(y, ty.detach().numpy(), atol=1e-12)
    dx, dg, db = ov.layernorm_bwd(dy, xh, g, r)
    assert np.allclose(dx, tx.grad.numpy(), atol=1e-11)
    assert np.allclose(dg, tg.grad.numpy(), atol=1e-11) and np.allclose(db, tb.grad.numpy(), atol=1e-12)


def test_gelu_matches_torch():
    x = np.linspace(-6, 6, 101)
    dy = np.cos(x)
    tx = torch.tensor(x, requires_grad=True)
    ty = torch.nn.functional.gelu(tx)
    ty.backward(torch.tensor(dy))
    assert np.allclose(ov.gelu_fwd(x), ty.detach().numpy(), atol=1e-14)
    assert np.allclose(ov.gelu_bwd(dy, x), tx.grad.numpy(), atol=1e-13)


def test_quickgelu_closed_forms_and_fd():
    assert ov.qgelu_fwd(np.array(0.0)) == 0.0
    assert ov.qgelu_bwd(np.array(1.0), np.array(0.0)) == pytest.approx(0.5)
    assert ov.qgelu_fwd(np.array(40.0)) == pytest.approx(40.0, rel=1e-12)
    assert abs(ov.qgelu_fwd(np.array(-40.0))) < 1e-25
    x = np.linspace(-4, 4, 41)
    e = 1e-6
    fd = (ov.qgelu_fwd(x + e) - ov.qgelu_fwd(x - e)) / (2 * e)
    assert np.allclose(ov.qgelu_bwd(np.ones_like(x), x), fd, atol=1e-8)


def test_bidirectional_attention_matches_sdpa():
    rng = np.random.default_rng(2)
    s, n, d = 9, 3, 5
    q, k, v, do = (rng.standard_normal((s, n, d)) for _ in range(4))
    o, _ = ov.attention_full_fwd(q, k, v)
    tq, tk, tv = (torch.tensor(a.transpose(1, 0, 2), requires_grad=True) for a in (q, k, v))
    to = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=False)
    to.backward(torch.tensor(do.transpose(1, 0, 2)))
    assert np.allclose(o, to.detach().numpy().transpose(1, 0, 2), atol=1e-12)
    dq, dk, dv = ov.attention_full_bwd(do, q, k, v, o)
    for got, ref in ((dq, tq), (dk, tk), (dv, tv)):
        assert np.allclose(got, ref.grad.numpy().transpose(1, 0, 2), atol=1e-11)


def _fd_check(loss_fn, params, grads, names, rng, eps=1e-5, probes=4):
    for name in names:
        a = params[name]
        for _ in range(probes):
            idx = tuple(rng.integers(0, sz) for sz in a.shape)
            old = a[idx]
            a[idx] = old + eps
            lp = loss_fn()
            a[idx] = old - eps
            lm = loss_fn()
            a[idx] = old
            fd = (lp - lm) / (2 * eps)
            g = grads[name][idx]
            assert abs(fd - g) <= 1e-6 * max(1.0, abs(fd)) + 1e-9, (name, idx, fd, g)


def test_vit_encoder_finite_differences():
    c = MICRO_V
    PV = _vparams(c)
    rng = np.random.default_rng(3)
    patches = rng.standard_normal((8, c.patch_dim))             # a 2 x 4 patch grid
    w = rng.standard_normal((8 // c.merge, c.out_hidden))   # loss = sum(w * out)
    out, cache = ov.vit_forward(PV, c, patches, (2, 4))
    gv = {k: np.zeros_like(v) for k, v in PV.items()}
    ov.vit_backward(PV, c, cache, w, gv)
    loss = lambda: float(np.sum(w * ov.vit_forward(PV, c, patches, (2, 4))[0]))  # noqa: E731
    _fd_check(loss, PV, gv, list(PV), np.random.default_rng(4))


def test_mllm_step_finite_differences():
    c, cfg = MICRO_V, MICRO_LM
    PV = _vparams(c, seed=5)
    P = si.make_params(cfg, seed=6, std=0.3, parity=True)
    rng = np.random.default_rng(7)
    m = 2
    patches = rng.standard_normal((m, 8, c.patch_dim))        # 8 patches -> 2 image rows
    n_text = cfg.seq - 8 // c.merge
    tokens = rng.integers(0, cfg.vocab, (m, n_text)).astype(np.int32)
    targets = rng.integers(0, cfg.vocab, (m, cfg.seq)).astype(np.int32)
    L, G, GV = ov.mllm_forward_backward(PV, c, P, cfg, patches, (2, 4), tokens, targets)

    def loss():
        return ov.mllm_forward_backward(PV, c, P, cfg, patches, (2, 4), tokens, targets)[0]
    _fd_check(loss, PV, GV, ["vit.patch", "vit.0.wqkv", "vit.1.b1", "vit.1.ln2_b", "merger.w1", "merger.b2",
                             "merger.ln_g"], np.random.default_rng(8), probes=3)
    _fd_check(loss, P, G, ["embed", "layers.0.wq", "layers.1.wd", "lm_head"], np.random.default_rng(9), probes=3)


def test_mllm_reduces_to_the_lm_when_rows_are_text():
    """With the image rows replaced by embedding rows of known tokens, the
    MLLM LM pass is the plain LM step (forward_mb with x0 == E[tok])."""
    cfg = MICRO_LM
    P = si.make_params(cfg, seed=10, std=0.3, parity=True)
    rng = np.random.default_rng(11)
    tok = rng.integers(0, cfg.vocab, (1, cfg.seq)).astype(np.int32)
    tgt = rng.integers(0, cfg.vocab, (1, cfg.seq)).astype(np.int32)
    l_ref, g_ref = om.forward_backward(P, cfg, tok, tgt)
    loss, cache = om.forward_mb(P, cfg, None, tgt[0], x0=P["embed"][tok[0]])
    g = {k: np.zeros_like(v) for k, v in P.items()}
    dx0 = om.backward_mb(P, cfg, cache, g, 1.0 / cfg.seq, embed_tok=tok[0])
    assert loss == pytest.approx(l_ref, rel=1e-14)
    for k in P:
        assert np.allclose(g[k], g_ref[k], atol=1e-14), k
    assert dx0.shape == (cfg.seq, cfg.hidden)


def test_vit600m_parameter_count():
    n = sum(int(np.prod(s)) for s in ov.vit_param_shapes(ov.VIT_600M).values())
    merger = 4 * 1280 * 4 * 1280 + 4 * 1280 + 3584 * 4 * 1280 + 3584 + 2 * 1280
    assert abs((n - merger) / 1e9 - 0.63) < 0.01


def test_vit_matches_hf_qwen2vl_vision_tower():
    """Qwen2-VL's vision tower (HuggingFace transformers, fp64, autograd) on a
    tiny config: patch embed, 2-D RoPE, LayerNorm blocks with QuickGELU MLPs,
    bidirectional attention, 2x2 merger; output and every parameter gradient
    of sum(w * out)."""
    from transformers.models.qwen2_vl.configuration_qwen2_vl import Qwen2VLVisionConfig
    from transformers.models.qwen2_vl.modeling_qwen2_vl import Qwen2VisionTransformerPretrainedModel
    hv, heads, mlp_ratio, out_h, ps, tps = 16, 2, 3, 12, 2, 2
    vc = Qwen2VLVisionConfig(depth=2, embed_dim=hv, num_heads=heads, mlp_ratio=mlp_ratio, hidden_size=out_h,
                             in_channels=3, patch_size=ps, temporal_patch_size=tps, spatial_merge_size=2,
                             hidden_act="quick_gelu")
    vc._attn_implementation = "sdpa"  # the eager path runs softmax in fp32
    import transformers.models.qwen2_vl.modeling_qwen2_vl as hfm

    def rope64(q, k, cos, sin):  # HF evaluates the vision RoPE in fp32; the pin runs it in fp64
        cos, sin = cos.unsqueeze(-2), sin.unsqueeze(-2)
        return q * cos + hfm.rotate_half(q) * sin, k * cos + hfm.rotate_half(k) * sin
    orig = hfm.apply_rotary_pos_emb_vision
    hfm.apply_rotary_pos_emb_vision = rope64
    torch.manual_seed(0)
    hf = Qwen2VisionTransformerPretrainedModel(vc).double()
    rot = hf.rotary_pos_emb
    rot.inv_freq = 1.0 / (rot.theta ** (torch.arange(0, rot.dim, 2, dtype=torch.float64) / rot.dim))
    for prm in hf.parameters():
        torch.nn.init.normal_(prm, std=0.3)
    c = ov.VitCfg(hidden=hv, n_layers=2, n_heads=heads, head_dim=hv // heads, mlp=hv * mlp_ratio,
                  patch_dim=3 * tps * ps * ps, merge=4, out_hidden=out_h)
    PV = {"vit.patch": hf.patch_embed.proj.weight.detach().reshape(hv, -1).numpy().copy()}
    for l, b in enumerate(hf.blocks):
        p = f"vit.{l}."
        PV.update({p + "ln1_g": b.norm1.weight, p + "ln1_b": b.norm1.bias, p + "wqkv": b.attn.qkv.weight,
                   p + "bqkv": b.attn.qkv.bias, p + "wo": b.attn.proj.weight, p + "bo": b.attn.proj.bias,
                   p + "ln2_g": b.norm2.weight, p + "ln2_b": b.norm2.bias, p + "w1": b.mlp.fc1.weight,
                   p + "b1": b.mlp.fc1.bias, p + "w2": b.mlp.fc2.weight, p + "b2": b.mlp.fc2.bias})
    PV.update({"merger.ln_g": hf.merger.ln_q.weight, "merger.ln_b": hf.merger.ln_q.bias,
               "merger.w1": hf.merger.mlp[0].weight, "merger.b1": hf.merger.mlp[0].bias,
               "merger.w2": hf.merger.mlp[2].weight, "merger.b2": hf.merger.mlp[2].bias})
    PV = {k: (v.detach().numpy().copy() if isinstance(v, torch.Tensor) else v) for k, v in PV.items()}
    gh, gw = 4, 6
    rng = np.random.default_rng(12)
    patches = rng.standard_normal((gh * gw, c.patch_dim))
    w = rng.standard_normal((gh * gw // 4, out_h))
    out = hf(torch.tensor(patches), grid_thw=torch.tensor([[1, gh, gw]]))
    out = getattr(out, "pooler_output", None) if not isinstance(out, torch.Tensor) else out
    if out is None or out.shape[0] != gh * gw // 4:
        out = hf(torch.tensor(patches), grid_thw=torch.tensor([[1, gh, gw]]))
        out = out.last_hidden_state if out.last_hidden_state.shape[0] == gh * gw // 4 else out.pooler_output
    (out * torch.tensor(w)).sum().backward()
    hfm.apply_rotary_pos_emb_vision = orig
    mine, cache = ov.vit_forward(PV, c, patches, (gh, gw))
    assert np.allclose(mine, out.detach().numpy(), rtol=0, atol=1e-11)
    gv = {k: np.zeros_like(v) for k, v in PV.items()}
    ov.vit_backward(PV, c, cache, w, gv)
    ref = {"vit.patch": hf.patch_embed.proj.weight.grad.reshape(hv, -1)}
    for l, b in enumerate(hf.blocks):
        p = f"vit.{l}."
        ref.update({p + "ln1_g": b.norm1.weight.grad, p + "wqkv": b.attn.qkv.weight.grad,
                    p + "bqkv": b.attn.qkv.bias.grad, p + "bo": b.attn.proj.bias.grad, p + "w1": b.mlp.fc1.weight.grad,
                    p + "b2": b.mlp.fc2.bias.grad, p + "ln2_b": b.norm2.bias.grad})
    ref.update({"merger.w1": hf.merger.mlp[0].weight.grad, "merger.ln_g": hf.merger.ln_q.weight.grad})
    for k, r in ref.items():
        assert np.allclose(gv[k], r.numpy(), rtol=0, atol=1e-10), k
