"""Pins for oracle/model.py — each check fixes the oracle against something
other than itself (SURVEY §8c.4 "Model math"):

* an independent library implementation of the same model (HuggingFace
  transformers Qwen2ForCausalLM, fp64, torch autograd for the gradients);
* library routines for sub-steps (torch SDPA for causal GQA attention,
  torch rms_norm);
* central finite differences of the oracle's own forward (pins the
  hand-derived backward to the forward);
* closed forms / special cases: W_lm = 0 => loss = ln V exactly; s = 1 =>
  attention output equals V; gradient linearity over microbatches;
* the sharded (TP/SP) emulation equals the unsharded result (PAPER.md P:L73
  "preserves computational equivalence"), for t in {1, 2, 4}.
"""
import dataclasses
import math

import numpy as np
import pytest
import torch

import stp_inputs as si
from oracle import schedule as sc
from oracle import model as om

MICRO = si.ModelCfg(vocab=16, hidden=8, n_layers=2, n_q_heads=2, n_kv_heads=1,
                    head_dim=4, ffn=16, seq=4)


def _hf_model(cfg, P):
    from transformers import Qwen2Config, Qwen2ForCausalLM
    c = Qwen2Config(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                    num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_q_heads,
                    num_key_value_heads=cfg.n_kv_heads, rms_norm_eps=cfg.rms_eps,
                    rope_theta=cfg.rope_theta, tie_word_embeddings=False,
                    max_position_embeddings=max(64, cfg.seq), attn_implementation="sdpa")
    torch.manual_seed(0)
    m = Qwen2ForCausalLM(c).double()
    # HF evaluates the RoPE angles in float32 by design; evaluate the same HF
    # formula (inv_freq = 1/base^(arange(0,d,2)/d), emb = cat(f, f)) in fp64 so
    # the comparison is not limited by float32 cos/sin.
    rot = m.model.rotary_emb
    inv64 = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, dtype=torch.float64) / cfg.head_dim))

    def rot_fwd64(x, position_ids):
        f = position_ids[:, :, None].double() * inv64[None, None, :]
        emb = torch.cat((f, f), dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)
    rot.forward = rot_fwd64
    # Likewise HF's Qwen2RMSNorm upcasts to float32 (a downcast for fp64
    # inputs); rebind each norm to the same formula without the cast.
    from transformers.models.qwen2 import modeling_qwen2 as mq
    for mod in m.modules():
        if isinstance(mod, mq.Qwen2RMSNorm):
            def norm64(x, mod=mod):
                var = x.pow(2).mean(-1, keepdim=True)
                return mod.weight * (x * torch.rsqrt(var + mod.variance_epsilon))
            mod.forward = norm64
    names = {"model.embed_tokens.weight": "embed", "model.norm.weight": "final_ln",
             "lm_head.weight": "lm_head"}
    for l in range(cfg.n_layers):
        a, b = f"model.layers.{l}.", f"layers.{l}."
        names.update({a + "self_attn.q_proj.weight": b + "wq", a + "self_attn.q_proj.bias": b + "bq",
                      a + "self_attn.k_proj.weight": b + "wk", a + "self_attn.k_proj.bias": b + "bk",
                      a + "self_attn.v_proj.weight": b + "wv", a + "self_attn.v_proj.bias": b + "bv",
                      a + "self_attn.o_proj.weight": b + "wo", a + "mlp.gate_proj.weight": b + "wg",
                      a + "mlp.up_proj.weight": b + "wu", a + "mlp.down_proj.weight": b + "wd",
                      a + "input_layernorm.weight": b + "ln1",
                      a + "post_attention_layernorm.weight": b + "ln2"})
    with torch.no_grad():
        for n, p in m.named_parameters():
            p.copy_(torch.from_numpy(P[names[n]]))
    return m, names


@pytest.mark.parametrize("cfg", [dataclasses.replace(si.TINY, n_layers=2), MICRO])
def test_oracle_matches_hf_qwen2_loss_and_grads(cfg):
    P = si.make_params(cfg, seed=3, std=0.2, parity=True)
    toks, tgts = si.make_tokens(cfg, 2, seed=5)
    loss, grads = om.forward_backward(P, cfg, toks, tgts)
    m, names = _hf_model(cfg, P)
    losses = []
    for b in range(toks.shape[0]):
        out = m(input_ids=torch.from_numpy(toks[b:b + 1].astype(np.int64)))
        lg = out.logits[0]
        losses.append(torch.nn.functional.cross_entropy(lg, torch.from_numpy(tgts[b].astype(np.int64))))
    L = torch.stack(losses).mean()
    L.backward()
    assert abs(loss - L.item()) <= 1e-12 * max(1.0, abs(loss))
    for n, p in m.named_parameters():
        ref = p.grad.numpy()
        got = grads[names[n]]
        err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
        assert err < 1e-10, (n, err)


def test_attention_matches_torch_sdpa_causal_gqa():
    rng = np.random.default_rng(0)
    s, nq, nkv, d = 37, 6, 2, 16
    q = rng.standard_normal((s, nq, d))
    k = rng.standard_normal((s, nkv, d))
    v = rng.standard_normal((s, nkv, d))
    o, lse = om.attention_fwd(q, k, v)
    tq, tk, tv = (torch.from_numpy(a).transpose(0, 1)[None] for a in (q, k, v))
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True, enable_gqa=True)
    assert np.abs(o - ref[0].transpose(0, 1).numpy()).max() < 1e-12
    # LSE via torch.logsumexp over explicitly masked scores
    S = torch.einsum("hsd,htd->hst", tq[0], tk[0].repeat_interleave(nq // nkv, 0)) / math.sqrt(d)
    S = S.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool), 1), -float("inf"))
    assert np.abs(lse - torch.logsumexp(S, -1).numpy()).max() < 1e-12
    # backward against autograd through SDPA
    tq2, tk2, tv2 = (a.clone().requires_grad_(True) for a in (tq, tk, tv))
    out = torch.nn.functional.scaled_dot_product_attention(tq2, tk2, tv2, is_causal=True, enable_gqa=True)
    do = rng.standard_normal((s, nq, d))
    out.backward(torch.from_numpy(do).transpose(0, 1)[None])
    dq, dk, dv = om.attention_bwd(do, q, k, v, o)
    for got, ref in ((dq, tq2), (dk, tk2), (dv, tv2)):
        assert np.abs(got - ref.grad[0].transpose(0, 1).numpy()).max() < 1e-11


def test_rmsnorm_matches_torch():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((9, 24))
    g = 1 + 0.1 * rng.standard_normal(24)
    y, r = om.rmsnorm_fwd(x, g, 1e-6)
    tx = torch.from_numpy(x).requires_grad_(True)
    tg = torch.from_numpy(g).requires_grad_(True)
    ty = torch.nn.functional.rms_norm(tx, (24,), tg, 1e-6)
    assert np.abs(y - ty.detach().numpy()).max() < 1e-13
    dy = rng.standard_normal((9, 24))
    ty.backward(torch.from_numpy(dy))
    dx, dg = om.rmsnorm_bwd(dy, x, g, r)
    assert np.abs(dx - tx.grad.numpy()).max() < 1e-12
    assert np.abs(dg - tg.grad.numpy()).max() < 1e-12


def test_finite_difference_gradients_micro():
    cfg = MICRO
    P = si.make_params(cfg, seed=11, std=0.3, parity=True)
    toks, tgts = si.make_tokens(cfg, 2, seed=2)
    _, grads = om.forward_backward(P, cfg, toks, tgts)
    rng = np.random.default_rng(0)
    eps = 1e-5
    for name, arr in P.items():
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in arr.shape)
            if name == "embed":  # pick a row that is actually used
                idx = (int(toks[0, 0]),) + idx[1:]
            old = arr[idx]
            arr[idx] = old + eps
            lp = om.loss_only(P, cfg, toks, tgts)
            arr[idx] = old - eps
            lm = om.loss_only(P, cfg, toks, tgts)
            arr[idx] = old
            fd = (lp - lm) / (2 * eps)
            an = grads[name][idx]
            assert abs(fd - an) <= 1e-6 * max(abs(fd), 1e-3), (name, idx, fd, an)


def test_zero_lm_head_gives_log_vocab():
    cfg = MICRO
    P = si.make_params(cfg, seed=1, parity=True)
    P["lm_head"][:] = 0.0
    toks, tgts = si.make_tokens(cfg, 3)
    assert om.loss_only(P, cfg, toks, tgts) == pytest.approx(math.log(cfg.vocab), abs=1e-15)


def test_single_token_attention_is_value():
    rng = np.random.default_rng(4)
    q = rng.standard_normal((1, 4, 8))
    k = rng.standard_normal((1, 2, 8))
    v = rng.standard_normal((1, 2, 8))
    o, _ = om.attention_fwd(q, k, v)
    assert np.array_equal(o, v[:, [0, 0, 1, 1], :])


def test_gradient_linearity_over_microbatches():
    cfg = MICRO
    P = si.make_params(cfg, seed=2, std=0.2, parity=True)
    toks, tgts = si.make_tokens(cfg, 3, seed=9)
    L, G = om.forward_backward(P, cfg, toks, tgts)
    parts = [om.forward_backward(P, cfg, toks[b:b + 1], tgts[b:b + 1]) for b in range(3)]
    assert L == pytest.approx(np.mean([p[0] for p in parts]), abs=1e-14)
    for k in G:
        assert np.allclose(G[k], np.mean([p[1][k] for p in parts], axis=0), rtol=0, atol=1e-15)


def _unshard_check(cfg, t, P, G, Gs):
    for r in range(t):
        ref = om.shard_params(G, cfg, t, r)
        for k, v in Gs[r].items():
            if k.endswith(("ln1", "ln2")) or k == "final_ln":
                continue
            assert np.abs(v - ref[k]).max() <= 1e-12 * max(1.0, np.abs(ref[k]).max()), (r, k)
    for k in G:
        if k.endswith(("ln1", "ln2")) or k == "final_ln":
            tot = sum(Gs[r][k] for r in range(t))
            assert np.abs(tot - G[k]).max() <= 1e-12, k


@pytest.mark.parametrize("t", [1, 2, 4])
def test_sharded_equals_unsharded(t):
    cfg = dataclasses.replace(si.TINY, n_layers=2, seq=16, n_q_heads=4, n_kv_heads=4 if t == 4 else 2)
    P = si.make_params(cfg, seed=7, std=0.1, parity=True)
    toks, tgts = si.make_tokens(cfg, 2, seed=8)
    L, G = om.forward_backward(P, cfg, toks, tgts)
    Ls, Gs = om.forward_backward_sp(P, cfg, toks, tgts, t)
    assert abs(L - Ls) <= 1e-12
    _unshard_check(cfg, t, P, G, Gs)


def test_qwen2_7b_param_count():
    shapes = si.param_shapes(si.QWEN2_7B)
    n = sum(int(np.prod(s)) for s in shapes.values())
    assert abs(n / 1e9 - 7.62) < 0.01      # Qwen2-7B: 7.62B


def test_paper_layer_split():
    # SPEC S:L61-63 worked examples of the "last stage two layers short" rule
    assert sc.paper_layer_split(30, 8) == [4, 4, 4, 4, 4, 4, 4, 2]
    assert sc.paper_layer_split(46, 16) == [3] * 15 + [1]
    with pytest.raises(ValueError):
        sc.paper_layer_split(8, 8)
    assert sc.paper_layer_split(28, 4) == [8, 8, 7, 5]
