"""Unsharded fp64 ViT encoder + 2x2 patch merger of the MLLM workload (the
heterogeneous first virtual stage, §5 P:L171 "the ViT encoder is
assigned to the first virtual stage on device 0"; Table 3 P:L231-263;
SURVEY §8f-f1, cfg5) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
Plain numpy fp64, one library primitive (matmul) per step, hand-derived
backward.

Model (Qwen2-VL vision tower as the paper uses it, readings V1-V4 in
DESIGN.md):
  X = patches @ Wpe^T                                  (patch embed, no bias)
  per layer: Xn = LN(X; g1, b1); [Q|K|V] = Xn Wqkv^T + bqkv (heads of d)
             Q, K <- 2-D rotate-half RoPE (angles [h pos * inv | w pos * inv],
                     inv_j = 10000^(-2j/(d/2)), patches in 2x2 merge-window
                     order, as Qwen2-VL's rot_pos_emb)
             O_i = softmax(Q_i K_i^T / sqrt(d)) V_i    (bidirectional)
             X += O Wo^T + bo
             Xn2 = LN(X; g2, b2); X += qgelu(Xn2 W1^T + b1) W2^T + b2
             qgelu(x) = x * sigmoid(1.702 x)
  merger:    Y = LN(X; gq, bq) -> rows of 4 consecutive patches [s/4, 4 hv]
             out = gelu(Y M1^T + c1) M2^T + c2         ([s/4, h_lm]; gelu = erf)
The MLLM step (mllm_forward_backward): the LM input sequence is
[merger output (image tokens) | E[text tokens]], run through the LM of
oracle/model.py; loss over every position's next-token target (reading V4).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict

import numpy as np

from . import model as om

Params = Dict[str, np.ndarray]


@dataclasses.dataclass(frozen=True)
class VitCfg:
    hidden: int = 1280
    n_layers: int = 32
    n_heads: int = 16
    head_dim: int = 80
    mlp: int = 5120
    patch_dim: int = 1176        # 3 * 2 * 14 * 14
    merge: int = 4               # 2 x 2 spatial merge
    out_hidden: int = 3584       # LM hidden
    ln_eps: float = 1e-6


VIT_600M = VitCfg()


def vit_param_shapes(c: VitCfg) -> Dict[str, tuple]:
    hv, m4 = c.hidden, c.merge * c.hidden
    sh = {"vit.patch": (hv, c.patch_dim)}
    for l in range(c.n_layers):
        p = f"vit.{l}."
        sh.update({p + "ln1_g": (hv,), p + "ln1_b": (hv,), p + "wqkv": (3 * hv, hv), p + "bqkv": (3 * hv,),
                   p + "wo": (hv, hv), p + "bo": (hv,), p + "ln2_g": (hv,), p + "ln2_b": (hv,),
                   p + "w1": (c.mlp, hv), p + "b1": (c.mlp,), p + "w2": (hv, c.mlp), p + "b2": (hv,)})
    sh.update({"merger.ln_g": (hv,), "merger.ln_b": (hv,), "merger.w1": (m4, m4), "merger.b1": (m4,),
               "merger.w2": (c.out_hidden, m4), "merger.b2": (c.out_hidden,)})
    return sh


# ---------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------

def layernorm_fwd(x, g, b, eps):
    """y = g * (x - mu) * r + b, r = (var + eps)^(-1/2).  Returns (y, xhat, r)."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    r = 1.0 / np.sqrt((xc * xc).mean(axis=-1, keepdims=True) + eps)
    xhat = xc * r
    return xhat * g + b, xhat, r


def layernorm_bwd(dy, xhat, g, r):
    """dx = r * (g dy - mean(g dy) - xhat * mean(g dy * xhat)); dg = sum dy xhat; db = sum dy."""
    gdy = g * dy
    dx = r * (gdy - gdy.mean(axis=-1, keepdims=True) - xhat * (gdy * xhat).mean(axis=-1, keepdims=True))
    return dx, np.sum(dy * xhat, axis=0), np.sum(dy, axis=0)


def qgelu_fwd(x):
    return x * om.sigmoid(1.702 * x)


def qgelu_bwd(dy, x):
    """d/dx [x sig(a x)] = sig(a x) + a x sig(a x)(1 - sig(a x)), a = 1.702."""
    s = om.sigmoid(1.702 * x)
    return dy * (s + 1.702 * x * s * (1.0 - s))


_erf = np.vectorize(math.erf)


def gelu_fwd(x):
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def gelu_bwd(dy, x):
    """d/dx [x Phi(x)] = Phi(x) + x phi(x)."""
    cdf = 0.5 * (1.0 + _erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return dy * (cdf + x * pdf)


def attention_full_fwd(q, k, v):
    """Bidirectional multi-head attention, q, k, v [s, n, d].  Returns O and
    the row LSE [n, s]."""
    s, n, d = q.shape
    scale = 1.0 / np.sqrt(d)
    o = np.empty_like(q)
    lse = np.empty((n, s))
    for i in range(n):
        S = (q[:, i, :] @ k[:, i, :].T) * scale
        m = S.max(axis=-1, keepdims=True)
        E = np.exp(S - m)
        Z = E.sum(axis=-1, keepdims=True)
        o[:, i, :] = (E / Z) @ v[:, i, :]
        lse[i] = (m + np.log(Z))[:, 0]
    return o, lse


def attention_full_bwd(do, q, k, v, o):
    """Same formulas as the causal case without the mask."""
    s, n, d = q.shape
    scale = 1.0 / np.sqrt(d)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for i in range(n):
        S = (q[:, i, :] @ k[:, i, :].T) * scale
        P = np.exp(S - S.max(axis=-1, keepdims=True))
        P /= P.sum(axis=-1, keepdims=True)
        dv[:, i, :] = P.T @ do[:, i, :]
        dP = do[:, i, :] @ v[:, i, :].T
        D = np.sum(do[:, i, :] * o[:, i, :], axis=-1, keepdims=True)
        dS = P * (dP - D)
        dq[:, i, :] = (dS @ k[:, i, :]) * scale
        dk[:, i, :] = (dS.T @ q[:, i, :]) * scale
    return dq, dk, dv


def vit_positions(gh: int, gw: int, merge_side: int = 2):
    """(h, w) grid position of every patch, patches listed in merge-window
    order (each 2x2 window's 4 patches consecutive, windows row-major)."""
    hp = np.arange(gh)[:, None].repeat(gw, 1).reshape(gh // merge_side, merge_side, gw // merge_side, merge_side)
    wp = np.arange(gw)[None, :].repeat(gh, 0).reshape(gh // merge_side, merge_side, gw // merge_side, merge_side)
    return hp.transpose(0, 2, 1, 3).reshape(-1), wp.transpose(0, 2, 1, 3).reshape(-1)


def vit_rope_tables(gh: int, gw: int, d: int, theta: float = 10000.0, merge_side: int = 2):
    """cos / sin [s, d] of the 2-D vision RoPE: angle row = [h * inv | w * inv]
    (d/2 angles, inv_j = theta^(-2j/(d/2)), j < d/4), duplicated for
    rotate-half."""
    hp, wp = vit_positions(gh, gw, merge_side)
    inv = 1.0 / theta ** (np.arange(0, d // 2, 2, dtype=np.float64) / (d // 2))
    ang = np.concatenate([hp[:, None] * inv[None, :], wp[:, None] * inv[None, :]], axis=1)
    emb = np.concatenate([ang, ang], axis=1)
    return np.cos(emb), np.sin(emb)


# ---------------------------------------------------------------------------
# encoder + merger
# ---------------------------------------------------------------------------

def vit_forward(PV: Params, c: VitCfg, patches, grid):
    """patches [s, patch_dim] in merge-window order of a grid = (gh, gw)
    image (s = gh * gw) -> ([s/merge, out_hidden], cache)."""
    s, hv, n, d = patches.shape[0], c.hidden, c.n_heads, c.head_dim
    assert s == grid[0] * grid[1]
    cos, sin = vit_rope_tables(grid[0], grid[1], d)
    x = patches @ PV["vit.patch"].T
    layers = []
    for l in range(c.n_layers):
        p = f"vit.{l}."
        xn, xh1, r1 = layernorm_fwd(x, PV[p + "ln1_g"], PV[p + "ln1_b"], c.ln_eps)
        qkv = xn @ PV[p + "wqkv"].T + PV[p + "bqkv"]
        q = om.rope_fwd(qkv[:, :hv].reshape(s, n, d), cos, sin)
        k = om.rope_fwd(qkv[:, hv:2 * hv].reshape(s, n, d), cos, sin)
        v = qkv[:, 2 * hv:].reshape(s, n, d)
        o, _ = attention_full_fwd(q, k, v)
        o2 = o.reshape(s, hv)
        x1 = x + o2 @ PV[p + "wo"].T + PV[p + "bo"]
        xn2, xh2, r2 = layernorm_fwd(x1, PV[p + "ln2_g"], PV[p + "ln2_b"], c.ln_eps)
        a = xn2 @ PV[p + "w1"].T + PV[p + "b1"]
        hh = qgelu_fwd(a)
        x2 = x1 + hh @ PV[p + "w2"].T + PV[p + "b2"]
        layers.append(dict(xn=xn, xh1=xh1, r1=r1, q=q, k=k, v=v, o=o, o2=o2, xn2=xn2, xh2=xh2, r2=r2, a=a, hh=hh))
        x = x2
    y, xhq, rq = layernorm_fwd(x, PV["merger.ln_g"], PV["merger.ln_b"], c.ln_eps)
    ym = y.reshape(s // c.merge, c.merge * hv)
    z = ym @ PV["merger.w1"].T + PV["merger.b1"]
    gz = gelu_fwd(z)
    out = gz @ PV["merger.w2"].T + PV["merger.b2"]
    cache = dict(patches=patches, cos=cos, sin=sin, layers=layers, xhq=xhq, rq=rq, ym=ym, z=z, gz=gz)
    return out, cache


def vit_backward(PV: Params, c: VitCfg, cache, dout, grads: Params):
    """Accumulate d/dparams of sum(dout * out) into grads."""
    s, hv, n, d = cache["patches"].shape[0], c.hidden, c.n_heads, c.head_dim
    grads["merger.w2"] += dout.T @ cache["gz"]
    grads["merger.b2"] += dout.sum(axis=0)
    dgz = dout @ PV["merger.w2"]
    dz = gelu_bwd(dgz, cache["z"])
    grads["merger.w1"] += dz.T @ cache["ym"]
    grads["merger.b1"] += dz.sum(axis=0)
    dy = (dz @ PV["merger.w1"]).reshape(s, hv)
    dx, dg, db = layernorm_bwd(dy, cache["xhq"], PV["merger.ln_g"], cache["rq"])
    grads["merger.ln_g"] += dg
    grads["merger.ln_b"] += db
    for l in reversed(range(c.n_layers)):
        p = f"vit.{l}."
        L = cache["layers"][l]
        grads[p + "w2"] += dx.T @ L["hh"]
        grads[p + "b2"] += dx.sum(axis=0)
        da = qgelu_bwd(dx @ PV[p + "w2"], L["a"])
        grads[p + "w1"] += da.T @ L["xn2"]
        grads[p + "b1"] += da.sum(axis=0)
        dxn2 = da @ PV[p + "w1"]
        dx1n, dg2, db2 = layernorm_bwd(dxn2, L["xh2"], PV[p + "ln2_g"], L["r2"])
        grads[p + "ln2_g"] += dg2
        grads[p + "ln2_b"] += db2
        dx1 = dx + dx1n
        grads[p + "wo"] += dx1.T @ L["o2"]
        grads[p + "bo"] += dx1.sum(axis=0)
        do = (dx1 @ PV[p + "wo"]).reshape(s, n, d)
        dq, dk, dv = attention_full_bwd(do, L["q"], L["k"], L["v"], L["o"])
        dq = om.rope_bwd(dq, cache["cos"], cache["sin"])
        dk = om.rope_bwd(dk, cache["cos"], cache["sin"])
        dqkv = np.concatenate([dq.reshape(s, hv), dk.reshape(s, hv), dv.reshape(s, hv)], axis=1)
        grads[p + "wqkv"] += dqkv.T @ L["xn"]
        grads[p + "bqkv"] += dqkv.sum(axis=0)
        dxn = dqkv @ PV[p + "wqkv"]
        dx0n, dg1, db1 = layernorm_bwd(dxn, L["xh1"], PV[p + "ln1_g"], L["r1"])
        grads[p + "ln1_g"] += dg1
        grads[p + "ln1_b"] += db1
        dx = dx1 + dx0n
    grads["vit.patch"] += dx.T @ cache["patches"]


def mllm_forward_backward(PV: Params, vcfg: VitCfg, P: Params, cfg, patches, grid, tokens, targets):
    """MLLM step over m microbatches: microbatch b's LM input is
    [vit(patches[b]) (n_img = s_v / merge rows) | E[tokens[b]]] (cfg.seq rows
    in total); L = mean_b mean_i CE; returns (L, LM grads, ViT grads)."""
    m = tokens.shape[0]
    s = cfg.seq
    grads = {k: np.zeros_like(v) for k, v in P.items()}
    gv = {k: np.zeros_like(v) for k, v in PV.items()}
    losses = []
    for b in range(m):
        img, vc = vit_forward(PV, vcfg, patches[b], grid)
        n_img = img.shape[0]
        x0 = np.concatenate([img, P["embed"][tokens[b]]], axis=0)
        assert x0.shape[0] == s
        loss_b, cache = om.forward_mb(P, cfg, None, targets[b], x0=x0)
        losses.append(loss_b)
        dx0 = om.backward_mb(P, cfg, cache, grads, 1.0 / (s * m), embed_tok=tokens[b], embed_row0=n_img)
        vit_backward(PV, vcfg, vc, dx0[:n_img], gv)
    return float(np.mean(losses)), grads, gv
