"""Unsharded fp64 Qwen2-style decoder: forward, hand-derived backward, and
microbatch gradient accumulation — the plain definition the STP step must
reach ("preserves computational equivalence").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy fp64; one
library primitive (matmul) per step; no blocking, fusion or reordering.

Model (readings Q9, Q11, Q16, Q19):
  X0 = E[tok]
  per layer: Xn = rms(X)*g1; Q,K,V = Xn W^T + b; RoPE(Q,K) (rotate-half);
             O_i = softmax(Q_i K_g^T / sqrt(d) + causal) V_g; X += O Wo^T;
             Xn2 = rms(X)*g2; X += (silu(Xn2 Wg^T) * (Xn2 Wu^T)) Wd^T
  logits = rms(X)*gf W_lm^T;  loss_b = mean_i CE(logits_i, target_i)
  L = mean_b loss_b;  result = (L, dL/dparams)

The sharded emulation at the bottom follows the sequence-parallel form of
PAPER.md Eq. 1-2 under reading Q10: activations between units
are row shards [s/t, h]; AG = concatenation of rows; RS = sum over ranks then
row-block r; each rank adds its own residual shard after the RS (Eq. 1's
detach(X)/t summed over t ranks, without the /t rounding).
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

Params = Dict[str, np.ndarray]


# ---------------------------------------------------------------------------
# building blocks (each: SURVEY §8c.1 "Backward the oracle implements by hand")
# ---------------------------------------------------------------------------

def rmsnorm_fwd(x, g, eps):
    """y = g * x * r, r = (mean_h x^2 + eps)^(-1/2).  Returns (y, r[...,1])."""
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * g, r


def rmsnorm_bwd(dy, x, g, r):
    """dx = r*(g*dy) - x*r^3*mean_h((g*dy)*x);  dg = sum_rows dy*x*r."""
    gdy = g * dy
    dx = r * gdy - x * (r ** 3) * np.mean(gdy * x, axis=-1, keepdims=True)
    dg = np.sum(dy * x * r, axis=0)
    return dx, dg


def rope_tables(s, d, theta, pos0=0):
    """cos/sin [s, d] for rotate-half RoPE: angle_i = pos * theta^(-2i/d)."""
    inv = 1.0 / theta ** (np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.arange(pos0, pos0 + s, dtype=np.float64)[:, None] * inv[None, :]
    emb = np.concatenate([ang, ang], axis=-1)
    return np.cos(emb), np.sin(emb)


def rotate_half(x):
    d2 = x.shape[-1] // 2
    return np.concatenate([-x[..., d2:], x[..., :d2]], axis=-1)


def rope_fwd(x, cos, sin):
    """x [s, n, d] -> x*cos + rot(x)*sin."""
    return x * cos[:, None, :] + rotate_half(x) * sin[:, None, :]


def rope_bwd(dy, cos, sin):
    """dx = dy*cos - rot(dy*sin)  (rot^T = -rot)."""
    return dy * cos[:, None, :] - rotate_half(dy * sin[:, None, :])


def attention_fwd(q, k, v):
    """Causal GQA attention. q [s, nq, d]; k, v [s, nkv, d].
    Returns O [s, nq, d] and the row log-sum-exp LSE [nq, s] (natural log,
    of the scaled, masked scores)."""
    s, nq, d = q.shape
    nkv = k.shape[1]
    grp = nq // nkv
    scale = 1.0 / np.sqrt(d)
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    o = np.empty_like(q)
    lse = np.empty((nq, s))
    for i in range(nq):
        g = i // grp
        S = (q[:, i, :] @ k[:, g, :].T) * scale
        S[mask] = -np.inf
        m = S.max(axis=-1, keepdims=True)
        E = np.exp(S - m)
        Z = E.sum(axis=-1, keepdims=True)
        P = E / Z
        o[:, i, :] = P @ v[:, g, :]
        lse[i] = (m + np.log(Z))[:, 0]
    return o, lse


def attention_bwd(do, q, k, v, o):
    """dV = P^T dO; dP = dO V^T; dS = P*(dP - rowsum(dO*O)); dQ = dS K/sqrt(d);
    dK = dS^T Q/sqrt(d); GQA: dK, dV summed over the group's query heads."""
    s, nq, d = q.shape
    nkv = k.shape[1]
    grp = nq // nkv
    scale = 1.0 / np.sqrt(d)
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for i in range(nq):
        g = i // grp
        S = (q[:, i, :] @ k[:, g, :].T) * scale
        S[mask] = -np.inf
        S = S - S.max(axis=-1, keepdims=True)
        P = np.exp(S)
        P /= P.sum(axis=-1, keepdims=True)
        dv[:, g, :] += P.T @ do[:, i, :]
        dP = do[:, i, :] @ v[:, g, :].T
        D = np.sum(do[:, i, :] * o[:, i, :], axis=-1, keepdims=True)
        dS = P * (dP - D)
        dq[:, i, :] = (dS @ k[:, g, :]) * scale
        dk[:, g, :] += (dS.T @ q[:, i, :]) * scale
    return dq, dk, dv


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def swiglu_fwd(G, U):
    return G * sigmoid(G) * U


def swiglu_bwd(dH, G, U):
    """dU = dH*silu(G); dG = dH*U*sig(G)*(1 + G*(1-sig(G)))."""
    sg = sigmoid(G)
    dU = dH * G * sg
    dG = dH * U * sg * (1.0 + G * (1.0 - sg))
    return dG, dU


def cross_entropy(logits, targets):
    """Per-token CE and the row statistics.  logits [s, V]."""
    m = logits.max(axis=-1, keepdims=True)
    Z = np.exp(logits - m).sum(axis=-1, keepdims=True)
    lse = (m + np.log(Z))[:, 0]
    tl = logits[np.arange(logits.shape[0]), targets]
    return lse - tl, lse


def cross_entropy_bwd(logits, targets, lse, scale):
    """d(scale * sum_i loss_i)/dlogits = scale * (softmax - onehot)."""
    p = np.exp(logits - lse[:, None])
    p[np.arange(logits.shape[0]), targets] -= 1.0
    return p * scale


# ---------------------------------------------------------------------------
# unsharded model
# ---------------------------------------------------------------------------

def _heads(x, n, d):
    return x.reshape(x.shape[0], n, d)


def forward_mb(P: Params, cfg, tok, tgt, x0=None):
    """One microbatch forward.  Returns (loss_b, cache).  x0 (optional)
    replaces the embedding lookup as the layer-0 input (the MLLM sequence of
    image + text rows, oracle/vit.py)."""
    x = P["embed"][tok] if x0 is None else x0
    s, d = x.shape[0], cfg.head_dim
    cos, sin = rope_tables(s, d, cfg.rope_theta)
    layers = []
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        c = {"x": x}
        xn, r1 = rmsnorm_fwd(x, P[p + "ln1"], cfg.rms_eps)
        q = xn @ P[p + "wq"].T
        k = xn @ P[p + "wk"].T
        v = xn @ P[p + "wv"].T
        if cfg.qkv_bias:
            q = q + P[p + "bq"]
            k = k + P[p + "bk"]
            v = v + P[p + "bv"]
        qr = rope_fwd(_heads(q, cfg.n_q_heads, d), cos, sin)
        kr = rope_fwd(_heads(k, cfg.n_kv_heads, d), cos, sin)
        vh = _heads(v, cfg.n_kv_heads, d)
        o, lse = attention_fwd(qr, kr, vh)
        o2 = o.reshape(s, -1)
        x1 = x + o2 @ P[p + "wo"].T
        xn2, r2 = rmsnorm_fwd(x1, P[p + "ln2"], cfg.rms_eps)
        G = xn2 @ P[p + "wg"].T
        U = xn2 @ P[p + "wu"].T
        H = swiglu_fwd(G, U)
        x2 = x1 + H @ P[p + "wd"].T
        c.update(xn=xn, r1=r1, qr=qr, kr=kr, vh=vh, o=o, lse=lse, o2=o2,
                 x1=x1, xn2=xn2, r2=r2, G=G, U=U, H=H)
        layers.append(c)
        x = x2
    xf, rf = rmsnorm_fwd(x, P["final_ln"], cfg.rms_eps)
    logits = xf @ P["lm_head"].T
    per_tok, lse_ce = cross_entropy(logits, tgt)
    cache = dict(tok=tok, tgt=tgt, cos=cos, sin=sin, layers=layers, x_last=x,
                 xf=xf, rf=rf, logits=logits, lse_ce=lse_ce)
    return float(per_tok.mean()), cache


def backward_mb(P: Params, cfg, cache, grads: Params, scale: float, embed_tok=None, embed_row0=0):
    """Accumulate scale * d(sum_i loss_i)/dparams into grads.
    With scale = 1/(s*m) this is d(L)/dparams for L = mean_b mean_i loss.
    Returns dL/dX0; the embedding gradient is scattered from rows
    embed_row0.. for embed_tok (default: all rows, cache["tok"])."""
    d = cfg.head_dim
    s = cache["x_last"].shape[0]
    cos, sin = cache["cos"], cache["sin"]
    dlogits = cross_entropy_bwd(cache["logits"], cache["tgt"], cache["lse_ce"], scale)
    grads["lm_head"] += dlogits.T @ cache["xf"]
    dxf = dlogits @ P["lm_head"]
    dx, dg = rmsnorm_bwd(dxf, cache["x_last"], P["final_ln"], cache["rf"])
    grads["final_ln"] += dg
    for l in reversed(range(cfg.n_layers)):
        p = f"layers.{l}."
        c = cache["layers"][l]
        # MLP: x2 = x1 + H Wd^T  (residual: gradient passes through, Eq. 2 "+1")
        grads[p + "wd"] += dx.T @ c["H"]
        dH = dx @ P[p + "wd"]
        dG, dU = swiglu_bwd(dH, c["G"], c["U"])
        grads[p + "wg"] += dG.T @ c["xn2"]
        grads[p + "wu"] += dU.T @ c["xn2"]
        dxn2 = dG @ P[p + "wg"] + dU @ P[p + "wu"]
        dx1n, dg2 = rmsnorm_bwd(dxn2, c["x1"], P[p + "ln2"], c["r2"])
        grads[p + "ln2"] += dg2
        dx1 = dx + dx1n
        # attention: x1 = x + O Wo^T
        grads[p + "wo"] += dx1.T @ c["o2"]
        do = _heads(dx1 @ P[p + "wo"], cfg.n_q_heads, d)
        dqr, dkr, dvh = attention_bwd(do, c["qr"], c["kr"], c["vh"], c["o"])
        dq = rope_bwd(dqr, cos, sin).reshape(s, -1)
        dk = rope_bwd(dkr, cos, sin).reshape(s, -1)
        dv = dvh.reshape(s, -1)
        grads[p + "wq"] += dq.T @ c["xn"]
        grads[p + "wk"] += dk.T @ c["xn"]
        grads[p + "wv"] += dv.T @ c["xn"]
        if cfg.qkv_bias:
            grads[p + "bq"] += dq.sum(axis=0)
            grads[p + "bk"] += dk.sum(axis=0)
            grads[p + "bv"] += dv.sum(axis=0)
        dxn = dq @ P[p + "wq"] + dk @ P[p + "wk"] + dv @ P[p + "wv"]
        dx0n, dg1 = rmsnorm_bwd(dxn, c["x"], P[p + "ln1"], c["r1"])
        grads[p + "ln1"] += dg1
        dx = dx1 + dx0n
    tok = cache["tok"] if embed_tok is None else embed_tok
    np.add.at(grads["embed"], tok, dx[embed_row0:])
    return dx


def forward_backward(P: Params, cfg, tokens, targets):
    """The plain result the STP step must reach: L = mean_b loss_b and
    dL/dparams, gradients accumulated over the m microbatches (reading Q19)."""
    m, s = tokens.shape
    grads = {k: np.zeros_like(v) for k, v in P.items()}
    losses = []
    for b in range(m):
        loss_b, cache = forward_mb(P, cfg, tokens[b], targets[b])
        losses.append(loss_b)
        backward_mb(P, cfg, cache, grads, 1.0 / (s * m))
    return float(np.mean(losses)), grads


def loss_only(P: Params, cfg, tokens, targets):
    return float(np.mean([forward_mb(P, cfg, tokens[b], targets[b])[0]
                          for b in range(tokens.shape[0])]))


# ---------------------------------------------------------------------------
# TP/SP sharding (SURVEY §8c.1 "Parameter storage ... TP shards")
# ---------------------------------------------------------------------------

def shard_params(P: Params, cfg, t: int, r: int) -> Params:
    """Rank r's shard of every parameter, in the GPU layout that
    include/stp.h documents (fused QKV rows = [q heads of r | k heads of r |
    v heads of r]; fused gate/up rows = [gate rows of r | up rows of r];
    Wo / Wd column blocks; vocab row blocks of embed / lm_head; gammas
    replicated).  Written independently of the product's packer."""
    d = cfg.head_dim
    qh, kh, fi, vv = cfg.n_q_heads // t, cfg.n_kv_heads // t, cfg.ffn // t, cfg.vocab // t
    qs = slice(r * qh * d, (r + 1) * qh * d)
    ks = slice(r * kh * d, (r + 1) * kh * d)
    fs = slice(r * fi, (r + 1) * fi)
    vs = slice(r * vv, (r + 1) * vv)
    out = {"embed": P["embed"][vs], "lm_head": P["lm_head"][vs],
           "final_ln": P["final_ln"]}
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        out[p + "ln1"] = P[p + "ln1"]
        out[p + "ln2"] = P[p + "ln2"]
        out[p + "wqkv"] = np.concatenate([P[p + "wq"][qs], P[p + "wk"][ks], P[p + "wv"][ks]], 0)
        if cfg.qkv_bias:
            out[p + "bqkv"] = np.concatenate([P[p + "bq"][qs], P[p + "bk"][ks], P[p + "bv"][ks]], 0)
        out[p + "wo"] = P[p + "wo"][:, qs]
        out[p + "wgu"] = np.concatenate([P[p + "wg"][fs], P[p + "wu"][fs]], 0)
        out[p + "wd"] = P[p + "wd"][:, fs]
    return out


def _ag(shards: List[np.ndarray]) -> np.ndarray:
    """All-gather of row shards = concatenation."""
    return np.concatenate(shards, axis=0)


def _rs(partials: List[np.ndarray]) -> List[np.ndarray]:
    """Reduce-scatter: row block r of the sum over ranks."""
    tot = sum(partials)
    return np.split(tot, len(partials), axis=0)


def forward_backward_sp(P: Params, cfg, tokens, targets, t: int):
    """The same step computed as t emulated TP ranks in the sequence-parallel
    dataflow the GPU path runs (AG before column-parallel GEMMs, RS after
    row-parallel GEMMs, residual added to the own shard after the RS,
    vocab-parallel embedding and cross-entropy).  Returns (loss, per-rank
    gradient dicts in the shard layout of `shard_params`, with gamma grads as
    per-rank partials)."""
    m, s = tokens.shape
    assert s % t == 0
    d = cfg.head_dim
    R = range(t)
    S = [shard_params(P, cfg, t, r) for r in R]
    G = [{k: np.zeros_like(v) for k, v in S[r].items()} for r in R]
    qh, kh, fi, vv = cfg.n_q_heads // t, cfg.n_kv_heads // t, cfg.ffn // t, cfg.vocab // t
    qd, kd = qh * d, kh * d
    cos, sin = rope_tables(s, d, cfg.rope_theta)
    losses = []
    for b in range(m):
        tok, tgt = tokens[b], targets[b]
        # vocab-parallel embedding: rank r contributes rows of its vocab range
        parts = []
        for r in R:
            e = np.zeros((s, cfg.hidden))
            own = (tok >= r * vv) & (tok < (r + 1) * vv)
            e[own] = S[r]["embed"][tok[own] - r * vv]
            parts.append(e)
        x = _rs(parts)                                   # x[r]: [s/t, h]
        cache = []
        for l in range(cfg.n_layers):
            p = f"layers.{l}."
            c = {"x": x}
            nr = [rmsnorm_fwd(x[r], S[r][p + "ln1"], cfg.rms_eps) for r in R]
            c["r1"] = [a[1] for a in nr]
            xn = _ag([a[0] for a in nr])                 # full [s, h], same on all ranks
            c["xn"] = xn
            part, st = [], []
            for r in R:
                qkv = xn @ S[r][p + "wqkv"].T
                if cfg.qkv_bias:
                    qkv = qkv + S[r][p + "bqkv"]
                q = rope_fwd(_heads(qkv[:, :qd], qh, d), cos, sin)
                k = rope_fwd(_heads(qkv[:, qd:qd + kd], kh, d), cos, sin)
                v = _heads(qkv[:, qd + kd:], kh, d)
                o, _ = attention_fwd(q, k, v)
                o2 = o.reshape(s, -1)
                part.append(o2 @ S[r][p + "wo"].T)
                st.append(dict(q=q, k=k, v=v, o=o, o2=o2))
            c["attn"] = st
            red = _rs(part)
            x1 = [red[r] + x[r] for r in R]              # Eq. 1, SP form (Q10)
            c["x1"] = x1
            nr = [rmsnorm_fwd(x1[r], S[r][p + "ln2"], cfg.rms_eps) for r in R]
            c["r2"] = [a[1] for a in nr]
            xn2 = _ag([a[0] for a in nr])
            c["xn2"] = xn2
            part, st = [], []
            for r in R:
                gu = xn2 @ S[r][p + "wgu"].T
                Gm, Um = gu[:, :fi], gu[:, fi:]
                H = swiglu_fwd(Gm, Um)
                part.append(H @ S[r][p + "wd"].T)
                st.append(dict(G=Gm, U=Um, H=H))
            c["mlp"] = st
            red = _rs(part)
            x = [red[r] + x1[r] for r in R]
            cache.append(c)
        nr = [rmsnorm_fwd(x[r], S[r]["final_ln"], cfg.rms_eps) for r in R]
        rf = [a[1] for a in nr]
        xf = _ag([a[0] for a in nr])
        logits = [xf @ S[r]["lm_head"].T for r in R]     # [s, V/t] per rank
        # vocab-parallel CE: combine per-rank (max, sum-exp, target logit)
        mloc = [lg.max(axis=-1) for lg in logits]
        M = np.max(np.stack(mloc), axis=0)
        Z = sum(np.exp(logits[r] - M[:, None]).sum(axis=-1) for r in R)
        lse = M + np.log(Z)
        tl = np.zeros(s)
        for r in R:
            own = (tgt >= r * vv) & (tgt < (r + 1) * vv)
            tl[own] = logits[r][np.nonzero(own)[0], tgt[own] - r * vv]
        losses.append(float(np.mean(lse - tl)))
        scale = 1.0 / (s * m)
        # ---- backward ----
        dxf_part = []
        for r in R:
            dl = np.exp(logits[r] - lse[:, None])
            own = (tgt >= r * vv) & (tgt < (r + 1) * vv)
            dl[np.nonzero(own)[0], tgt[own] - r * vv] -= 1.0
            dl *= scale
            G[r]["lm_head"] += dl.T @ xf
            dxf_part.append(dl @ S[r]["lm_head"])
        dxf = _rs(dxf_part)
        dx = []
        for r in R:
            a, g = rmsnorm_bwd(dxf[r], x[r], S[r]["final_ln"], rf[r])
            G[r]["final_ln"] += g
            dx.append(a)
        for l in reversed(range(cfg.n_layers)):
            p = f"layers.{l}."
            c = cache[l]
            dY = _ag(dx)                                 # full [s, h]
            part = []
            for r in R:
                st = c["mlp"][r]
                G[r][p + "wd"] += dY.T @ st["H"]
                dH = dY @ S[r][p + "wd"]
                dG, dU = swiglu_bwd(dH, st["G"], st["U"])
                dGU = np.concatenate([dG, dU], axis=1)
                G[r][p + "wgu"] += dGU.T @ c["xn2"]
                part.append(dGU @ S[r][p + "wgu"])
            red = _rs(part)
            dx1 = []
            for r in R:
                a, g = rmsnorm_bwd(red[r], c["x1"][r], S[r][p + "ln2"], c["r2"][r])
                G[r][p + "ln2"] += g
                dx1.append(a + dx[r])                    # residual (Eq. 2 "+1")
            dY = _ag(dx1)
            part = []
            for r in R:
                st = c["attn"][r]
                G[r][p + "wo"] += dY.T @ st["o2"]
                do = _heads(dY @ S[r][p + "wo"], qh, d)
                dq, dk, dv = attention_bwd(do, st["q"], st["k"], st["v"], st["o"])
                dq = rope_bwd(dq, cos, sin).reshape(s, -1)
                dk = rope_bwd(dk, cos, sin).reshape(s, -1)
                dqkv = np.concatenate([dq, dk, dv.reshape(s, -1)], axis=1)
                G[r][p + "wqkv"] += dqkv.T @ c["xn"]
                if cfg.qkv_bias:
                    G[r][p + "bqkv"] += dqkv.sum(axis=0)
                part.append(dqkv @ S[r][p + "wqkv"])
            red = _rs(part)
            ndx = []
            for r in R:
                a, g = rmsnorm_bwd(red[r], c["x"][r], S[r][p + "ln1"], c["r1"][r])
                G[r][p + "ln1"] += g
                ndx.append(a + dx1[r])
            dx = ndx
        dX0 = _ag(dx)
        for r in R:
            own = (tok >= r * vv) & (tok < (r + 1) * vv)
            np.add.at(G[r]["embed"], tok[own] - r * vv, dX0[own])
    return float(np.mean(losses)), G
