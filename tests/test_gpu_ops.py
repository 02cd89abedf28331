"""Each fused kernel vs the oracle's sub-function (oracle/model.py) on the
same seeded inputs, fp32 and bf16 storage.

Tolerances: fp32 kernels compute in fp32 against an
fp64 oracle -> relative Frobenius error <= 1e-5 (RoPE/attention 2e-5); bf16
kernels round inputs to bf16 (the oracle receives the same rounded inputs) and
outputs to bf16 -> relative Frobenius error <= 1e-2 (attention 2e-2), which is
a few bf16 ulps (2^-8) of accumulated rounding.
"""
import numpy as np
import pytest
import torch

from oracle import model as om

pytestmark = pytest.mark.gpu

DT = {"f32": torch.float32, "bf16": torch.bfloat16}
TOL = {"f32": 1e-5, "bf16": 1e-2}


def _ops():
    from paper_2510_27257_b200 import ops
    return ops


def _in(shape, seed, dt, scale=1.0, offset=0.0):
    a = offset + scale * np.random.default_rng(seed).standard_normal(shape)
    t = torch.from_numpy(a).to(DT[dt])
    return t.double().numpy(), t.cuda()


def _np(t):
    return t.double().cpu().numpy()


def _rel(got, ref):
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("rows,h", [(1, 64), (37, 136), (1024, 3584)])
def test_rmsnorm_fwd_bwd(dt, rows, h):
    ops = _ops()
    x, dx_ = _in((rows, h), 1, dt)
    g, dg_ = _in((h,), 2, dt, 0.1, 1.0)
    r, dr_ = _in((rows, h), 3, dt)
    dy, ddy = _in((rows, h), 4, dt)
    xin = x + r
    y_ref, rs_ref = om.rmsnorm_fwd(xin, g, 1e-6)
    y = torch.empty_like(dx_)
    xo = torch.empty_like(dx_)
    rs = torch.empty(rows, dtype=torch.float32, device="cuda")
    ops.rmsnorm_fwd(dx_, dg_, 1e-6, y, rs, resid=dr_, x_out=xo)
    torch.cuda.synchronize()
    assert _rel(_np(xo), xin) <= TOL[dt]
    assert _rel(_np(y), y_ref) <= TOL[dt]
    # rstd is computed from the stored (rounded) residual sum
    assert _rel(_np(rs), om.rmsnorm_fwd(_np(xo), g, 1e-6)[1][:, 0]) <= 1e-5
    # backward with residual-grad term (Eq. 2 "+1"), x = rounded x_out
    xr = _np(xo)
    _, rs2 = om.rmsnorm_fwd(xr, g, 1e-6)
    dx_ref, dg_ref = om.rmsnorm_bwd(dy, xr, g, rs2)
    dx_ref = dx_ref + r
    dx = torch.empty_like(dx_)
    dgam = torch.zeros(h, dtype=torch.float32, device="cuda")
    ops.rmsnorm_bwd(ddy, xo, dg_, rs, dx, dgam, dres=dr_)
    torch.cuda.synchronize()
    assert _rel(_np(dx), dx_ref) <= TOL[dt]
    assert _rel(_np(dgam), dg_ref) <= (1e-5 if dt == "f32" else 3e-3)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("s,nh,d,theta", [(7, 2, 16, 1e6), (300, 3, 128, 1e6), (4096, 2, 128, 1e4)])
def test_rope(dt, s, nh, d, theta):
    ops = _ops()
    extra = 16
    x, dx_ = _in((s, nh * d + 2 * extra), 5, dt)
    cos, sin = om.rope_tables(s, d, theta)
    ref = x.copy()
    sl = slice(extra, extra + nh * d)
    ref[:, sl] = om.rope_fwd(x[:, sl].reshape(s, nh, d), cos, sin).reshape(s, -1)
    ops.rope(dx_, extra, nh, d, theta)
    torch.cuda.synchronize()
    tol = 2e-5 if dt == "f32" else TOL[dt]
    assert _rel(_np(dx_), ref) <= tol
    assert np.array_equal(_np(dx_)[:, :extra], x[:, :extra])
    g = _np(dx_)
    bref = g.copy()
    bref[:, sl] = om.rope_bwd(g[:, sl].reshape(s, nh, d), cos, sin).reshape(s, -1)
    ops.rope(dx_, extra, nh, d, theta, backward=True)
    torch.cuda.synchronize()
    assert _rel(_np(dx_), bref) <= tol


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("s,I", [(5, 8), (100, 176), (512, 4736)])
def test_swiglu(dt, s, I):
    ops = _ops()
    gu, dgu_ = _in((s, 2 * I), 6, dt, 2.0)
    H = torch.empty(s, I, dtype=DT[dt], device="cuda")
    ops.swiglu_fwd(dgu_, H)
    torch.cuda.synchronize()
    assert _rel(_np(H), om.swiglu_fwd(gu[:, :I], gu[:, I:])) <= TOL[dt]
    dH, ddH = _in((s, I), 7, dt)
    out = torch.empty_like(dgu_)
    ops.swiglu_bwd(ddH, dgu_, out)
    torch.cuda.synchronize()
    dG, dU = om.swiglu_bwd(dH, gu[:, :I], gu[:, I:])
    assert _rel(_np(out), np.concatenate([dG, dU], 1)) <= TOL[dt]


ATT = [(1, 2, 1, 16), (33, 4, 2, 16), (130, 4, 4, 32), (200, 6, 2, 64), (257, 7, 1, 128), (1024, 4, 2, 128),
       (2048, 7, 1, 128), (300, 2, 2, 128)]


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("s,nq,nkv,d", ATT)
def test_attention_fwd_bwd(dt, s, nq, nkv, d):
    if dt == "f32" and s > 300:
        pytest.skip("fp32 SIMT attention is the small-shape parity path")
    ops = _ops()
    W = (nq + 2 * nkv) * d
    qkv, dqkv_ = _in((s, W), 8, dt)
    q = qkv[:, :nq * d].reshape(s, nq, d)
    k = qkv[:, nq * d:(nq + nkv) * d].reshape(s, nkv, d)
    v = qkv[:, (nq + nkv) * d:].reshape(s, nkv, d)
    o_ref, lse_ref = om.attention_fwd(q, k, v)
    o = torch.empty(s, nq * d, dtype=DT[dt], device="cuda")
    lse = torch.empty(nq, s, dtype=torch.float32, device="cuda")
    ops.attn_fwd(dqkv_, nq, nkv, d, o, lse)
    torch.cuda.synchronize()
    tol = 2e-5 if dt == "f32" else 2e-2
    assert _rel(_np(o), o_ref.reshape(s, -1)) <= tol
    assert np.abs(_np(lse) - lse_ref).max() <= (1e-4 if dt == "f32" else 2e-2)
    do, ddo = _in((s, nq * d), 9, dt)
    og = _np(o).reshape(s, nq, d)   # backward uses the kernel's (rounded) O, as the unit does
    dq, dk, dv = om.attention_bwd(do.reshape(s, nq, d), q, k, v, og)
    dqkv = torch.zeros(s, W, dtype=DT[dt], device="cuda")
    ops.attn_bwd(dqkv_, nq, nkv, d, o, ddo, lse, dqkv)
    torch.cuda.synchronize()
    got = _np(dqkv)
    tol = 5e-5 if dt == "f32" else 3e-2
    assert _rel(got[:, :nq * d], dq.reshape(s, -1)) <= tol
    assert _rel(got[:, nq * d:(nq + nkv) * d], dk.reshape(s, -1)) <= tol
    assert _rel(got[:, (nq + nkv) * d:], dv.reshape(s, -1)) <= tol


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_embedding_vocab_parallel(dt):
    ops = _ops()
    V, h, s, t = 64, 32, 50, 4
    E, dE_ = _in((V, h), 10, dt)
    tok = np.random.default_rng(11).integers(0, V, s).astype(np.int32)
    dtok = torch.from_numpy(tok).cuda()
    Vl = V // t
    tot = np.zeros((s, h))
    dX, ddX = _in((s, h), 12, dt)
    for r in range(t):
        Er = dE_[r * Vl:(r + 1) * Vl].contiguous()
        out = torch.empty(s, h, dtype=DT[dt], device="cuda")
        ops.embed_fwd(dtok, Er, r * Vl, out)
        acc = torch.zeros(Vl, h, dtype=torch.float32, device="cuda")
        ops.embed_bwd(dtok, ddX, r * Vl, acc)
        torch.cuda.synchronize()
        tot += _np(out)
        ref = np.zeros((Vl, h))
        own = (tok >= r * Vl) & (tok < (r + 1) * Vl)
        np.add.at(ref, tok[own] - r * Vl, dX[own])
        assert np.abs(_np(acc) - ref).max() <= 1e-5
    assert np.array_equal(tot, E[tok])


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("t", [1, 2, 4])
def test_vocab_parallel_cross_entropy(dt, t):
    ops = _ops()
    s, V = 96, 1000
    z, dz_ = _in((s, V), 13, dt, 3.0)
    tgt = np.random.default_rng(14).integers(0, V, s).astype(np.int32)
    dtgt = torch.from_numpy(tgt).cuda()
    per_tok, lse_ref = om.cross_entropy(z, tgt)
    Vl = V // t
    st = torch.empty(t, s, 3, dtype=torch.float32, device="cuda")
    parts = [dz_[:, r * Vl:(r + 1) * Vl] for r in range(t)]
    for r in range(t):
        ops.ce_stats(parts[r], dtgt, r * Vl, st[r])
    lse = torch.empty(s, dtype=torch.float32, device="cuda")
    loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    ops.ce_combine(st, lse, loss, 1.0 / s)
    torch.cuda.synchronize()
    assert abs(loss.item() - per_tok.mean()) <= 1e-5 * abs(per_tok.mean())
    assert np.abs(_np(lse) - lse_ref).max() <= 1e-4
    scale = 0.37
    ref = om.cross_entropy_bwd(z, tgt, lse_ref, scale)
    for r in range(t):
        ops.ce_grad(parts[r], dtgt, r * Vl, lse, scale)
    torch.cuda.synchronize()
    assert _rel(_np(dz_), ref) <= (1e-5 if dt == "f32" else 1e-2)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_colsum(dt):
    ops = _ops()
    X, dX_ = _in((700, 300), 15, dt)
    acc = torch.ones(300, dtype=torch.float32, device="cuda")
    ops.colsum_acc(dX_, acc)
    torch.cuda.synchronize()
    assert np.abs(_np(acc) - (1 + X.sum(0))).max() <= 1e-3


@pytest.mark.parametrize("s,nq,nkv", [(257, 7, 1), (1024, 4, 2), (2048, 7, 1), (300, 2, 2), (64, 2, 1), (65, 2, 1),
                                      (2, 2, 1), (63, 4, 4), (129, 2, 1), (4096, 4, 1), (6144, 7, 1)])
def test_attention_tcgen05_shapes(s, nq, nkv):
    """The tcgen05 forward and fused backward (d = 128) over ragged lengths,
    GQA group sizes 1-7 and the TP4 bench shape, against the oracle."""
    test_attention_fwd_bwd("bf16", s, nq, nkv, 128)


def test_attention_bwd_repeatable():
    """The fused backward adds dQ / dK / dV partials with L2 reductions, so
    the fp32 summation order varies between runs: two runs must agree to
    within a few bf16 ulps (the oracle comparison bounds the error itself)."""
    ops = _ops()
    s, nq, nkv, d = 2048, 7, 1, 128
    W = (nq + 2 * nkv) * d
    _, qkv = _in((s, W), 21, "bf16")
    o = torch.empty(s, nq * d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(nq, s, dtype=torch.float32, device="cuda")
    ops.attn_fwd(qkv, nq, nkv, d, o, lse)
    _, do = _in((s, nq * d), 22, "bf16")
    outs = []
    for _ in range(8):
        dqkv = torch.zeros(s, W, dtype=torch.bfloat16, device="cuda")
        ops.attn_bwd(qkv, nq, nkv, d, o, do, lse, dqkv)
        outs.append(dqkv.float())
    torch.cuda.synchronize()
    for x in outs[1:]:
        diff = (x - outs[0]).abs()
        assert (diff <= 2 ** -6 * outs[0].abs() + 1e-6).all()


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("s,h,Vl", [(5, 64, 200), (300, 256, 1000), (1024, 3584, 4096)])
def test_lm_head_ce_statistics_fp32(dt, s, h, Vl):
    """F_HEAD: logits = xf W^T stored in the model dtype, and the local CE
    statistics (row max, sum exp(z - max), target logit) from the fp32
    accumulators (GEMM epilogue for bf16; reading Q18) -- compared with the
    exact statistics of the fp64 product of the same (rounded) inputs, so the
    bf16 rounding of the logits does not enter the statistics."""
    ops = _ops()
    x, dx_ = _in((s, h), 21, dt)
    w, dw_ = _in((Vl, h), 22, dt, 0.05)
    v0 = 3 * Vl
    tgt = np.random.default_rng(23).integers(0, 4 * Vl, s).astype(np.int32)
    z = x @ w.T
    logits = torch.empty(s, Vl, dtype=DT[dt], device="cuda")
    stats = torch.empty(s, 3, dtype=torch.float32, device="cuda")
    ops.lm_head_ce(dx_, dw_, logits, torch.from_numpy(tgt).cuda(), v0, stats)
    torch.cuda.synchronize()
    st = _np(stats)
    mx = z.max(axis=1)
    se = np.exp(z - mx[:, None]).sum(axis=1)
    own = (tgt >= v0) & (tgt < v0 + Vl)
    tl = np.where(own, z[np.arange(s), np.clip(tgt - v0, 0, Vl - 1)], 0.0)
    assert np.abs(st[:, 0] - mx).max() <= 1e-4 * (1 + np.abs(mx).max())
    assert np.abs(st[:, 1] / se - 1).max() <= 1e-4
    assert np.abs(st[:, 2] - tl).max() <= 1e-4 * (1 + np.abs(tl).max())
    assert _rel(_np(logits), z) <= (1e-5 if dt == "f32" else 1e-2)
