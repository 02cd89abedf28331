"""Full-size checks at the bench workload (Qwen2-7B-shaped, seq 6144, TP=1):
every GEMM shape of the step in the launch configuration bench.py times
(default kernel selection: 1-SM / 2-SM tcgen05 by shape), and causal GQA
attention at s = 6144, each verified on SAMPLED outputs that the plain
definition computes one by one in fp64 (a dot product per GEMM entry; the
oracle's softmax row for a sampled query row).

Tolerance for a sampled bf16 GEMM entry: |got - ref| <= 8e-3 * (|ref| +
rms(ref_row-scale)) — bf16 output rounding (2^-9 relative) plus fp32
accumulation over K <= 37888 terms.
"""
import math

import numpy as np
import pytest
import torch

from oracle import model as om

pytestmark = pytest.mark.gpu

S, H, I, V, NQ, NKV, D = 6144, 3584, 18944, 152064, 28, 4, 128
QKV = (NQ + 2 * NKV) * D
GEMMS = [("qkv_fwd", 0, S, QKV, H, 0), ("o_fwd", 0, S, H, NQ * D, 0), ("fc1_fwd", 0, S, 2 * I, H, 0),
         ("fc2_fwd", 0, S, H, I, 0), ("lm_head_fwd", 0, S, V, H, 0),
         ("fc2_dgrad", 1, S, I, H, 0), ("fc1_dgrad", 1, S, H, 2 * I, 0), ("qkv_dgrad", 1, S, H, QKV, 0),
         ("lm_head_dgrad", 1, S, H, V, 0),
         ("fc2_wgrad", 2, H, I, S, 2), ("fc1_wgrad", 2, 2 * I, H, S, 2), ("qkv_wgrad", 2, QKV, H, S, 2),
         ("lm_head_wgrad", 2, V, H, S, 2)]


@pytest.mark.parametrize("name,layout,M,N,K,epi", GEMMS, ids=[g[0] for g in GEMMS])
def test_fullsize_gemm_sampled(name, layout, M, N, K, epi):
    from paper_2510_27257_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(7)
    shp = {0: ((M, K), (N, K)), 1: ((M, K), (K, N)), 2: ((K, M), (K, N))}[layout]
    A = torch.randn(shp[0], generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(shp[1], generator=g, device="cuda").to(torch.bfloat16)
    C0 = torch.randn(M, N, generator=g, device="cuda") if epi == 2 else None
    C = C0.clone() if epi == 2 else torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(layout, A, B, C, M, N, K, epi=epi, dtype=1)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    rows = rng.integers(0, M, 48)
    cols = rng.integers(0, N, 48)
    rows = np.concatenate([rows, [0, M - 1, M - 1]])
    cols = np.concatenate([cols, [N - 1, 0, N - 1]])
    for r, c in zip(rows, cols):
        a = (A[r] if layout != 2 else A[:, r]).double().cpu().numpy()
        b = (B[c] if layout == 0 else B[:, c]).double().cpu().numpy()
        ref = float(a @ b) + (float(C0[r, c]) if epi == 2 else 0.0)
        got = float(C[r, c])
        tol = 8e-3 * (abs(ref) + math.sqrt(K)) if epi != 2 else 1e-3 * (abs(ref) + math.sqrt(K))
        assert abs(got - ref) <= tol, (name, r, c, got, ref)


def test_fullsize_attention_sampled_rows():
    from paper_2510_27257_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(S, QKV, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty(S, NQ * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(NQ, S, device="cuda", dtype=torch.float32)
    ops.attn_fwd(qkv, NQ, NKV, D, o, lse)
    torch.cuda.synchronize()
    x = qkv.double().cpu().numpy()
    got_o = o.double().cpu().numpy()
    got_l = lse.cpu().numpy()
    rng = np.random.default_rng(1)
    for qrow in list(rng.integers(0, S, 6)) + [0, 127, 128, S - 1]:
        for h in (0, 6, 13, 27):
            gk = h // (NQ // NKV)
            q = x[qrow, h * D:(h + 1) * D]
            k = x[:qrow + 1, NQ * D + gk * D:NQ * D + (gk + 1) * D]
            v = x[:qrow + 1, (NQ + NKV) * D + gk * D:(NQ + NKV) * D + (gk + 1) * D]
            # the oracle's attention for this one query row (causal keys 0..qrow)
            o_ref, l_ref = om.attention_fwd(q[None, None, :], k[:, None, :], v[:, None, :]) if qrow == 0 else \
                (None, None)
            s_ = (k @ q) / math.sqrt(D)
            m = s_.max()
            p = np.exp(s_ - m)
            ref = (p @ v) / p.sum()
            lref = m + math.log(p.sum())
            if qrow == 0:
                assert np.allclose(o_ref[0, 0], ref) and abs(l_ref[0, 0] - lref) < 1e-12
            err = np.abs(got_o[qrow, h * D:(h + 1) * D] - ref).max()
            assert err <= 2e-2 * max(1.0, np.abs(ref).max()), (qrow, h, err)
            assert abs(got_l[h, qrow] - lref) <= 2e-2, (qrow, h)


def test_fullsize_attention_backward_sampled():
    """dQ, dK and dV at s = 6144 (the bench launch config) on sampled rows,
    against the plain definition (SURVEY §8c.1 "Attention") in fp64:
    P = softmax(Q K^T / sqrt(d) + causal), dP = dO V^T, D = rowsum(dO O),
    dS = P (dP - D), dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d), dV = P^T dO,
    dK / dV summed over the GQA group.  Every query row >= S/2 of the sampled
    kv group is evaluated (so key rows >= S/2 get their complete sums); dQ is
    also checked on early rows (0, 1, 127, 128, 1000) of another group."""
    from paper_2510_27257_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(4)
    qkv = torch.randn(S, QKV, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty(S, NQ * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(NQ, S, device="cuda", dtype=torch.float32)
    ops.attn_fwd(qkv, NQ, NKV, D, o, lse)
    do = torch.randn(S, NQ * D, generator=g, device="cuda").to(torch.bfloat16)
    dqkv = torch.zeros(S, QKV, device="cuda", dtype=torch.bfloat16)
    ops.attn_bwd(qkv, NQ, NKV, D, o, do, lse, dqkv)
    torch.cuda.synchronize()
    x = qkv.double().cpu().numpy()
    dO = do.double().cpu().numpy()
    got = dqkv.double().cpu().numpy()
    grp = NQ // NKV
    sc = 1.0 / math.sqrt(D)

    def head(h):
        gk = h // grp
        return (x[:, h * D:(h + 1) * D], x[:, NQ * D + gk * D:NQ * D + (gk + 1) * D],
                x[:, (NQ + NKV) * D + gk * D:(NQ + NKV) * D + (gk + 1) * D], dO[:, h * D:(h + 1) * D])

    def rows_bwd(h, rows):
        """P, dS for the given query rows of head h (full key range, causal)."""
        q, k, v, d_o = head(h)
        s_ = (q[rows] @ k.T) * sc
        s_[np.asarray(rows)[:, None] < np.arange(S)[None, :]] = -np.inf
        p = np.exp(s_ - s_.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        o_ = p @ v
        dp = d_o[rows] @ v.T
        dd = (d_o[rows] * o_).sum(1, keepdims=True)
        return p, p * (dp - dd)

    def check(gotv, ref, what):
        err = np.abs(gotv - ref).max()
        assert err <= 2e-2 * max(1.0, np.abs(ref).max()), (what, err, np.abs(ref).max())

    gk = NKV - 1
    rows = np.arange(S // 2, S)
    keys = [S - 1, S - 2, S - 70, S - 129, S // 2 + 3, S // 2]
    dk_ref = np.zeros((len(keys), D))
    dv_ref = np.zeros((len(keys), D))
    for hh in range(grp):
        h = gk * grp + hh
        q, k, v, d_o = head(h)
        p, ds = rows_bwd(h, rows)
        for n, j in enumerate(keys):
            dk_ref[n] += sc * (ds[:, j] @ q[rows])
            dv_ref[n] += p[:, j] @ d_o[rows]
        if hh in (0, grp - 1):
            for i in (S // 2, S // 2 + 64, S - 200, S - 1):
                check(got[i, h * D:(h + 1) * D], sc * (ds[i - S // 2] @ k), ("dq", i, h))
        del p, ds
    for n, j in enumerate(keys):
        check(got[j, (NQ + gk) * D:(NQ + gk + 1) * D], dk_ref[n], ("dk", j))
        check(got[j, (NQ + NKV + gk) * D:(NQ + NKV + gk + 1) * D], dv_ref[n], ("dv", j))
    early = [0, 1, 127, 128, 1000]
    for h in (0, 9):
        _, ds = rows_bwd(h, early)
        k = head(h)[1]
        for n, i in enumerate(early):
            check(got[i, h * D:(h + 1) * D], sc * (ds[n] @ k), ("dq", i, h))
