"""Tensor-level wrappers of the stp_op_* entry points (include/stp_ops.h).

Marshalling only: extracts device pointers, strides, dtype and the current
CUDA stream from torch tensors and calls libstp.so.  torch is used for
device memory and streams; all arithmetic runs in the library's kernels.
"""
from __future__ import annotations

import torch

from ._lib import call, lib

F32, BF16 = 0, 1
NT, NN, TN = 0, 1, 2
EPI_STORE, EPI_BIAS, EPI_ACCUM_F32, EPI_RESID = 0, 1, 2, 3


def dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def ptr(t):
    return None if t is None else t.data_ptr()


def stream():
    return torch.cuda.current_stream().cuda_stream


def gemm(layout, A, B, C, M, N, K, epi=EPI_STORE, bias=None, R=None, max_ctas=0, dtype=None):
    """C = op(A) op(B) with the layouts of stp_op_gemm; leading dims from the
    tensors' row strides."""
    dtype = dt(A) if dtype is None else dtype
    call("stp_op_gemm", dtype, layout, epi, M, N, K, ptr(A), A.stride(0), ptr(B), B.stride(0),
         ptr(C), C.stride(0), ptr(bias), ptr(R), R.stride(0) if R is not None else 0, max_ctas, stream())


def rmsnorm_fwd(x, gamma, eps, y, rstd=None, resid=None, x_out=None):
    rows, h = x.shape
    call("stp_op_rmsnorm_fwd", dt(x), rows, h, ptr(x), ptr(resid), ptr(x_out), ptr(gamma), eps,
         ptr(y), ptr(rstd), stream())


def rmsnorm_bwd(dy, x, gamma, rstd, dx, dgamma_acc=None, dres=None):
    rows, h = x.shape
    call("stp_op_rmsnorm_bwd", dt(x), rows, h, ptr(dy), ptr(x), ptr(gamma), ptr(rstd), ptr(dres),
         ptr(dx), ptr(dgamma_acc), stream())


def rope(x, col0, n_heads, d, theta, backward=False, pos0=0):
    s = x.shape[0]
    call("stp_op_rope", dt(x), int(backward), s, x.stride(0), col0, n_heads, d, theta, pos0, ptr(x), stream())


def swiglu_fwd(gu, H):
    s, I = H.shape
    call("stp_op_swiglu_fwd", dt(gu), s, I, ptr(gu), ptr(H), stream())


def swiglu_bwd(dH, gu, dgu):
    s, I = dH.shape
    call("stp_op_swiglu_bwd", dt(gu), s, I, ptr(dH), ptr(gu), ptr(dgu), stream())


def attn_fwd(qkv, nq, nkv, d, o, lse):
    """qkv: [s, (nq+2nkv)d] (q | k | v columns); o: [s, nq d]; lse fp32 [nq, s]."""
    s = qkv.shape[0]
    es = qkv.element_size()
    base = qkv.data_ptr()
    call("stp_op_attn_fwd", dt(qkv), s, nq, nkv, d, base, base + nq * d * es, base + (nq + nkv) * d * es,
         qkv.stride(0), ptr(o), o.stride(0), ptr(lse), stream())


def attn_bwd(qkv, nq, nkv, d, o, dout, lse, dqkv):
    s = qkv.shape[0]
    es = qkv.element_size()
    ws = torch.empty(max(1, lib.stp_op_attn_bwd_ws_bytes(s, nq, nkv, d)), dtype=torch.uint8, device=qkv.device)
    b, g = qkv.data_ptr(), dqkv.data_ptr()
    call("stp_op_attn_bwd", dt(qkv), s, nq, nkv, d, b, b + nq * d * es, b + (nq + nkv) * d * es, qkv.stride(0),
         ptr(o), o.stride(0), ptr(dout), ptr(lse), g, g + nq * d * es, g + (nq + nkv) * d * es, dqkv.stride(0),
         ptr(ws), stream())


def attn_full_fwd(qkv, nh, d, o, lse):
    """Bidirectional attention (ViT): qkv [s, 3 nh d] (q | k | v); o [s, nh d]; lse fp32 [nh, s]."""
    call("stp_op_attn_full_fwd", dt(qkv), qkv.shape[0], nh, d, ptr(qkv), qkv.stride(0), ptr(o), o.stride(0),
         ptr(lse), stream())


def attn_full_bwd(qkv, nh, d, o, dout, lse, dqkv):
    s = qkv.shape[0]
    ws = torch.empty(max(1, lib.stp_op_attn_bwd_ws_bytes(s, nh, nh, d)), dtype=torch.uint8, device=qkv.device)
    call("stp_op_attn_full_bwd", dt(qkv), s, nh, d, ptr(qkv), qkv.stride(0), ptr(o), o.stride(0), ptr(dout),
         ptr(lse), ptr(dqkv), dqkv.stride(0), ptr(ws), stream())


def layernorm_fwd(x, gamma, beta, eps, y, mean=None, rstd=None, resid=None, x_out=None):
    rows, h = x.shape
    call("stp_op_layernorm_fwd", dt(x), rows, h, ptr(x), ptr(resid), ptr(x_out), ptr(gamma), ptr(beta), eps,
         ptr(y), ptr(mean), ptr(rstd), stream())


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dgamma_acc=None, dbeta_acc=None, dres=None):
    rows, h = x.shape
    call("stp_op_layernorm_bwd", dt(x), rows, h, ptr(dy), ptr(x), ptr(gamma), ptr(mean), ptr(rstd), ptr(dres),
         ptr(dx), ptr(dgamma_acc), ptr(dbeta_acc), stream())


QGELU, GELU = 0, 1


def act_fwd(kind, a, y):
    call("stp_op_act_fwd", dt(a), kind, a.numel(), ptr(a), ptr(y), stream())


def act_bwd(kind, dy, a, da):
    call("stp_op_act_bwd", dt(a), kind, a.numel(), ptr(dy), ptr(a), ptr(da), stream())


def rope2d(x, col0, n_heads, d, grid_w, theta=10000.0, backward=False):
    call("stp_op_rope2d", dt(x), int(backward), x.shape[0], x.stride(0), col0, n_heads, d, grid_w, theta, ptr(x),
         stream())


def embed_fwd(tok, E, v0, out):
    s, h = out.shape
    call("stp_op_embed_fwd", dt(E), s, h, ptr(tok), v0, E.shape[0], ptr(E), ptr(out), stream())


def embed_bwd(tok, dX, v0, dE_acc):
    s, h = dX.shape
    call("stp_op_embed_bwd", dt(dX), s, h, ptr(tok), v0, dE_acc.shape[0], ptr(dX), ptr(dE_acc), stream())


def ce_stats(logits, tgt, v0, stats):
    s, Vl = logits.shape
    call("stp_op_ce_stats", dt(logits), s, Vl, ptr(logits), logits.stride(0), ptr(tgt), v0, ptr(stats), stream())


def lm_head_ce(xf, W, logits, tgt, v0, stats):
    """logits = xf W^T (stored) + fp32 CE statistics of the accumulators -> stats [s, 3]."""
    s_, h = xf.shape
    Vl = W.shape[0]
    ws = torch.empty(max(1, lib.stp_op_lm_head_ce_ws_bytes(s_, Vl)), dtype=torch.uint8, device=xf.device)
    call("stp_op_lm_head_ce", dt(xf), s_, Vl, h, ptr(xf), ptr(W), ptr(logits), ptr(tgt), v0, ptr(ws), ptr(stats),
         stream())


def ce_combine(stats_all, lse, loss_acc, loss_scale):
    t, s, _ = stats_all.shape
    call("stp_op_ce_combine", s, t, ptr(stats_all), ptr(lse), ptr(loss_acc), loss_scale, stream())


def ce_grad(logits, tgt, v0, lse, grad_scale):
    s, Vl = logits.shape
    call("stp_op_ce_grad", dt(logits), s, Vl, ptr(logits), logits.stride(0), ptr(tgt), v0, ptr(lse),
         grad_scale, stream())


def colsum_acc(X, acc):
    rows, n = X.shape
    call("stp_op_colsum_acc", dt(X), rows, n, ptr(X), X.stride(0), ptr(acc), stream())
