"""Helpers shared by the GPU stage parity tests and smoke(): run the oracle
and the C-ABI stage on the same seeded inputs and compare (SURVEY §8c.4
numerics gates: fp32 loss/grad rel 1e-4; bf16 loss rel 2e-2, grad-norm rel
5e-2 — plus, for bf16, a per-tensor difference gate ||g - g_ref|| /
||g_ref|| <= 3e-2, so a permuted, transposed or sign-flipped gradient with
the right norm cannot pass).

The per-tensor gate is applied with the oracle evaluated on the SAME
bf16-rounded parameters the stage computes with (bf16_inputs=True) and the
model's N(0, 0.02^2) initialisation.  Measured on B200 (tools/diag_bf16.py,
Qwen2-7B layer shapes, 2 layers, s = 256 / 1024, V = 4096): stage vs that
oracle 1.2-2.4e-2 per tensor; for scale, rounding the weights alone moves the
fp64 oracle's gradients by 1.1-2.2e-2 (a random-init LM's gradient is that
sensitive), so 3e-2 sits just above the arithmetic's own floor.  With the
harder parity init (std 0.05, random gammas / biases) the same rounding moves
gradients by up to 14%: those cases keep north_star's norm gate only."""
import numpy as np

import stp_inputs as si
from oracle import model as om


def round_bf16(P):
    """Parameters rounded to bf16 (round-to-nearest-even), kept in fp64: the
    values a bf16 stage actually computes with, so the oracle sees the same
    inputs as the kernels (as in the per-op tests)."""
    import torch
    return {k: torch.from_numpy(v).to(torch.bfloat16).double().numpy() for k, v in P.items()}


def oracle_reference(cfg, m, seed=3, parity=True, std=0.05, bf16_inputs=False):
    P = si.make_params(cfg, seed=seed, std=std, parity=parity)
    if bf16_inputs:
        P = round_bf16(P)
    toks, tgts = si.make_tokens(cfg, m, seed=seed + 100)
    loss, G = om.forward_backward(P, cfg, toks, tgts)
    return P, toks, tgts, loss, G


def rank_grads_ref(cfg, G, tp, r):
    return om.shard_params(G, cfg, tp, r)


BF16_DIFF_TOL = 3e-2


def compare(cfg, got: dict, ref: dict, loss, ref_loss, dtype, names=None, elementwise=False):
    """Returns a list of failure strings (empty = pass)."""
    bad = []
    lt = 1e-4 if dtype == "f32" else 2e-2
    if abs(loss - ref_loss) > lt * abs(ref_loss):
        bad.append(f"loss {loss} vs {ref_loss}")
    for k, g in got.items():
        if names is not None and k not in names:
            continue
        r = ref[k]
        nr = np.linalg.norm(r)
        if dtype == "f32":
            err = np.linalg.norm(g - r) / max(nr, 1e-30)
            if err > 1e-4:
                bad.append(f"{k}: rel err {err:.3e}")
        else:
            err = abs(np.linalg.norm(g) - nr) / max(nr, 1e-30)
            if err > 5e-2:
                bad.append(f"{k}: grad-norm rel err {err:.3e}")
            if elementwise:
                derr = np.linalg.norm(g - r) / max(nr, 1e-30)
                if derr > BF16_DIFF_TOL:
                    bad.append(f"{k}: rel diff {derr:.3e}")
    return bad
