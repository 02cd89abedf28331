"""Helpers shared by the GPU stage parity tests and smoke(): run the oracle
and the C-ABI stage on the same seeded inputs and compare (SURVEY §8c.4
numerics gates: fp32 loss/grad rel 1e-4; bf16 loss rel 2e-2, grad-norm rel
5e-2)."""
import numpy as np

import stp_inputs as si
from oracle import model as om


def oracle_reference(cfg, m, seed=3, parity=True, std=0.05):
    P = si.make_params(cfg, seed=seed, std=std, parity=parity)
    toks, tgts = si.make_tokens(cfg, m, seed=seed + 100)
    loss, G = om.forward_backward(P, cfg, toks, tgts)
    return P, toks, tgts, loss, G


def rank_grads_ref(cfg, G, tp, r):
    return om.shard_params(G, cfg, tp, r)


def compare(cfg, got: dict, ref: dict, loss, ref_loss, dtype, names=None):
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
    return bad
