"""Helpers of the MLLM (ViT first chunk) parity tests: the oracle's MLLM step
(oracle/vit.py mllm_forward_backward) on seeded inputs, and rank r's shards
of its gradients in the stage layout (written here, independently of the
product's packer: heads / MLP / merger columns split in contiguous blocks)."""
import dataclasses

import numpy as np

import stp_inputs as si
from oracle import model as om
from oracle import vit as ov

# fp32 micro case: ViT 2 layers, h 64 (4 heads x 16), 4 x 4 patches -> 4 image
# tokens; LM = TINY at seq 32 (28 text tokens)
VIT_F32 = si.VitShape(hidden=64, n_layers=2, n_heads=4, head_dim=16, mlp=128, patch_dim=48, grid_h=4, grid_w=4,
                      out_hidden=64)
LM_F32 = dataclasses.replace(si.TINY, n_layers=2, seq=32)
# bf16 case on the tcgen05 kernels: d = 80 heads (ViT-600M head dim)
VIT_BF16 = si.VitShape(hidden=160, n_layers=2, n_heads=2, head_dim=80, mlp=320, patch_dim=96, grid_h=16, grid_w=8,
                       out_hidden=128)
LM_BF16 = dataclasses.replace(si.TINY, hidden=128, n_q_heads=4, n_kv_heads=2, head_dim=32, ffn=256, n_layers=2,
                              seq=96)


def oracle_vit_cfg(v: si.VitShape) -> ov.VitCfg:
    return ov.VitCfg(hidden=v.hidden, n_layers=v.n_layers, n_heads=v.n_heads, head_dim=v.head_dim, mlp=v.mlp,
                     patch_dim=v.patch_dim, merge=4, out_hidden=v.out_hidden, ln_eps=v.ln_eps)


def round_bf16(P):
    import torch
    return {k: torch.from_numpy(v).to(torch.bfloat16).double().numpy() for k, v in P.items()}


def mllm_reference(cfg, v: si.VitShape, m, seed=7, std=0.05, bf16_inputs=False):
    P = si.make_params(cfg, seed=seed, std=std, parity=True)
    PV = si.make_vit_params(v, seed=seed + 1, std=std, parity=True)
    patches = si.make_patches(v, m, seed=seed + 2)
    if bf16_inputs:
        P, PV = round_bf16(P), round_bf16(PV)
        patches = round_bf16({"x": patches})["x"]
    text, full, tgts = si.make_mllm_tokens(cfg, v.n_img, m, seed=seed + 3)
    loss, G, GV = ov.mllm_forward_backward(PV, oracle_vit_cfg(v), P, cfg, patches, (v.grid_h, v.grid_w), text, tgts)
    return P, PV, patches, full, tgts, loss, G, GV


def shard_vit_grads(GV, v: si.VitShape, t: int, r: int):
    out = {}
    hv, nl, ml, m4l = v.hidden, v.n_heads // t * v.head_dim, v.mlp // t, 4 * v.hidden // t
    for k, g in GV.items():
        short = k.rsplit(".", 1)[1]
        if k.startswith("merger."):
            if short in ("w1", "b1"):
                g = g[r * m4l:(r + 1) * m4l]
            elif short == "w2":
                g = g[:, r * m4l:(r + 1) * m4l]
        elif k != "vit.patch":
            if short in ("wqkv", "bqkv"):
                g = np.concatenate([g[j * hv + r * nl:j * hv + (r + 1) * nl] for j in range(3)], 0)
            elif short == "wo":
                g = g[:, r * nl:(r + 1) * nl]
            elif short in ("w1", "b1"):
                g = g[r * ml:(r + 1) * ml]
            elif short == "w2":
                g = g[:, r * ml:(r + 1) * ml]
        out[k] = g
    return out


def rank_reference(cfg, v, G, GV, t, r):
    ref = om.shard_params(G, cfg, t, r)
    ref.update(shard_vit_grads(GV, v, t, r))
    return ref
