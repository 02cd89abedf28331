"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no model math, no schedule
logic): only model-shape presets, a seeded token generator and a seeded
parameter initialiser.  Both `oracle/` (CPU fp64) and the GPU path consume
exactly these arrays, so a parity test compares the two on identical inputs.

Recipe:
  * tokens: one sequence of length s+1 per microbatch, uniform int in [0, V),
    numpy default_rng(seed + 1000003*mb); tokens = seq[:-1], targets = seq[1:]
    (next-token prediction, reading Q16).
  * weights: N(0, std^2) per tensor (std 0.02), from a per-tensor seed
    crc32(name) ^ seed; RMSNorm gammas = 1 and biases = 0 unless
    `parity=True`, in which case gammas = 1 + 0.1 N(0,1) and biases
    = 0.02 N(0,1) so a dropped gamma or bias cannot hide.

Parameter names and shapes follow PyTorch Linear order [out, in]
(SURVEY.md §8c.1).
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, List

import numpy as np


@dataclasses.dataclass(frozen=True)
class ModelCfg:
    """Qwen2-style decoder shape (Table 2; readings Q9-Q14)."""
    vocab: int
    hidden: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    seq: int
    rms_eps: float = 1e-6
    rope_theta: float = 1e6
    qkv_bias: bool = True

    @property
    def q_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim


# BASELINE.json configs[0]: tiny 4-layer, hidden 64, 4 heads, seq 32 (fp32).
TINY = ModelCfg(vocab=256, hidden=64, n_layers=4, n_q_heads=4, n_kv_heads=2,
                head_dim=16, ffn=176, seq=32)
# Qwen2-7B layer shape: h 3584, 28/4 heads, d 128, I 18944.
QWEN2_7B = ModelCfg(vocab=152064, hidden=3584, n_layers=28, n_q_heads=28,
                    n_kv_heads=4, head_dim=128, ffn=18944, seq=4096)
# TP=8 variant (reading Q14): 32/8 heads, h unchanged.
QWEN2_7B_TP8 = dataclasses.replace(QWEN2_7B, n_q_heads=32, n_kv_heads=8)
# Qwen2.5-14B shape (reading Q13).
QWEN25_14B = ModelCfg(vocab=152064, hidden=5120, n_layers=48, n_q_heads=40,
                      n_kv_heads=8, head_dim=128, ffn=13824, seq=4096)

@dataclasses.dataclass(frozen=True)
class VitShape:
    """MLLM vision tower shape (ViT-600M of Qwen2-VL, Table 2 /
    P:L171): patches of a grid_h x grid_w image in 2x2
    merge-window order, merged 4:1 into out_hidden-wide LM input rows."""
    hidden: int = 1280
    n_layers: int = 32
    n_heads: int = 16
    head_dim: int = 80
    mlp: int = 5120
    patch_dim: int = 1176     # 3 * 2 * 14 * 14
    grid_h: int = 56
    grid_w: int = 56
    out_hidden: int = 3584
    ln_eps: float = 1e-6
    rope_theta: float = 10000.0

    @property
    def seq(self) -> int:
        return self.grid_h * self.grid_w

    @property
    def n_img(self) -> int:
        return self.seq // 4


VIT_600M = VitShape()


def vit_param_shapes(v: VitShape) -> Dict[str, tuple]:
    hv, m4 = v.hidden, 4 * v.hidden
    sh = {"vit.patch": (hv, v.patch_dim)}
    for l in range(v.n_layers):
        p = f"vit.{l}."
        sh.update({p + "ln1_g": (hv,), p + "ln1_b": (hv,), p + "wqkv": (3 * hv, hv), p + "bqkv": (3 * hv,),
                   p + "wo": (hv, hv), p + "bo": (hv,), p + "ln2_g": (hv,), p + "ln2_b": (hv,),
                   p + "w1": (v.mlp, hv), p + "b1": (v.mlp,), p + "w2": (hv, v.mlp), p + "b2": (hv,)})
    sh.update({"merger.ln_g": (hv,), "merger.ln_b": (hv,), "merger.w1": (m4, m4), "merger.b1": (m4,),
               "merger.w2": (v.out_hidden, m4), "merger.b2": (v.out_hidden,)})
    return sh


def make_vit_params(v: VitShape, seed: int = 0, std: float = 0.02, parity: bool = False) -> Dict[str, np.ndarray]:
    """LayerNorm gains 1 and all biases 0 (parity: 1 + 0.1 N(0,1) and
    0.02 N(0,1)); weights N(0, std^2); per-tensor seeds as make_param."""
    out = {}
    for name, shape in vit_param_shapes(v).items():
        rng = np.random.default_rng(_tensor_seed(name, seed))
        short = name.rsplit(".", 1)[-1]
        if short.endswith("_g"):
            out[name] = 1.0 + 0.1 * rng.standard_normal(shape) if parity else np.ones(shape)
        elif short.endswith("_b") or short.startswith("b"):
            out[name] = 0.02 * rng.standard_normal(shape) if parity else np.zeros(shape)
        else:
            out[name] = std * rng.standard_normal(shape)
    return out


def make_patches(v: VitShape, n_micro: int, seed: int = 4321) -> np.ndarray:
    """Random patch rows [n_micro, grid_h * grid_w, patch_dim], N(0, 1)
    (random patches [3136, 1176])."""
    return np.random.default_rng(seed).standard_normal((n_micro, v.seq, v.patch_dim))


def make_mllm_tokens(cfg: ModelCfg, n_img: int, n_micro: int, seed: int = 1234):
    """MLLM microbatch = [n_img image rows | cfg.seq - n_img text tokens]:
    text tokens [m, seq - n_img], the stage's token rows [m, seq] (0 at the
    image positions, which the embedding skips) and next-token targets
    [m, seq] for every position."""
    toks, tgts = make_tokens(cfg, n_micro, seed)
    text = np.ascontiguousarray(toks[:, n_img:])
    full = toks.copy()
    full[:, :n_img] = 0
    return text, full, tgts


PRESETS = {"tiny": TINY, "qwen2-7b": QWEN2_7B, "qwen2-7b-tp8": QWEN2_7B_TP8,
           "qwen2.5-14b": QWEN25_14B}


def layer_param_names(layer: int) -> List[str]:
    p = f"layers.{layer}."
    return [p + n for n in ("ln1", "wq", "bq", "wk", "bk", "wv", "bv", "wo",
                            "ln2", "wg", "wu", "wd")]


def param_shapes(cfg: ModelCfg) -> Dict[str, tuple]:
    h, I = cfg.hidden, cfg.ffn
    shapes = {"embed": (cfg.vocab, h)}
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        shapes.update({
            p + "ln1": (h,),
            p + "wq": (cfg.q_dim, h), p + "bq": (cfg.q_dim,),
            p + "wk": (cfg.kv_dim, h), p + "bk": (cfg.kv_dim,),
            p + "wv": (cfg.kv_dim, h), p + "bv": (cfg.kv_dim,),
            p + "wo": (h, cfg.q_dim),
            p + "ln2": (h,),
            p + "wg": (I, h), p + "wu": (I, h), p + "wd": (h, I),
        })
    shapes["final_ln"] = (h,)
    shapes["lm_head"] = (cfg.vocab, h)
    return shapes


def _tensor_seed(name: str, seed: int) -> int:
    return (zlib.crc32(name.encode()) ^ (seed * 2654435761)) & 0xFFFFFFFF


def make_param(name: str, shape: tuple, seed: int = 0, std: float = 0.02,
               parity: bool = False) -> np.ndarray:
    """One parameter tensor, float64, deterministic in (name, seed)."""
    rng = np.random.default_rng(_tensor_seed(name, seed))
    short = name.rsplit(".", 1)[-1]
    if short in ("ln1", "ln2", "final_ln"):
        if parity:
            return 1.0 + 0.1 * rng.standard_normal(shape)
        return np.ones(shape)
    if short in ("bq", "bk", "bv"):
        if parity:
            return 0.02 * rng.standard_normal(shape)
        return np.zeros(shape)
    return std * rng.standard_normal(shape)


def make_params(cfg: ModelCfg, seed: int = 0, std: float = 0.02,
                parity: bool = False) -> Dict[str, np.ndarray]:
    out = {}
    for name, shape in param_shapes(cfg).items():
        if not cfg.qkv_bias and name.rsplit(".", 1)[-1] in ("bq", "bk", "bv"):
            continue
        out[name] = make_param(name, shape, seed, std, parity)
    return out


def make_tokens(cfg: ModelCfg, n_micro: int, seed: int = 1234):
    """tokens, targets: int32 [n_micro, seq]; targets are the next tokens."""
    toks = np.empty((n_micro, cfg.seq), np.int32)
    tgts = np.empty((n_micro, cfg.seq), np.int32)
    for b in range(n_micro):
        rng = np.random.default_rng(seed + 1000003 * b)
        seq = rng.integers(0, cfg.vocab, size=cfg.seq + 1, dtype=np.int64)
        toks[b] = seq[:-1]
        tgts[b] = seq[1:]
    return toks, tgts
