"""smoke(): three small STP train steps on cuda:0 through the C-ABI library,
each checked against the CPU fp64 oracle:
  1. TINY fp32 (TP=1, PP=1, two virtual stages, R-STP braided schedule):
     loss and every gradient, rel 1e-4;
  2. one bf16 step on a Qwen-style model with head_dim 128 (2 layers, h 1024,
     8 q / 2 kv heads, I 2816, s 512, V 4096), which runs the default tcgen05
     kernels (2-SM / 1-SM GEMMs, tcgen05 attention forward and fused
     backward): loss rel 2e-2, grad norms 5e-2, per-tensor difference 3e-2
     against the oracle on the same bf16-rounded parameters (N(0, 0.02^2));
  3. one bf16 MLLM step (ViT with d = 80 heads + 2x2 merger on virtual stage
     0, small LM on virtual stage 1): the ViT kernels (LayerNorm, QuickGELU /
     GELU, 2-D RoPE, bidirectional tcgen05 attention) against the oracle's
     MLLM step (oracle/vit.py), same gates.
"""
import dataclasses

import torch

import stp_inputs as si


def _one(cfg, m, dtype, lay=None, **kw):
    from paper_2510_27257_b200.stage import Stage
    from tests.stage_parity import compare, oracle_reference, rank_grads_ref
    P, toks, tgts, ref_loss, G = oracle_reference(cfg, m, **kw)
    st = Stage(cfg, n_micro=m, dtype=dtype, sched="stp", device=0, layers_per_vstage=lay)
    st.load_params(P)
    dt = torch.from_numpy(toks).cuda()
    dg = torch.from_numpy(tgts).cuda()
    loss, stats = st.step(dt, dg)
    bad = compare(cfg, st.grads_numpy(), rank_grads_ref(cfg, G, 1, 0), loss, ref_loss, dtype,
                  elementwise=kw.get("bf16_inputs", False))
    st.close()
    if bad:
        raise AssertionError(f"smoke parity failed ({dtype}): " + "; ".join(bad[:5]))
    print(f"smoke ok ({dtype}): loss {loss:.6f} (oracle {ref_loss:.6f}), {stats.n_units} units, "
          f"{stats.n_kernels} kernels")


def run():
    assert torch.cuda.is_available(), "smoke() needs a GPU"
    _one(si.TINY, 4, "f32")
    qcfg = dataclasses.replace(si.QWEN2_7B, hidden=1024, n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128,
                               ffn=2816, seq=512, vocab=4096)
    _one(qcfg, 2, "bf16", lay=[1, 1], std=0.02, bf16_inputs=True)
    _mllm()


def _mllm():
    from paper_2510_27257_b200.stage import Stage
    from tests import mllm_parity as mp
    from tests.stage_parity import compare
    cfg, vit, m = mp.LM_BF16, mp.VIT_BF16, 2
    P, PV, patches, full, tgts, ref_loss, G, GV = mp.mllm_reference(cfg, vit, m, bf16_inputs=True)
    st = Stage(cfg, n_micro=m, dtype="bf16", sched="stp", device=0, layers_per_vstage=[vit.n_layers, cfg.n_layers],
               vit=vit)
    st.load_params(P, PV)
    st.bind_images(torch.from_numpy(patches).to(torch.bfloat16).cuda().contiguous())
    loss, stats = st.step(torch.from_numpy(full).cuda(), torch.from_numpy(tgts).cuda())
    bad = compare(cfg, st.grads_numpy(), mp.rank_reference(cfg, vit, G, GV, 1, 0), loss, ref_loss, "bf16",
                  elementwise=True)
    st.close()
    if bad:
        raise AssertionError("smoke MLLM parity failed: " + "; ".join(bad[:5]))
    print(f"smoke ok (bf16 MLLM, ViT d=80): loss {loss:.6f} (oracle {ref_loss:.6f}), {stats.n_units} units, "
          f"{stats.n_kernels} kernels")
