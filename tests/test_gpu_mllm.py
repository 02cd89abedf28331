"""MLLM whole-step parity on one GPU (SURVEY §8f-f1, cfg5's heterogeneous
first chunk): virtual stage 0 = ViT encoder + 2x2 merger +
text embedding, the LM on the other virtual stages; the C-ABI stage vs the
oracle's MLLM step (oracle/vit.py mllm_forward_backward) on the same seeded
inputs.  Gates as the LM step (tests/stage_parity.py): fp32 loss and every
gradient within relative 1e-4; bf16 loss 2e-2, gradient norms 5e-2 and the
per-tensor difference 3e-2 against the oracle on the same bf16-rounded
parameters and patches.  The executed unit order equals
stp_schedule_units_mllm."""
import numpy as np
import pytest
import torch

from tests import mllm_parity as mp
from tests.stage_parity import compare

pytestmark = pytest.mark.gpu


def _run(cfg, vit, m, dtype, sched, lay, bf16_inputs=False):
    from paper_2510_27257_b200.stage import Stage, schedule_units
    P, PV, patches, full, tgts, ref_loss, G, GV = mp.mllm_reference(cfg, vit, m, bf16_inputs=bf16_inputs)
    st = Stage(cfg, n_micro=m, dtype=dtype, sched=sched, layers_per_vstage=lay, vit=vit)
    st.load_params(P, PV)
    st.bind_images(torch.from_numpy(patches).to(st.torch_dtype).cuda().contiguous())
    loss, stats = st.step(torch.from_numpy(full).cuda(), torch.from_numpy(tgts).cuda())
    got = st.grads_numpy()
    ref = mp.rank_reference(cfg, vit, G, GV, 1, 0)
    assert set(got) == set(ref), sorted(set(got) ^ set(ref))
    trace_ok = st.trace() == schedule_units(sched, 1, m, 1, 0, lay, mllm=True)
    st.close()
    return loss, ref_loss, got, ref, trace_ok


@pytest.mark.parametrize("sched", ["stp", "1f1b-i", "zb", "stp-nobraid", "stp-nosep"])
def test_mllm_fp32_step_matches_oracle(sched):
    cfg, vit = mp.LM_F32, mp.VIT_F32
    loss, ref_loss, got, ref, trace_ok = _run(cfg, vit, 2, "f32", sched, [vit.n_layers, cfg.n_layers])
    bad = compare(cfg, got, ref, loss, ref_loss, "f32")
    assert not bad, bad
    assert trace_ok


def test_mllm_bf16_step_tcgen05_d80():
    cfg, vit = mp.LM_BF16, mp.VIT_BF16
    loss, ref_loss, got, ref, trace_ok = _run(cfg, vit, 2, "bf16", "stp", [vit.n_layers, cfg.n_layers],
                                              bf16_inputs=True)
    bad = compare(cfg, got, ref, loss, ref_loss, "bf16", elementwise=True)
    assert not bad, bad
    assert trace_ok
