"""smoke(): one tiny STP train step (TP=1, PP=1, two virtual stages, the
R-STP braided schedule, fp32) on cuda:0 through the C-ABI library, checked
against the CPU oracle (loss and every gradient, rel 1e-4)."""
import torch

import stp_inputs as si


def run():
    from paper_2510_27257_b200.stage import Stage
    from tests.stage_parity import compare, oracle_reference, rank_grads_ref
    assert torch.cuda.is_available(), "smoke() needs a GPU"
    cfg = si.TINY
    m = 4
    P, toks, tgts, ref_loss, G = oracle_reference(cfg, m)
    st = Stage(cfg, n_micro=m, dtype="f32", sched="stp", device=0)
    st.load_params(P)
    dt = torch.from_numpy(toks).cuda()
    dg = torch.from_numpy(tgts).cuda()
    loss, stats = st.step(dt, dg)
    bad = compare(cfg, st.grads_numpy(), rank_grads_ref(cfg, G, 1, 0), loss, ref_loss, "f32")
    st.close()
    if bad:
        raise AssertionError("smoke parity failed: " + "; ".join(bad[:5]))
    print(f"smoke ok: loss {loss:.6f} (oracle {ref_loss:.6f}), {stats.n_units} units, {stats.n_kernels} kernels")
