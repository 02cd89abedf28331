"""Diagnostic: per-tensor bf16 step error vs the fp64 oracle (fp64 weights and
bf16-rounded weights), for one Qwen-shaped configuration."""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import stp_inputs as si  # noqa: E402
from oracle import model as om  # noqa: E402
from paper_2510_27257_b200.stage import Stage  # noqa: E402


def main(seq=256, m=2, layers=2, vocab=4096, h=0, std_milli=50):
    cfg = dataclasses.replace(si.QWEN2_7B, n_layers=layers, seq=seq, vocab=vocab)
    if h:
        cfg = dataclasses.replace(cfg, hidden=h, n_q_heads=8, n_kv_heads=2, ffn=2816)
    P = si.make_params(cfg, seed=5, std=std_milli / 1000, parity=True)
    toks, tgts = si.make_tokens(cfg, m, seed=105)
    loss_ref, G = om.forward_backward(P, cfg, toks, tgts)
    Pr = {k: torch.from_numpy(v).to(torch.bfloat16).double().numpy() for k, v in P.items()}
    loss_r, Gr = om.forward_backward(Pr, cfg, toks, tgts)
    st = Stage(cfg, n_micro=m, dtype="bf16", sched="stp", layers_per_vstage=[1] * layers if layers == 2 else None)
    st.load_params(P)
    loss, _ = st.step(torch.from_numpy(toks).cuda(), torch.from_numpy(tgts).cuda())
    got = st.grads_numpy()
    ref = om.shard_params(G, cfg, 1, 0)
    refr = om.shard_params(Gr, cfg, 1, 0)
    print(cfg, 'std', std_milli / 1000)
    print(f"loss gpu {loss:.6f} oracle {loss_ref:.6f} oracle(bf16 w) {loss_r:.6f}")
    for k in got:
        nr = np.linalg.norm(ref[k])
        print(f"{k:22s} |g|={nr:.3e} rel diff {np.linalg.norm(got[k]-ref[k])/nr:.3e}  vs bf16-w oracle "
              f"{np.linalg.norm(got[k]-refr[k])/np.linalg.norm(refr[k]):.3e}  norm ratio "
              f"{np.linalg.norm(got[k])/nr:.4f}  oracle-vs-oracle {np.linalg.norm(refr[k]-ref[k])/nr:.3e}")
    st.close()


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
