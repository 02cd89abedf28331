"""Per-unit timing of one training step on a TP x PP grid (run under torchrun):
mean / median CUDA-event duration of every unit kind (compute units by op, TP
comm phases split into RS+AG / AG-only / RS-only by direction), measured on
the stage's own streams in timing mode.  The comm phases are compared with the
NVLink bound: a phase moves (t-1)/t * s*h*2 bytes per collective per rank, at
900 GB/s per direction.  Diagnostic tool (not the bench).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/comm_phase_times.py --tp 4 --pp 1
"""
import argparse
import dataclasses
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_27257_b200  # noqa: E402,F401
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import stp_inputs as si  # noqa: E402

OPS = {0: "F_ATTN", 1: "F_MLP", 2: "B_MLP", 3: "B_ATTN", 4: "W_MLP", 5: "W_ATTN", 6: "CF", 7: "CB", 8: "F_EMB",
       9: "W_EMB", 10: "F_HEAD", 11: "B_HEAD", 12: "W_HEAD", 13: "PP_SEND", 14: "PP_RECV"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, required=True)
    ap.add_argument("--pp", type=int, default=1)
    ap.add_argument("--sched", default="stp")
    ap.add_argument("--n-micro", type=int, default=8)
    ap.add_argument("--layers", type=int, default=28)
    ap.add_argument("--seq", type=int, default=6144)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_27257_b200.stage import Stage, broadcast_nccl_id
    cfg = dataclasses.replace(si.QWEN2_7B, n_layers=a.layers, seq=a.seq)
    tp_rank, pp_rank = rank % a.tp, rank // a.tp
    st = Stage(cfg, tp=a.tp, pp=a.pp, n_micro=a.n_micro, tp_rank=tp_rank, pp_rank=pp_rank, dtype="bf16",
               sched=a.sched, device=local, world_nccl_id=broadcast_nccl_id())
    g = torch.Generator(device="cuda").manual_seed(rank)
    for name, prm in zip(st.names, st.params):
        if name.endswith(("ln1", "ln2")) or name == "final_ln":
            prm.fill_(1.0)
        else:
            prm.copy_(torch.randn(prm.shape, generator=g, device="cuda") * 0.02)
    toks, tgts = si.make_tokens(cfg, a.n_micro)
    dt, dg = torch.from_numpy(toks).cuda(), torch.from_numpy(tgts).cuda()
    for _ in range(2):
        st.step(dt, dg)
    st.set_timing(True)
    _, stats = st.step(dt, dg)
    t0, t1 = st.unit_times()
    units = st.trace()
    kinds = {}
    for u, a0, a1 in zip(units, t0, t1):
        op = OPS.get(u[2], str(u[2]))
        if op in ("CF", "CB"):
            op = f"{op}_k0" if u[3] == 0 else op
        kinds.setdefault(op, []).append(a1 - a0)
    if rank == 0:
        bytes_coll = (a.tp - 1) / a.tp * a.seq * cfg.hidden * 2
        out = {"tp": a.tp, "pp": a.pp, "sched": a.sched, "seq": a.seq, "layers": a.layers,
               # the stage's default rule (stage.cu init): ce for the braided schedules
               "transport": os.environ.get("STP_TP_TRANSPORT", "ce" if a.sched in ("stp", "stp-nosep") else "p2p"),
               "step_ms": stats.step_ms,
               "exposed_tp_ms": stats.exposed_tp_ms, "pp_bubble_ms": stats.pp_bubble_ms,
               "nvlink_bound_ms_per_collective": bytes_coll / 900e9 * 1e3,
               "units": {k: {"n": len(v), "mean_ms": statistics.mean(v), "median_ms": statistics.median(v)}
                         for k, v in sorted(kinds.items())}}
        print(json.dumps(out), flush=True)
    st.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
