"""Run under torchrun: one timed STP step on a TP x PP grid, every rank's
per-unit CUDA-event times gathered to rank 0, then the executor-consistency
check of SURVEY §8d.4: the oracle's discrete-event simulator, fed the measured
time of every action (ratio: compute units only; ratio_span: the action's
span on the compute stream, i.e. its units plus the TP-comm waits between
them, and the median PP message time as the latency of every cross-device
dependency), must reproduce the measured step time.  A large
gap means a hidden synchronisation / serialisation in the executor.  Prints
one JSON line on rank 0."""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_27257_b200  # noqa: E402,F401
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import stp_inputs as si  # noqa: E402
from oracle import schedule as sc  # noqa: E402
from oracle import simulate as sm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, required=True)
    ap.add_argument("--pp", type=int, required=True)
    ap.add_argument("--sched", default="stp")
    ap.add_argument("--n-micro", type=int, default=8)
    ap.add_argument("--layers", type=int, default=10)
    ap.add_argument("--seq", type=int, default=2048)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_27257_b200.stage import SCHED, Stage, broadcast_nccl_id
    cfg = dataclasses.replace(si.QWEN2_7B, n_layers=a.layers, seq=a.seq, vocab=32768)
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
    gathered = [None] * world
    dist.all_gather_object(gathered, (pp_rank, tp_rank, units, t0, t1, stats.step_ms, stats.exposed_tp_ms,
                                      stats.pp_bubble_ms))
    if rank == 0:
        kind = SCHED[a.sched]
        progs = sc.build_program(kind, a.pp, a.n_micro)
        dur, span, busy_tp, pp_msgs = [], [], [], []
        measured = max(x[5] for x in gathered)
        for d in range(a.pp):
            pr, tr, us, s0, s1, *_ = next(x for x in gathered if x[0] == d and x[1] == 0)
            per = [0.0] * len(progs[d])
            first = [None] * len(progs[d])
            last = [0.0] * len(progs[d])
            for u, b, e in zip(us, s0, s1):
                if u[1] == 0:                    # compute-stream units
                    per[u[0]] += e - b
                    first[u[0]] = b if first[u[0]] is None else first[u[0]]
                    last[u[0]] = e
                elif u[2] == 13:                 # STP_U_PP_SEND: one PP message
                    pp_msgs.append(e - b)
            dur.append(per)
            # compute + exposed TP per action: the compute-stream gaps the
            # executor classifies as TP waits (a compute unit waiting on a comm
            # phase that itself is not waiting on a PP message; stage.cu
            # run_step) belong to the action's cost, as T_AR does in Table 1's
            # block costs; waits for PP inputs do not (the simulator adds them)
            bt = list(per)
            prev_end = 0.0
            first_u = True
            for i_u, (u, b, e) in enumerate(zip(us, s0, s1)):
                if u[1] != 0:
                    continue
                gap = b if first_u else b - prev_end
                if gap > 0 and u[6] >= 0 and us[u[6]][1] == 1:
                    c = us[u[6]]
                    waits_pp = c[6] >= 0 and us[c[6]][1] == 2 and s1[c[6]] > prev_end
                    if not waits_pp and s1[u[6]] > prev_end:
                        bt[u[0]] += gap
                prev_end = max(prev_end, e)
                first_u = False
            busy_tp.append(bt)
            # action span on the compute stream: its units plus the TP-comm waits
            # between them (exposed TP inside the action)
            span.append([(l - f) if f is not None else 0.0 for f, l in zip(first, last)])
        lat = sorted(pp_msgs)[len(pp_msgs) // 2] if pp_msgs else 0.0
        simulated = sm.simulate_durations(kind, a.pp, progs, dur)
        simulated_span = sm.simulate_durations(kind, a.pp, progs, span, pp_latency=lat)
        simulated_tp = sm.simulate_durations(kind, a.pp, progs, busy_tp, pp_latency=lat)
        print(json.dumps({"tp": a.tp, "pp": a.pp, "sched": a.sched, "n_micro": a.n_micro, "layers": a.layers,
                          "seq": a.seq, "measured_ms": measured, "simulated_ms": simulated,
                          "ratio": measured / simulated,
                          "simulated_span_ms": simulated_span, "pp_msg_ms_median": lat,
                          "ratio_span": measured / simulated_span,
                          "simulated_tp_ms": simulated_tp, "ratio_tp": measured / simulated_tp,
                          "exposed_tp_pct": [100 * x[6] / x[5] for x in gathered],
                          "pp_bubble_pct": [100 * x[7] / x[5] for x in gathered]}), flush=True)
    st.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
