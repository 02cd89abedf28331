"""Run under torchrun (one rank per GPU): TP x PP stage parity vs the CPU
oracle.  Each rank compares its own gradient shards (oracle.shard_params of
the unsharded fp64 gradients) and, on the rank(s) holding the last virtual
stage, the loss; prints PASS/FAIL per rank and exits non-zero on failure."""
import argparse
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_27257_b200  # noqa: E402,F401  (sets CUDA_DEVICE_MAX_CONNECTIONS before CUDA init)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import stp_inputs as si  # noqa: E402
from tests.stage_parity import compare, oracle_reference, rank_grads_ref  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, required=True)
    ap.add_argument("--pp", type=int, required=True)
    ap.add_argument("--n-micro", type=int, default=4)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--sched", default="stp")
    ap.add_argument("--seq", type=int, default=32)
    ap.add_argument("--layers", type=str, default="")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == a.tp * a.pp
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_27257_b200.stage import Stage, broadcast_nccl_id
    cfg = dataclasses.replace(si.TINY, seq=a.seq, n_kv_heads=max(2, a.tp), ffn=176 if a.tp <= 2 else 192)
    lay = [int(x) for x in a.layers.split(",")] if a.layers else [1] * (2 * a.pp if a.sched != "1f1b" else a.pp)
    cfg = dataclasses.replace(cfg, n_layers=sum(lay))
    P, toks, tgts, ref_loss, G = oracle_reference(cfg, a.n_micro)
    tp_rank, pp_rank = rank % a.tp, rank // a.tp
    uid = broadcast_nccl_id()
    st = Stage(cfg, tp=a.tp, pp=a.pp, n_micro=a.n_micro, tp_rank=tp_rank, pp_rank=pp_rank, dtype=a.dtype, sched=a.sched,
               layers_per_vstage=lay, device=local, world_nccl_id=uid)
    st.load_params(P)
    loss, stats = st.step(torch.from_numpy(toks).cuda(), torch.from_numpy(tgts).cuda())
    got = st.grads_numpy()
    ref = rank_grads_ref(cfg, G, a.tp, tp_rank)
    holds_loss = "lm_head" in got
    bad = compare(cfg, got, ref, loss if holds_loss else ref_loss, ref_loss, a.dtype)
    # the executed unit order equals the schedule's unit order
    from paper_2510_27257_b200.stage import schedule_units
    if st.trace() != schedule_units(a.sched, a.pp, a.n_micro, a.tp, pp_rank, lay):
        bad.append("trace != schedule units")
    st.close()
    flag = torch.tensor([len(bad)], device="cuda")
    dist.all_reduce(flag)
    print(f"rank {rank} (tp {tp_rank} pp {pp_rank}) {'PASS' if not bad else 'FAIL ' + '; '.join(bad[:4])} "
          f"loss {loss:.6f} ref {ref_loss:.6f}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if flag.item() else 0)


if __name__ == "__main__":
    main()
