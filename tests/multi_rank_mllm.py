"""Run under torchrun: MLLM TP x PP stage parity (ViT + merger on virtual
stage 0, LM on the rest) vs the oracle's MLLM step; each
rank compares its own gradient shards; prints PASS / FAIL per rank."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_27257_b200  # noqa: E402,F401
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from tests import mllm_parity as mp  # noqa: E402
from tests.stage_parity import compare  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, required=True)
    ap.add_argument("--pp", type=int, required=True)
    ap.add_argument("--n-micro", type=int, default=4)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--sched", default="stp")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_27257_b200.stage import Stage, broadcast_nccl_id, schedule_units
    cfg, vit = (mp.LM_F32, mp.VIT_F32) if a.dtype == "f32" else (mp.LM_BF16, mp.VIT_BF16)
    V = 2 * a.pp
    lay = [vit.n_layers] + [1] * (V - 1)
    import dataclasses
    cfg = dataclasses.replace(cfg, n_layers=V - 1, n_kv_heads=max(cfg.n_kv_heads, a.tp))
    P, PV, patches, full, tgts, ref_loss, G, GV = mp.mllm_reference(cfg, vit, a.n_micro,
                                                                    bf16_inputs=a.dtype == "bf16")
    tp_rank, pp_rank = rank % a.tp, rank // a.tp
    st = Stage(cfg, tp=a.tp, pp=a.pp, n_micro=a.n_micro, tp_rank=tp_rank, pp_rank=pp_rank, dtype=a.dtype,
               sched=a.sched, layers_per_vstage=lay, device=local, world_nccl_id=broadcast_nccl_id(), vit=vit)
    st.load_params(P, PV)
    st.bind_images(torch.from_numpy(patches).to(st.torch_dtype).cuda().contiguous())
    loss, _ = st.step(torch.from_numpy(full).cuda(), torch.from_numpy(tgts).cuda())
    got = st.grads_numpy()
    ref = mp.rank_reference(cfg, vit, G, GV, a.tp, tp_rank)
    holds_loss = "lm_head" in got
    bad = compare(cfg, got, {k: ref[k] for k in got}, loss if holds_loss else ref_loss, ref_loss, a.dtype,
                  elementwise=a.dtype == "bf16")
    if st.trace() != schedule_units(a.sched, a.pp, a.n_micro, a.tp, pp_rank, lay, mllm=True):
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
