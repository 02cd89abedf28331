"""Overlap-contention calibration (SURVEY §8d.4 "App. F analogue": GEMM || RS/AG
on B200).  PAPER.md App. F (Table 11) measures how much a GEMM slows down when
a TP collective runs beside it (9.251 / 8.605 = 1.075 on A800); the braid's
gain is bounded by that factor.  Here, per rank of a TP group of N = world
GPUs, at the Qwen2-7B unit shapes (seq 6144, TP = N):

  gemm_alone    the forward MLP unit's GEMMs (FC1 + FC2) on stream A
  comm_alone    RS + AG of one [s, h] bf16 activation on stream B
  overlapped    both at once; contention = gemm_overlapped / gemm_alone,
                comm_slowdown = comm_overlapped / comm_alone

for NCCL with several CTA caps (ncclConfig_t.maxCTAs; 0 = NCCL default) and,
when available, torch's copy-engine ("low contention") AG/RS.  Times are
CUDA events on the launching streams, max over ranks.  Measurement tool only:
not on the product path.

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/contention.py [--ctas 0,16,8,4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_27257_b200  # noqa: E402,F401  (sets CUDA_DEVICE_MAX_CONNECTIONS)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_27257_b200 import ops  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


class Clocks:
    """Median SM clock (MHz) and board power (W) of this rank's GPU while a
    measured region runs (NVML, 10 ms period)."""

    def __init__(self, index):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nv = None
        self.threading = threading

    def __enter__(self):
        self.samples, self.stop = [], False

        def run():
            while not self.stop and self.nv:
                try:
                    self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                         self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
                except Exception:
                    break
                import time
                time.sleep(0.01)
        self.th = self.threading.Thread(target=run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *exc):
        self.stop = True
        self.th.join()

    def median(self):
        if not self.samples:
            return None, None
        c = sorted(x[0] for x in self.samples)
        w = sorted(x[1] for x in self.samples)
        return c[len(c) // 2], w[len(w) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", default="0,32,16,8,4")
    ap.add_argument("--seq", type=int, default=6144)
    ap.add_argument("--gemm-iters", type=int, default=20)
    ap.add_argument("--ce", action="store_true", help="also try torch symmetric-memory copy-engine AG/RS")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    t, s, h, I = world, a.seq, 3584, 18944 // world
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(rank)
    xn = torch.randn(s, h, generator=g, device=dev).to(bf)
    wgu = torch.randn(2 * I, h, generator=g, device=dev).to(bf) * 0.02
    gu = torch.empty(s, 2 * I, device=dev, dtype=bf)
    hh = torch.randn(s, I, generator=g, device=dev).to(bf)
    wd = torch.randn(h, I, generator=g, device=dev).to(bf) * 0.02
    part = torch.empty(s, h, device=dev, dtype=bf)
    full = torch.randn(s, h, generator=g, device=dev).to(bf)
    shard = torch.randn(s // t, h, generator=g, device=dev).to(bf)
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    clk = Clocks(torch.cuda.current_device())

    def gemm_loop(n):
        for _ in range(n):
            ops.gemm(0, xn, wgu, gu, s, 2 * I, h, epi=0, dtype=1)
            ops.gemm(0, hh, wd, part, s, h, I, epi=0, dtype=1)

    def run(stream, fn, n):
        with torch.cuda.stream(stream):
            e0, e1 = ev(), ev()
            e0.record()
            fn(n)
            e1.record()
        return e0, e1

    def maxr(x):
        v = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def measure(name, comm_fn):
        # comm alone (per RS+AG pair)
        for _ in range(3):
            comm_fn(1)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = run(sB, comm_fn, 10)
        torch.cuda.synchronize()
        comm_alone = maxr(e0.elapsed_time(e1) / 10)
        gemm_loop(2)
        torch.cuda.synchronize()
        with clk as c_alone:
            e0, e1 = run(sA, gemm_loop, a.gemm_iters)
            torch.cuda.synchronize()
        gemm_alone = maxr(e0.elapsed_time(e1))
        n_comm = max(4, int(1.4 * gemm_alone / comm_alone) + 1)
        dist.barrier()
        torch.cuda.synchronize()
        with clk as c_ov:
            c0, c1 = run(sB, comm_fn, n_comm)
            g0, g1 = run(sA, gemm_loop, a.gemm_iters)
            torch.cuda.synchronize()
        gemm_ov = maxr(g0.elapsed_time(g1))
        comm_ov = maxr(c0.elapsed_time(c1) / n_comm)
        flops = a.gemm_iters * 2 * s * h * 3 * I  # FC1 (N = 2I) + FC2 (K = I)
        rec = {"variant": name, "tp": t, "seq": s, "comm_alone_ms": comm_alone, "comm_overlapped_ms": comm_ov,
               "comm_busbw_alone_GBps": 2 * (t - 1) / t * s * h * 2 / comm_alone / 1e6,
               "gemm_alone_ms": gemm_alone, "gemm_overlapped_ms": gemm_ov,
               "gemm_alone_tflops": flops / gemm_alone / 1e9,
               "contention": gemm_ov / gemm_alone, "comm_slowdown": comm_ov / comm_alone,
               "rank0_sm_mhz_power_w": {"gemm_alone": c_alone.median(), "overlapped": c_ov.median()}}
        if rank == 0:
            print(json.dumps(rec), flush=True)

    for c in [int(x) for x in a.ctas.split(",")]:
        opts = dist.ProcessGroupNCCL.Options()
        if c > 0:
            opts.config.max_ctas = c
            opts.config.min_ctas = min(c, 2)
        pg = dist.new_group(list(range(world)), backend="nccl", pg_options=opts)

        def nccl_pair(n, pg=pg):
            for _ in range(n):
                dist.reduce_scatter_tensor(shard, full, group=pg)
                dist.all_gather_into_tensor(full, shard, group=pg)

        measure(f"nccl_ctas{c if c else 'default'}", nccl_pair)

    if a.ce:
        try:
            import torch.distributed._symmetric_memory as symm
            grp = dist.group.WORLD
            symm.enable_symm_mem_for_group(grp.group_name)
            buf = symm.empty(s, h, device=dev, dtype=bf)
            symm.rendezvous(buf, grp.group_name)
            buf.copy_(full)
            sh = buf[: s // t]

            def ce_pair(n):
                for _ in range(n):
                    torch.ops.symm_mem._low_contention_reduce_scatter(buf, "sum", grp.group_name)
                    torch.ops.symm_mem._low_contention_all_gather(sh, grp.group_name)

            measure("torch_symm_mem_copy_engine", ce_pair)
        except Exception as e:  # measurement probe only
            if rank == 0:
                print(json.dumps({"variant": "torch_symm_mem_copy_engine", "error": repr(e)[:300]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
