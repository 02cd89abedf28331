"""TP x PP parity on 2 / 4 GPUs: launches tests/multi_rank_parity.py under
torchrun (NCCL over NVLink) and requires every rank to match the oracle.
On timeout the whole process group is killed (no rank keeps spinning on a
GPU after the test)."""
import os
import signal
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [(2, 1, "stp", "f32"), (1, 2, "stp", "f32"), (2, 1, "stp", "bf16"), (1, 2, "1f1b-i", "f32"),
         (1, 2, "stp-mem", "f32"), (2, 2, "stp-mem", "f32"),
         (1, 2, "zb", "f32"), (1, 2, "stp-nobraid", "f32"), (2, 2, "stp", "f32"), (2, 2, "stp", "bf16"),
         (2, 2, "1f1b-i", "f32"), (2, 2, "zb", "f32"), (4, 1, "stp", "f32"), (1, 4, "stp", "f32")]


def run_torchrun(n, args, port, timeout=120, script="multi_rank_parity.py", env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", script)] + args
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, cwd=ROOT,
                         start_new_session=True, env=dict(os.environ, **(env or {})))
    try:
        out, _ = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, _ = p.communicate()
        return -9, out
    return p.returncode, out


@pytest.mark.parametrize("tp,pp,sched,dtype", CASES)
def test_multi_rank_parity(tp, pp, sched, dtype):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    seq = 64 if dtype == "bf16" else 32
    args = ["--tp", str(tp), "--pp", str(pp), "--sched", sched, "--dtype", dtype, "--seq", str(seq),
            "--n-micro", str(2 * pp if sched != "stp" else 4)]
    rc, out = run_torchrun(n, args, 29500 + 7 * tp + 3 * pp + len(sched))
    assert rc == 0, out[-4000:]
    assert out.count("PASS") == n, out[-4000:]


# Every TP transport explicitly (CASES above run each schedule's default: "ce"
# for the braided STP family, "p2p" otherwise): "p2p" = one fused kernel per
# comm phase, NVLink loads of the peers' partials, residual + RMSNorm (bwd),
# NVLink stores of the all-gather; "ce" = copy-engine NVLink pulls + fused
# RS-sum / residual / RMSNorm kernel; "nccl" = NCCL reduce-scatter /
# all-gather (the baseline transport).
CE_CASES = [(2, 1, "stp", "f32"), (2, 1, "stp", "bf16"), (4, 1, "stp", "f32"), (4, 1, "1f1b-i", "bf16"),
            (2, 2, "stp", "f32"), (2, 2, "1f1b-i", "f32")]


@pytest.mark.parametrize("transport", ["p2p", "ce", "nccl"])
@pytest.mark.parametrize("tp,pp,sched,dtype", CE_CASES)
def test_multi_rank_parity_symmetric(tp, pp, sched, dtype, transport):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    seq = 64 if dtype == "bf16" else 32
    args = ["--tp", str(tp), "--pp", str(pp), "--sched", sched, "--dtype", dtype, "--seq", str(seq),
            "--n-micro", str(2 * pp if sched != "stp" else 4)]
    rc, out = run_torchrun(n, args, 29700 + 7 * tp + 3 * pp + len(sched) + len(dtype) + 50 * (transport == "nccl")
                           + 100 * (transport == "p2p"),
                           env={"STP_TP_TRANSPORT": transport})
    assert rc == 0, out[-4000:]
    assert out.count("PASS") == n, out[-4000:]


# MLLM (ViT + merger on virtual stage 0) over TP x PP; the ViT comm
# phases run on NCCL (STP_TP_TRANSPORT=nccl, include/stp.h).
MLLM_CASES = [(2, 1, "stp", "f32"), (1, 2, "stp", "f32"), (2, 2, "stp", "f32"), (2, 2, "stp", "bf16"),
              (2, 2, "1f1b-i", "f32")]


@pytest.mark.parametrize("tp,pp,sched,dtype", MLLM_CASES)
def test_multi_rank_mllm_parity(tp, pp, sched, dtype):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    args = ["--tp", str(tp), "--pp", str(pp), "--sched", sched, "--dtype", dtype, "--n-micro", str(2 * pp)]
    rc, out = run_torchrun(n, args, 29900 + 7 * tp + 3 * pp + len(sched) + len(dtype), script="multi_rank_mllm.py",
                           env={"STP_TP_TRANSPORT": "nccl"})
    assert rc == 0, out[-4000:]
    assert out.count("PASS") == n, out[-4000:]


# p2p transport with the reduce-scatter's transfer fused into the row-parallel
# GEMMs' epilogues (STP_P2P_PUSH=1: each rank's O / FC2 / dgrad GEMM stores row
# block q of its partial into TP peer q's partial buffer over NVLink).
PUSH_CASES = [(2, 1, "stp", "bf16"), (2, 2, "stp", "bf16"), (4, 1, "stp", "bf16"), (4, 1, "1f1b-i", "bf16"),
              (2, 2, "zb", "bf16")]


@pytest.mark.parametrize("tp,pp,sched,dtype", PUSH_CASES)
def test_multi_rank_parity_gemm_push(tp, pp, sched, dtype):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    args = ["--tp", str(tp), "--pp", str(pp), "--sched", sched, "--dtype", dtype, "--seq", "64",
            "--n-micro", str(2 * pp if sched != "stp" else 4)]
    rc, out = run_torchrun(n, args, 30100 + 7 * tp + 3 * pp + len(sched),
                           env={"STP_P2P_PUSH": "1", "STP_TP_TRANSPORT": "p2p"})
    assert rc == 0, out[-4000:]
    assert out.count("PASS") == n, out[-4000:]
