"""TP x PP parity on 2 / 4 GPUs: launches tests/multi_rank_parity.py under
torchrun (NCCL over NVLink) and requires every rank to match the oracle."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [(2, 1, "stp", "f32"), (1, 2, "stp", "f32"), (2, 1, "stp", "bf16"), (1, 2, "1f1b-i", "f32"),
         (1, 2, "zb", "f32"), (2, 2, "stp", "f32"), (2, 2, "stp", "bf16"), (2, 2, "1f1b-i", "f32"),
         (2, 2, "zb", "f32"), (4, 1, "stp", "f32"), (1, 4, "stp", "f32")]


@pytest.mark.parametrize("tp,pp,sched,dtype", CASES)
def test_multi_rank_parity(tp, pp, sched, dtype):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    seq = 64 if dtype == "bf16" else 32
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + 7 * tp + 3 * pp}",
           os.path.join(ROOT, "tests", "multi_rank_parity.py"), "--tp", str(tp), "--pp", str(pp),
           "--sched", sched, "--dtype", dtype, "--seq", str(seq), "--n-micro", str(2 * pp if sched != "stp" else 4)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=150, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("PASS") == n, out[-4000:]
