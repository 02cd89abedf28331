"""Executor consistency check on 2 / 4 GPUs: the simulator fed
with the measured per-action costs (the action's compute-unit durations plus
the compute-stream gaps spent waiting on its own TP comm phases, i.e. Table 1's
block cost with the exposed T_AR, and the median PP message time as the
latency of every cross-device dependency) reproduces the measured step time
within SURVEY's 5%.  (Compute-only costs under-predict by the exposed TP time:
1.08 / 1.13 for STP / 1F1B-I at TP2 x PP2 in round 2's 4-GPU run.)  The
"span" variant (action span incl. its internal waits + PP message latency) is
reported beside it for information only: a braided action's span already
contains the wait for its backward input from the other device, which the
simulator adds again as a dependency, so it over-counts (measured 0.89 for
STP at 1x2, round 2)."""
import json

import pytest
import torch

from tests.test_gpu_multi import run_torchrun

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tp,pp,sched", [(1, 2, "stp"), (1, 2, "1f1b-i"), (2, 2, "stp"), (2, 2, "1f1b-i")])
def test_executor_matches_simulator(tp, pp, sched):
    n = tp * pp
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    rc, out = run_torchrun(n, ["--tp", str(tp), "--pp", str(pp), "--sched", sched], 29700 + 10 * tp + pp + len(sched),
                           timeout=300, script="multi_rank_timeline.py")
    assert rc == 0, out[-3000:]
    line = json.loads([x for x in out.splitlines() if x.startswith("{")][-1])
    print(line)
    assert 0.95 <= line["ratio_tp"] <= 1.05, line
