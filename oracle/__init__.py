"""CPU oracle for the STP hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_2510_27257_b200/`, the C-ABI library) never imports, links or
calls it, and this package imports nothing from the product path: the two
share only `stp_inputs` (seeded generators with none of the method's
arithmetic).

Contents
  model.py     unsharded fp64 Qwen2-style forward / hand-derived backward with
               microbatch gradient accumulation, plus an
               in-process TP/SP sharded emulation (AG = concat, RS = sum+slice)
               following PAPER.md Eq. 1-2 in the SP reading Q10.
  schedule.py  the schedule builders (R-STP reading of PAPER.md §4.2
               P:L117-122 + App. A; Megatron 1F1B-I; plain 1F1B;
               ZB-V-style greedy) and the unit expansion of the braided
               execution blocks (Fig. 3), with the canonical text
               serialisation.
  simulate.py  discrete-event simulator that evaluates a program under the
               Table 1 cost model: makespan, PP bubble, exposed
               TP communication, peak in-flight activations.

Parity pins (what fixes each function other than itself) are in
tests/test_oracle_*.py; see DESIGN.md "Oracle pins".  Functions without an
external pin are listed there as "parity unpinned".
"""
