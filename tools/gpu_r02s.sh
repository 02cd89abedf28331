#!/usr/bin/env bash
# (historical: STP_ATTN_DP_EARLY was removed after this measurement -- DESIGN.md §7c)
# attention backward MMA issue order A/B: dP(i+1) after dV(i) (default) or right after S(i+1).
mkdir -p gpurun_out
for e in 0 1; do
  STP_ATTN_DP_EARLY=$e timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02s_kbench_dpearly$e.jsonl 2>&1; echo "kbench dp_early=$e rc=$?"
  grep -E "attn_bwd" gpurun_out/r02s_kbench_dpearly$e.jsonl | cut -c1-160
done
STP_ATTN_DP_EARLY=1 timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_vit_ops.py -q -k "attn or attention" > gpurun_out/r02s_tests.txt 2>&1; echo "tests(dp_early=1) rc=$?"; tail -1 gpurun_out/r02s_tests.txt
