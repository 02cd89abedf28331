#!/usr/bin/env bash
# attention backward: dQ drained through smem + bulk (TMA) reductions, dQ MMA before dK:
# parity, kbench A/B (STP_ATTN_DQ_BULK=0/1), ncu of the new kernel, N=1 headline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_vit_ops.py -q -rA -k "attn or attention" > gpurun_out/r02o_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02o_tests.txt | tail -4
for o in 0 1; do
  STP_ATTN_DQ_BULK=$o timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02o_kbench_bulk$o.jsonl 2>&1; echo "kbench bulk$o rc=$?"
  grep -E "attn" gpurun_out/r02o_kbench_bulk$o.jsonl | cut -c1-200
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^attn_bwd_fused" -s 0 -c 1 -o gpurun_out/r02o_ncu_lm_bwd python tools/kbench.py --skip-gemm --skip-elementwise --iters 1 > gpurun_out/r02o_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02o_bench_n1.json 2> gpurun_out/r02o_bench_n1.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02o_bench_n1.json
