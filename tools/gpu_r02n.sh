#!/usr/bin/env bash
# attention backward CTA order (kv-head grouped vs key-tile major over all heads):
# parity, kbench A/B, DRAM bytes per launch (ncu), N=1 headline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_vit_ops.py -q -rA -k "attn or attention" > gpurun_out/r02n_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02n_tests.txt | tail -4
for o in 0 1; do
  STP_ATTN_BWD_ORDER=$o timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02n_kbench_order$o.jsonl 2>&1; echo "kbench order$o rc=$?"
  grep -E "attn" gpurun_out/r02n_kbench_order$o.jsonl | cut -c1-200
  STP_ATTN_BWD_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum --clock-control none -k "regex:^attn_bwd_fused" -s 0 -c 2 --csv python tools/kbench.py --skip-gemm --skip-elementwise --iters 1 > gpurun_out/r02n_ncu_order$o.csv 2> gpurun_out/r02n_ncu_order$o.err; echo "ncu order$o rc=$?"
  grep -E "dram__bytes|duration|red" gpurun_out/r02n_ncu_order$o.csv | cut -c1-300 | tail -8
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02n_bench_n1.json 2> gpurun_out/r02n_bench_n1.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r02n_bench_n1.json
