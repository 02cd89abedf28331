#!/usr/bin/env bash
# attention forward softmax: tree row max + split row-sum chains; ncu of both
# attention kernels (stall attribution), N=1 headline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_vit_ops.py -q -rA -k "attn or attention" > gpurun_out/r02q_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02q_tests.txt | tail -4
timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02q_kbench.jsonl 2>&1; echo "kbench rc=$?"
grep -E "attn" gpurun_out/r02q_kbench.jsonl | cut -c1-200
KB="python tools/kbench.py --skip-gemm --skip-elementwise --iters 1"
for spec in "attn_fwd_sm100:lm_fwd" "attn_bwd_fused_sm100:lm_bwd"; do
  K=${spec%%:*}; NM=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^${K}" -s 0 -c 1 -o gpurun_out/r02q_ncu_${NM} $KB > gpurun_out/r02q_ncu_${NM}.log 2>&1; echo "ncu $NM rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02q_bench_n1.json 2> gpurun_out/r02q_bench_n1.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02q_bench_n1.json
