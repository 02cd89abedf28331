#!/usr/bin/env bash
# attention kernels with shared-space LDS / STS (no generic LD / ST): parity,
# kbench, N=1 headline (compute-sanitizer is closed on the GPU pool).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_vit_ops.py -q -rA -k "attn or attention" > gpurun_out/r02p_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02p_tests.txt | tail -4
timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02p_kbench.jsonl 2>&1; echo "kbench rc=$?"
grep -E "attn" gpurun_out/r02p_kbench.jsonl | cut -c1-200
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02p_bench_n1.json 2> gpurun_out/r02p_bench_n1.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02p_bench_n1.json
