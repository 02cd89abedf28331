#!/usr/bin/env bash
# (historical: STP_ATTN_EXP_EMU was removed after this measurement -- DESIGN.md §7c)
# attention forward with part of the exponentials on the FMA pipe (STP_ATTN_EXP_EMU
# pairs of 8): parity at the default, kbench sweep 0..4, N=1 headline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_vit_ops.py tests/test_gpu_stage.py -q -rA -k "attn or attention or bf16" > gpurun_out/r02r_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02r_tests.txt | tail -4
for e in 0 1 2 3 4; do
  STP_ATTN_EXP_EMU=$e timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02r_kbench_emu$e.jsonl 2>&1; echo "kbench emu$e rc=$?"
  grep -E "attn_fwd" gpurun_out/r02r_kbench_emu$e.jsonl | cut -c1-160
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02r_bench_n1.json 2> gpurun_out/r02r_bench_n1.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02r_bench_n1.json
