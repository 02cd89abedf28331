#!/usr/bin/env bash
# batch I (1 GPU): GEMM / stage parity with the 256-bit epilogue, kbench TP1 / TP4 GEMMs, N=1 bench.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_ops.py tests/test_gpu_stage.py tests/test_gpu_fullsize.py -q -rA > gpurun_out/${TAG}_gputest_i.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_i.txt | tail -6
for t in 1 4; do timeout 600 python tools/kbench.py --tp $t --iters 10 --gemm-mc 1 --skip-attn 2>/dev/null > gpurun_out/${TAG}_kbench_gemm_tp$t.jsonl || timeout 600 python tools/kbench.py --tp $t --iters 10 --gemm-mc 1 > gpurun_out/${TAG}_kbench_gemm_tp$t.jsonl 2>&1; echo "kbench tp$t rc=$?"; done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n1_i.json 2> gpurun_out/${TAG}_bench_n1_i.err; echo "bench rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_n1_i.json
