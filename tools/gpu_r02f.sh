#!/usr/bin/env bash
# round-2 batch F (1 GPU): graph / offload / GEMM (128x192 tiles) tests, TP4 GEMM kbench,
# N=1 bench eager vs graph.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests/test_gpu_stage.py tests/test_gpu_offload.py tests/test_gpu_gemm.py tests/test_gpu_ops.py -q -rA > gpurun_out/${TAG}_gputest_f.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_f.txt | tail -8
timeout 600 python tools/kbench.py --tp 4 --iters 10 --gemm-mc 1 > gpurun_out/${TAG}_kbench_tp4_b.jsonl 2>&1; echo "kbench rc=$?"
grep -E "qkv|o_fwd" gpurun_out/${TAG}_kbench_tp4_b.jsonl
for g in 0 1; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --graph $g > gpurun_out/${TAG}_bench_n1_graph$g.json 2> gpurun_out/${TAG}_bench_n1_graph$g.err; echo "bench graph=$g rc=$?"; tail -c 150 gpurun_out/${TAG}_bench_n1_graph$g.json; tail -1 gpurun_out/${TAG}_bench_n1_graph$g.err; done
