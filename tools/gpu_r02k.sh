#!/usr/bin/env bash
# batch K (1 GPU): attention / ViT / full-size / stage / MLLM parity with the d-major dQ
# accumulator, attention kbench, smoke, N=1 headline bench.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest_k.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_k.txt | tail -6
timeout 300 python tools/kbench.py --skip-gemm --iters 10 > gpurun_out/${TAG}_kbench_attn_k.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/${TAG}_kbench_attn_k.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_k.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke_k.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n1_k.json 2> gpurun_out/${TAG}_bench_n1_k.err; echo "bench rc=$?"; tail -c 400 gpurun_out/${TAG}_bench_n1_k.json
