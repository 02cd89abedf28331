#!/usr/bin/env bash
# batch L (1 GPU): full GPU suite on the final build, smoke, attention kbench, N=1
# headline bench and the N=1 schedule comparison (costed ZB).
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest_l.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_l.txt | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_l.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke_l.txt
timeout 300 python tools/kbench.py --skip-gemm --iters 10 > gpurun_out/${TAG}_kbench_attn_l.jsonl 2>&1; echo "kbench rc=$?"; head -4 gpurun_out/${TAG}_kbench_attn_l.jsonl
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n1_l.json 2> gpurun_out/${TAG}_bench_n1_l.err; echo "bench rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_n1_l.json
timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu --compare --compare-scheds stp,1f1b-i,zb,stp-mem > gpurun_out/${TAG}_bench_n1_compare_l.json 2> gpurun_out/${TAG}_bench_n1_compare_l.err; echo "compare rc=$?"
