#!/usr/bin/env bash
# round-2 batch B: offload / stp-mem / CE-epilogue tests, full single-GPU suite,
# N=1 bench with the schedule comparison (incl. stp-mem and stp with offload).
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest_n1_b.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_n1_b.txt | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_b.txt 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py --steps 5 --warmup 3 --compare --compare-scheds stp,1f1b-i,1f1b-i-naive,zb,stp-mem,stp@0.5 > gpurun_out/${TAG}_bench_n1_compare.json 2> gpurun_out/${TAG}_bench_n1_compare.err; echo "bench rc=$?"
tail -c 400 gpurun_out/${TAG}_bench_n1_compare.json; tail -2 gpurun_out/${TAG}_bench_n1_compare.err
