#!/usr/bin/env bash
# final 1-GPU batch: full GPU suite, smoke, N=1 headline bench (cfg2) and MLLM cfg5 N=1.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest_final.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_final.txt | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_final.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke_final.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n1_headline.json 2> gpurun_out/${TAG}_bench_n1_headline.err; echo "bench rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_n1_headline.json
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_cfg5_n1_final.json 2> gpurun_out/${TAG}_bench_cfg5_n1_final.err; echo "cfg5 rc=$?"; tail -c 200 gpurun_out/${TAG}_bench_cfg5_n1_final.json
