#!/usr/bin/env bash
# final 1-GPU batch (last build): full GPU suite, smoke, N=1 headline (cfg2), MLLM cfg5 N=1,
# launch list of one headline step (ncu, per-launch durations; never a bench value).
mkdir -p gpurun_out
TAG=${TAG:-r02z}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest.txt | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err; echo "bench rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_n1.json
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_cfg5_n1.json 2> gpurun_out/${TAG}_bench_cfg5_n1.err; echo "cfg5 rc=$?"; tail -c 200 gpurun_out/${TAG}_bench_cfg5_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/${TAG}_launches_n1.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch list rc=$?"; gzip -f gpurun_out/${TAG}_launches_n1.csv
