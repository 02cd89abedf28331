#!/usr/bin/env bash
# round-2 batch E (1 GPU): graph-replay and offload tests, GEMM kbench at the TP2 / TP4
# per-rank shapes, N=1 bench eager vs CUDA graph, launch list of one N=1 step.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_offload.py -q -rA -k "graph or offload" > gpurun_out/${TAG}_gputest_graph_offload.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_graph_offload.txt | tail -6
for t in 2 4; do timeout 600 python tools/kbench.py --tp $t --iters 10 --gemm-mc 1 > gpurun_out/${TAG}_kbench_tp$t.jsonl 2>&1; echo "kbench tp$t rc=$?"; done
for g in 0 1; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --graph $g > gpurun_out/${TAG}_bench_n1_graph$g.json 2> gpurun_out/${TAG}_bench_n1_graph$g.err; echo "bench graph=$g rc=$?"; tail -c 200 gpurun_out/${TAG}_bench_n1_graph$g.json; done
BC="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6400 --csv --log-file gpurun_out/${TAG}_launches_n1.csv $BC > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"; gzip -f gpurun_out/${TAG}_launches_n1.csv
