#!/usr/bin/env bash
# round-2 batch G (1 GPU): graph / offload / GEMM tests, N=1 eager vs graph, ncu of the
# short-K O-projection GEMM at TP4 shapes, launch list of one full N=1 step.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests/test_gpu_stage.py tests/test_gpu_offload.py tests/test_gpu_gemm.py -q -rA > gpurun_out/${TAG}_gputest_g.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_g.txt | tail -6
for g in 0 1; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --graph $g > gpurun_out/${TAG}_bench_n1_graph$g.json 2> gpurun_out/${TAG}_bench_n1_graph$g.err; echo "bench graph=$g rc=$?"; tail -c 150 gpurun_out/${TAG}_bench_n1_graph$g.json; tail -1 gpurun_out/${TAG}_bench_n1_graph$g.err; done
KB="python tools/kbench.py --tp 4 --iters 1 --gemm-mc 1 --only o_fwd"
$KB > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemm_bf16" -s 3 -c 1 -o gpurun_out/${TAG}_ncu_gemm_o_fwd_tp4 $KB > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
BC="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 7300 --csv --log-file gpurun_out/${TAG}_launches_n1.csv $BC > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"; gzip -f gpurun_out/${TAG}_launches_n1.csv
