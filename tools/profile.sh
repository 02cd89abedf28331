#!/usr/bin/env bash
# ncu evidence for profiles/ (run under gpurun on ONE GPU, after the same
# bench command exited 0 without ncu in this call):
#   1. launch list (every launch of one timed step, device time) -> launches.csv
#   2. --set full on the top kernels (GEMM, attention fwd/bwd)  -> *.ncu-rep
set -u
mkdir -p gpurun_out
CMD=${CMD:-"python bench.py --steps 1 --warmup 3 --no-cpu"}
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
tail -1 gpurun_out/plain.log
# launches per step (for -s: skip init + warm-up launches)
SKIP=${SKIP:-0}
COUNT=${COUNT:-6000}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s "$SKIP" -c "$COUNT" --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for K in ${KERNELS:-gemm_bf16_sm100 attn_fwd_sm100 attn_bwd_dkdv_sm100 attn_bwd_dq_sm100}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${KSKIP:-40} -c 1 \
      -o "gpurun_out/prof_$K" $CMD > "gpurun_out/ncu_$K.log" 2>&1
  echo "$K rc=$?"
done
