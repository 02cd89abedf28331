#!/usr/bin/env bash
# ncu evidence for profiles/ — ONE ncu invocation per gpurun call, and only
# after the same command has exited 0 without ncu in that call:
#   MODE=launches  launch list (device time of every launch)  -> gpurun_out/launches.csv.gz
#   MODE=full      --set full on one kernel (KERNEL regex, KSKIP launches skipped) -> gpurun_out/prof_<name>.ncu-rep
# e.g. gpurun --timeout 900 -- 'MODE=full KERNEL=gemm_bf16_sm100_2sm CMD="python tools/kbench.py --only fc1_fwd --iters 1" bash tools/profile.sh'
set -u
mkdir -p gpurun_out
MODE=${MODE:-launches}
CMD=${CMD:-"python bench.py --steps 1 --warmup 3 --no-cpu"}
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
if [ "$MODE" = launches ]; then
  timeout ${NCU_TIMEOUT:-800} ncu --metrics gpu__time_duration.sum --clock-control none -c "${COUNT:-40000}" --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
  echo "launch list rc=$?"
  gzip -f gpurun_out/launches.csv
else
  K=${KERNEL:?set KERNEL}
  timeout ${NCU_TIMEOUT:-800} ncu --set full --clock-control none --import-source on -k "regex:$K" -s "${KSKIP:-3}" \
      -c "${KCOUNT:-1}" -o "gpurun_out/prof_${K//[^A-Za-z0-9_]/_}" $CMD > "gpurun_out/ncu_full.log" 2>&1
  echo "$K rc=$?"
fi
