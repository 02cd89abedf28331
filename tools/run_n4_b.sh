#!/usr/bin/env bash
# 4-GPU batch D: push-mode / stp-mem / consistency tests; cfg2 TP4 schedule
# comparison with and without the GEMM-epilogue push; comm-phase unit times
# (NVLink fraction table).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_consistency.py -k "push or stp-mem or consistency or executor" -q -rA > gpurun_out/${TAG}_gputest_n4_b.txt 2>&1
tail -2 gpurun_out/${TAG}_gputest_n4_b.txt
for push in 0 1; do
  STP_P2P_PUSH=$push timeout 1200 $RUN --master-port 2967$push bench.py --gpus 4 --config cfg2 --steps 5 --warmup 3 --no-cpu --compare \
    --compare-scheds stp,1f1b-i,1f1b-i-naive,stp-mem > gpurun_out/${TAG}_bench_n4_cfg2_push$push.json 2> gpurun_out/${TAG}_bench_n4_cfg2_push$push.err
  echo "push=$push rc=$?"; tail -1 gpurun_out/${TAG}_bench_n4_cfg2_push$push.err
done
for push in 0 1; do
  for sched in stp 1f1b-i-naive; do
    STP_P2P_PUSH=$push timeout 600 $RUN --master-port 2968$push tools/comm_phase_times.py --tp 4 --pp 1 --sched $sched > gpurun_out/${TAG}_unit_times_tp4_${sched}_push$push.json 2> gpurun_out/ct.err
    echo "unit times $sched push=$push rc=$?"
  done
done
