#!/usr/bin/env bash
# 4-GPU batch H: multi-rank parity on the new per-schedule transport defaults (+ explicit
# p2p / ce / nccl), comm-phase unit times on ce, and the N=4 headline + comparison lines
# of cfg2 / cfg3 / cfg4 / cfg5 with the round-2 build.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_gpu_multi.py tests/test_gpu_consistency.py -q -rA > gpurun_out/${TAG}_gputest_n4_final.txt 2>&1
tail -2 gpurun_out/${TAG}_gputest_n4_final.txt
STP_TP_TRANSPORT=ce timeout 600 $RUN --master-port 29690 tools/comm_phase_times.py --tp 4 --pp 1 --sched stp > gpurun_out/${TAG}_unit_times_tp4_stp_ce.json 2> gpurun_out/ct.err; echo "unit times ce rc=$?"
for cfg in cfg2 cfg3 cfg4 cfg5; do
  timeout 1500 $RUN --master-port 2975${#cfg} bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 --no-cpu --compare \
      --compare-scheds ${SCHEDS:-stp,1f1b-i,1f1b-i-naive,zb,stp-mem} > gpurun_out/${TAG}_final_n4_${cfg}.json \
      2> gpurun_out/${TAG}_final_n4_${cfg}.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/${TAG}_final_n4_${cfg}.err
done
