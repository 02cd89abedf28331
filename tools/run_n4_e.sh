#!/usr/bin/env bash
# 4-GPU batch J: parity of the transports after the fused copy-engine backward phase,
# ce unit times, final cfg2 / cfg3 comparisons with the round-2 build.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA -k "test_multi_rank_parity[ or symmetric" > gpurun_out/${TAG}_gputest_n4_j.txt 2>&1
tail -2 gpurun_out/${TAG}_gputest_n4_j.txt
timeout 600 $RUN --master-port 29691 tools/comm_phase_times.py --tp 4 --pp 1 --sched stp > gpurun_out/${TAG}_unit_times_tp4_stp_ce_b.json 2> gpurun_out/ct.err; echo "unit times rc=$?"
for cfg in cfg2 cfg3; do
  timeout 1500 $RUN --master-port 2976${#cfg} bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 --no-cpu --compare \
      --compare-scheds stp,1f1b-i,1f1b-i-naive,zb,stp-mem > gpurun_out/${TAG}_final_n4_${cfg}_b.json 2> gpurun_out/${TAG}_final_n4_${cfg}_b.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/${TAG}_final_n4_${cfg}_b.err
done
