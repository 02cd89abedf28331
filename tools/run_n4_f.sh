#!/usr/bin/env bash
# 4-GPU batch M (last build): ZB (cost-aware list schedule) in the cfg2 / cfg4 comparisons,
# multi-rank ZB parity.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -rA -k "zb" > gpurun_out/${TAG}_gputest_n4_zb.txt 2>&1; tail -1 gpurun_out/${TAG}_gputest_n4_zb.txt
for cfg in cfg2 cfg4; do
  timeout 1500 $RUN --master-port 2978${#cfg} bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 --no-cpu --compare \
      --compare-scheds stp,1f1b-i,1f1b-i-naive,zb,stp-mem > gpurun_out/${TAG}_last_n4_${cfg}.json 2> gpurun_out/${TAG}_last_n4_${cfg}.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/${TAG}_last_n4_${cfg}.err
done
