#!/usr/bin/env bash
# 4-GPU batch F: overlap-contention sweep at cfg2 TP4 (STP vs 1F1B-I on the same kernels):
# p2p comm-kernel CTA caps, the copy-engine transport, and SM partitioning
# (GEMM capped at 148-k CTAs, comm kernels forced onto the free SMs).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for cfg in "default:" "ctas148:STP_P2P_CTAS=148" "ctas74:STP_P2P_CTAS=74" "ce:STP_TP_TRANSPORT=ce" \
           "part12:STP_GEMM_MAX_CTAS=136 STP_COMM_SMEM=65536 STP_P2P_CTAS=24" \
           "part20:STP_GEMM_MAX_CTAS=128 STP_COMM_SMEM=65536 STP_P2P_CTAS=40"; do
  name=${cfg%%:*}; envs=${cfg#*:}; i=$((i+1))
  env $envs timeout 900 $RUN --master-port 2970$i bench.py --gpus 4 --config cfg2 --steps 5 --warmup 3 --no-cpu --compare \
    --compare-scheds stp,1f1b-i > gpurun_out/${TAG}_sweep_${name}.json 2> gpurun_out/${TAG}_sweep_${name}.err
  echo "$name rc=$?"
done
