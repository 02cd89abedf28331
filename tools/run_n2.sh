#!/usr/bin/env bash
# 2-GPU: cfg2 TP2 headline on the per-schedule default (STP on ce) and on p2p, with the
# STP vs 1F1B-I comparison; cfg5 MLLM at TP2.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1200 $RUN --master-port 29801 bench.py --gpus 2 --config cfg2 --steps 5 --warmup 3 --no-cpu --compare --compare-scheds stp,1f1b-i > gpurun_out/${TAG}_final_n2_cfg2.json 2> gpurun_out/${TAG}_final_n2_cfg2.err; echo "cfg2 ce rc=$?"
STP_TP_TRANSPORT=p2p timeout 1200 $RUN --master-port 29802 bench.py --gpus 2 --config cfg2 --steps 5 --warmup 3 --no-cpu --compare --compare-scheds stp,1f1b-i > gpurun_out/${TAG}_final_n2_cfg2_p2p.json 2> gpurun_out/${TAG}_final_n2_cfg2_p2p.err; echo "cfg2 p2p rc=$?"
