#!/usr/bin/env bash
# 4-GPU MLLM evidence: multi-rank MLLM parity, then the cfg5 proxy (TP2 x PP2)
# bench with the schedule comparison.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -k mllm -q -rA > gpurun_out/${TAG}_gputest_mllm_n4.txt 2>&1
tail -2 gpurun_out/${TAG}_gputest_mllm_n4.txt
timeout 1500 $RUN --master-port 29655 bench.py --gpus 4 --config cfg5 --steps ${STEPS:-5} --warmup 3 --compare \
    --compare-scheds ${SCHEDS:-stp,1f1b-i,1f1b-i-naive,zb} > gpurun_out/${TAG}_bench_n4_cfg5.json \
    2> gpurun_out/${TAG}_bench_n4_cfg5.err
echo "cfg5 rc=$?"; tail -2 gpurun_out/${TAG}_bench_n4_cfg5.err
