#!/usr/bin/env bash
# 4-GPU batch (final build: epilogue without spills, attention backward second pass):
# bf16 / TP4 multi-rank parity on every transport, cfg2 TP4 schedule comparison.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1100 python -m pytest tests/test_gpu_multi.py -q -rA -k "(bf16 or (4-1 and stp)) and not push and not mllm" > gpurun_out/${TAG}_gputest_n4_g.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_n4_g.txt | tail -3
timeout 1200 $RUN --master-port 29791 bench.py --gpus 4 --config cfg2 --steps 5 --warmup 3 --no-cpu --compare \
    --compare-scheds stp,1f1b-i,1f1b-i-naive > gpurun_out/${TAG}_g_n4_cfg2_compare.json 2> gpurun_out/${TAG}_g_n4_cfg2_compare.err
echo "cfg2 rc=$?"; tail -2 gpurun_out/${TAG}_g_n4_cfg2_compare.err
