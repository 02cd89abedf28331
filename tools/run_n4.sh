#!/usr/bin/env bash
# 4-GPU evidence for profiles/ (one gpurun --gpus 4 call): the multi-GPU
# pytest pass list, then bench lines with the schedule comparison for the
# cfg2 TP4 proxy, the cfg3 proxy (TP2 x PP2) and the cfg4 proxy (TP2 x PP2).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  nvidia-smi -L > gpurun_out/${TAG}_gputest_n4.txt
  timeout 1800 python -m pytest tests/test_gpu_multi.py tests/test_gpu_consistency.py -q -rA >> gpurun_out/${TAG}_gputest_n4.txt 2>&1
  tail -2 gpurun_out/${TAG}_gputest_n4.txt
fi
for cfg in ${CFGS:-cfg2 cfg3 cfg4}; do
  timeout 1500 $RUN --master-port 2962${#cfg} bench.py --gpus 4 --config $cfg --steps ${STEPS:-5} --warmup 3 --compare \
      --compare-scheds ${SCHEDS:-stp,1f1b-i,1f1b-i-naive,zb,stp-nobraid} > gpurun_out/${TAG}_bench_n4_${cfg}.json \
      2> gpurun_out/${TAG}_bench_n4_${cfg}.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/${TAG}_bench_n4_${cfg}.err
done
