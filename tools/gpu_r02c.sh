#!/usr/bin/env bash
# round-2 batch C: offload tests, N=1 bench comparison, ncu of the attention
# kernels (LM and ViT shapes), launch list of the N=1 headline step.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 600 python -m pytest tests/test_gpu_offload.py -q -rA > gpurun_out/${TAG}_gputest_offload.txt 2>&1; echo "offload pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gputest_offload.txt | tail -6
timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu --compare --compare-scheds stp,1f1b-i,1f1b-i-naive,zb,stp-mem,stp@0.25 > gpurun_out/${TAG}_bench_n1_compare.json 2> gpurun_out/${TAG}_bench_n1_compare.err; echo "bench rc=$?"
tail -c 300 gpurun_out/${TAG}_bench_n1_compare.json; tail -2 gpurun_out/${TAG}_bench_n1_compare.err
# ncu: attention kernels (kbench, attention only, 1 timed iteration: 4 launches per kernel and shape)
KB="python tools/kbench.py --skip-gemm --iters 1"
$KB > gpurun_out/kb_plain.log 2>&1 && echo "kbench plain ok"
for spec in "attn_fwd_sm100:0:lm_fwd" "attn_bwd_fused_sm100:0:lm_bwd" "attn_fwd_sm100:4:vit_fwd" "attn_bwd_fused_sm100:4:vit_bwd"; do
  K=${spec%%:*}; rest=${spec#*:}; SK=${rest%%:*}; NM=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^${K}" -s $SK -c 1 -o gpurun_out/${TAG}_ncu_${NM} $KB > gpurun_out/ncu_${NM}.log 2>&1
  echo "ncu $NM rc=$?"
done
# launch list of one N=1 headline step (cfg2, TP1)
BC="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/${TAG}_launches_n1.csv $BC > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"; gzip -f gpurun_out/${TAG}_launches_n1.csv
