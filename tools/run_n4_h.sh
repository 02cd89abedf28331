#!/usr/bin/env bash
# 4-GPU: multi-rank MLLM parity (ViT chunk on vs 0; LayerNorm row kernels, d = 80 attention) on the final build.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -rA -k "mllm" > gpurun_out/r02_gputest_n4_mllm_final.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02_gputest_n4_mllm_final.txt | tail -3
