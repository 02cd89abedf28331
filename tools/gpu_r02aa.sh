#!/usr/bin/env bash
# RMSNorm / LayerNorm backward row kernels with the residual gradient loaded in the first pass:
# op parity, kbench (elementwise) A/B against the warp-per-row LayerNorm switch for reference.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_vit_ops.py -q -k "rmsnorm or layernorm" > gpurun_out/r02aa_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02aa_tests.txt
timeout 300 python tools/kbench.py --skip-gemm --seq 16384 > gpurun_out/r02aa_kbench.jsonl 2>&1; echo "kbench rc=$?"
grep -E "rmsnorm|layernorm" gpurun_out/r02aa_kbench.jsonl
