#!/usr/bin/env bash
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python -m pytest tests/test_gpu_vit_ops.py tests/test_gpu_mllm.py tests/test_gpu_ops.py tests/test_gpu_stage.py -q -rA > gpurun_out/${TAG}_vit_tests.txt 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_vit_tests.txt | tail -12
