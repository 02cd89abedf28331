#!/usr/bin/env bash
# ViT / MLLM checks on one GPU: kernel parity, MLLM stage parity, regression of
# the LM attention tests, kernel bench incl. ViT attention, a short cfg5 bench.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python -m pytest tests/test_gpu_vit_ops.py tests/test_gpu_mllm.py tests/test_gpu_ops.py tests/test_gpu_stage.py -q -rA -x > gpurun_out/${TAG}_vit_tests.txt 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error" gpurun_out/${TAG}_vit_tests.txt | tail -5
timeout 300 python tools/kbench.py --skip-gemm --iters 10 > gpurun_out/${TAG}_kbench_attn.jsonl 2>&1; echo "kbench rc=$?"
cat gpurun_out/${TAG}_kbench_attn.jsonl
if [ "${BENCH5:-1}" = 1 ]; then
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_cfg5_n1.json 2> gpurun_out/${TAG}_bench_cfg5_n1.err; echo "bench cfg5 rc=$?"
tail -c 600 gpurun_out/${TAG}_bench_cfg5_n1.json; tail -3 gpurun_out/${TAG}_bench_cfg5_n1.err
fi
