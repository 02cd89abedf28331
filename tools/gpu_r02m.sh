#!/usr/bin/env bash
# row-per-CTA LayerNorm: ViT / MLLM parity, LN A/B microbenchmark, cfg5 N=1.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vit_ops.py tests/test_gpu_mllm.py tests/test_gpu_offload.py -q -rA > gpurun_out/r02m_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02m_tests.txt | tail -4
for rb in 0 1; do
  STP_LN_ROWBLOCK=$rb timeout 300 python tools/kbench.py --skip-gemm --seq 16384 > gpurun_out/r02m_kbench_ln$rb.jsonl 2>&1; echo "kbench ln$rb rc=$?"
  grep -E "layernorm|rmsnorm" gpurun_out/r02m_kbench_ln$rb.jsonl
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02m_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02m_smoke.txt
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02m_bench_cfg5_n1.json 2> gpurun_out/r02m_bench_cfg5_n1.err; echo "cfg5 rc=$?"; tail -c 250 gpurun_out/r02m_bench_cfg5_n1.json
