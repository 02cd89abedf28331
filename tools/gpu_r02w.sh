#!/usr/bin/env bash
# GEMM epilogue without local-memory spills (no runtime indexing of the accumulator
# registers): GEMM / CE parity, ours vs cuBLAS at TP1 / TP4, N=1 headline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_ops.py -q -rA -k "gemm or lm_head or ce" > gpurun_out/r02w_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02w_tests.txt | tail -3
for t in 1 4; do
  timeout 900 python tools/kbench.py --tp $t --cublas --iters 20 --only qkv_fwd,o_fwd,fc1_fwd,fc2_fwd,lm_head_fwd,fc2_dgrad,fc1_dgrad,qkv_dgrad,fc2_wgrad,fc1_wgrad,qkv_wgrad > gpurun_out/r02w_kbench_cublas_tp$t.jsonl 2>&1; echo "tp$t rc=$?"
  python - gpurun_out/r02w_kbench_cublas_tp$t.jsonl <<'PY'
import json, sys
o = {}
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        if d["kernel"] == "gemm":
            o[d["name"]] = d["tflops"]
        else:
            print(f'{d["name"]:12s} ours {o[d["name"]]:6.0f} cublas {d["tflops"]:6.0f} speed ours/cublas {d["speed_ours_vs_cublas"]:.3f}')
PY
done
timeout 600 ncu --set full --clock-control none -k "regex:gemm_bf16" -s 3 -c 1 -o gpurun_out/r02w_ncu_ours_fc1_fwd python tools/kbench.py --tp 1 --iters 1 --only fc1_fwd > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02w_bench_n1.json 2> gpurun_out/r02w_bench_n1.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02w_bench_n1.json
