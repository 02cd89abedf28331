#!/usr/bin/env bash
# GEMM kernels vs cuBLAS (torch.matmul) on the TP1 and TP4 production shapes.
mkdir -p gpurun_out
for t in 1 4; do
  timeout 600 python tools/kbench.py --tp $t --cublas --iters 20 --only qkv_fwd,o_fwd,fc1_fwd,fc2_fwd,lm_head_fwd,fc2_dgrad,fc1_dgrad,qkv_dgrad,fc2_wgrad,fc1_wgrad,qkv_wgrad > gpurun_out/r02u_kbench_cublas_tp$t.jsonl 2>&1; echo "tp$t rc=$?"
  python - gpurun_out/r02u_kbench_cublas_tp$t.jsonl <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        if d["kernel"] == "gemm_cublas":
            print(f'{d["name"]:12s} cublas {d["tflops"]:7.0f} ours speed / cublas {d["speed_ours_vs_cublas"]:.3f}')
PY
done
