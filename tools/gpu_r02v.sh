#!/usr/bin/env bash
# GEMM kernels vs cuBLAS: alternating best-of-3 timings (TP1 / TP4 shapes) and ncu
# --set full of ours and cuBLAS's kernel on FC1 forward and FC2 wgrad (TP1).
mkdir -p gpurun_out
for t in 1 4; do
  timeout 900 python tools/kbench.py --tp $t --cublas --iters 20 --only qkv_fwd,o_fwd,fc1_fwd,fc2_fwd,lm_head_fwd,fc2_dgrad,fc1_dgrad,qkv_dgrad,fc2_wgrad,fc1_wgrad,qkv_wgrad > gpurun_out/r02v_kbench_cublas_tp$t.jsonl 2>&1; echo "tp$t rc=$?"
  python - gpurun_out/r02v_kbench_cublas_tp$t.jsonl <<'PY'
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
for g in fc1_fwd fc2_wgrad; do
  KB="python tools/kbench.py --tp 1 --cublas --iters 1 --only $g"
  timeout 300 ncu --metrics gpu__time_duration.sum --csv $KB > gpurun_out/r02v_names_$g.csv 2>/dev/null
  CB=$(grep -v gemm_bf16 gpurun_out/r02v_names_$g.csv | grep -oE '"(nvjet|sm100|cutlass|void cutlass)[^"(]*' | head -1 | tr -d '"' | awk '{print $NF}')
  echo "$g cublas kernel: $CB"
  timeout 600 ncu --set full --clock-control none -k "regex:gemm_bf16" -s 3 -c 1 -o gpurun_out/r02v_ncu_ours_$g $KB > /dev/null 2>&1; echo "ncu ours $g rc=$?"
  if [ -n "$CB" ]; then
    timeout 600 ncu --set full --clock-control none -k "regex:${CB:0:40}" -s 3 -c 1 -o gpurun_out/r02v_ncu_cublas_$g $KB > /dev/null 2>&1; echo "ncu cublas $g rc=$?"
  fi
done
