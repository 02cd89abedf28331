#!/usr/bin/env bash
# Phase timeline of the attention backward (clock64 stamps of one CTA, kt = 0, h = 0).
# Needs the instrumented kernel: git apply tools/attn_bwd_trace.patch && python -m paper_2510_27257_b200.build
mkdir -p gpurun_out
STP_ATTN_BWD_TRACE=gpurun_out/r02t_bwd_trace.txt timeout 300 python tools/kbench.py --skip-gemm --skip-elementwise > gpurun_out/r02t_kbench.jsonl 2>&1; echo "rc=$?"; grep attn_bwd gpurun_out/r02t_kbench.jsonl | cut -c1-150; wc -l gpurun_out/r02t_bwd_trace.txt
