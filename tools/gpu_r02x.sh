#!/usr/bin/env bash
# (historical: STP_SWIGLU_EPI was removed after this measurement -- DESIGN.md §7c)
# SwiGLU backward fused into the FC2 dgrad epilogue (STP_SWIGLU_EPI=1; re-measured now that the
# epilogue keeps its registers): whole-step bf16 parity with it on, N=1 A/B.
mkdir -p gpurun_out
STP_SWIGLU_EPI=1 timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_gpu_offload.py -q -rA -k "bf16 or qwen or offload" > gpurun_out/r02x_tests.txt 2>&1; echo "tests rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r02x_tests.txt | tail -3
for e in 0 1 0 1; do
  STP_SWIGLU_EPI=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02x_bench_epi$e.json 2>/dev/null; echo "bench epi=$e rc=$?"
  python -c "
import json;L=[l for l in open('gpurun_out/r02x_bench_epi$e.json') if l.startswith('{')];d=json.loads(L[-1]);print('epi=$e', round(d['value']), round(d['roofline']['gemm_ms_per_step']), round(d['ms_per_step']), d['clocks']['sm_mhz'])"
done
