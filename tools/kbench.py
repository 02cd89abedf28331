"""Kernel microbenchmark at the production shapes (Qwen2-7B layer, TP = t,
seq 6144): every GEMM of the unit set (forward NT, dgrad NN, wgrad TN with
fp32 accumulation) and causal GQA attention fwd / bwd, timed with CUDA events
(warm-up 3, mean of N), for each tuning-knob variant.  One JSON line per case.

  python tools/kbench.py [--tp 1] [--iters 10] [--gemm-mc 0,1,3] [--skip-gemm]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_27257_b200  # noqa: E402,F401
import torch  # noqa: E402

from paper_2510_27257_b200 import _lib, ops  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--seq", type=int, default=6144)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--gemm-mc", default="1")
    ap.add_argument("--skip-gemm", action="store_true")
    ap.add_argument("--skip-elementwise", action="store_true")
    ap.add_argument("--only", default="", help="comma list of GEMM names (e.g. fc1_wgrad); skips attention")
    ap.add_argument("--cublas", action="store_true",
                    help="also time torch.matmul (cuBLAS) on each GEMM shape and layout (bf16 output)")
    a = ap.parse_args()
    t, s = a.tp, a.seq
    h, I, V = 3584, 18944 // t, 152064 // t
    nq, nkv, d = 28 // t, 4 // t, 128
    qkv = (nq + 2 * nkv) * d
    bf = torch.bfloat16
    dev = "cuda"
    gemms = [  # name, layout, M, N, K, epilogue
        ("qkv_fwd", 0, s, qkv, h, 0), ("o_fwd", 0, s, h, nq * d, 0), ("fc1_fwd", 0, s, 2 * I, h, 0),
        ("fc2_fwd", 0, s, h, I, 0), ("lm_head_fwd", 0, s, V, h, 0),
        ("fc2_dgrad", 1, s, I, h, 0), ("fc1_dgrad", 1, s, h, 2 * I, 0), ("qkv_dgrad", 1, s, h, qkv, 0),
        ("fc2_wgrad", 2, h, I, s, 2), ("fc1_wgrad", 2, 2 * I, h, s, 2), ("qkv_wgrad", 2, qkv, h, s, 2),
    ]
    if not a.skip_gemm:
        for mc in [int(x) for x in a.gemm_mc.split(",")]:
            _lib.call("stp_set_option", b"gemm_mc", mc)
            for name, lay, M, N, K, epi in gemms:
                if a.only and name not in a.only.split(","):
                    continue
                if lay == 0:
                    A = torch.randn(M, K, device=dev, dtype=bf)
                    B = torch.randn(N, K, device=dev, dtype=bf)
                elif lay == 1:
                    A = torch.randn(M, K, device=dev, dtype=bf)
                    B = torch.randn(K, N, device=dev, dtype=bf)
                else:
                    A = torch.randn(K, M, device=dev, dtype=bf)
                    B = torch.randn(K, N, device=dev, dtype=bf)
                C = torch.zeros(M, N, device=dev, dtype=torch.float32 if epi == 2 else bf)
                ours = lambda: ops.gemm(lay, A, B, C, M, N, K, epi=epi, dtype=1)  # noqa: E731
                ms = timed(ours, a.iters)
                if not a.cublas:
                    print(json.dumps({"kernel": "gemm", "name": name, "gemm_mc": mc, "M": M, "N": N, "K": K,
                                      "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}), flush=True)
                if a.cublas:  # same operands and layout; bf16 output (no fp32 accumulate epilogue)
                    Ct = torch.empty(M, N, device=dev, dtype=bf)
                    mm = {0: lambda: torch.matmul(A, B.t(), out=Ct), 1: lambda: torch.matmul(A, B, out=Ct),
                          2: lambda: torch.matmul(A.t(), B, out=Ct)}[lay]
                    ms_c = timed(mm, a.iters)
                    for _ in range(2):  # alternate (same power / clock state), best of three each
                        ms = min(ms, timed(ours, a.iters))
                        ms_c = min(ms_c, timed(mm, a.iters))
                    print(json.dumps({"kernel": "gemm", "name": name, "gemm_mc": mc, "M": M, "N": N, "K": K,
                                      "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}), flush=True)
                    print(json.dumps({"kernel": "gemm_cublas", "name": name, "M": M, "N": N, "K": K, "ms": ms_c,
                                      "tflops": 2 * M * N * K / ms_c / 1e9, "speed_ours_vs_cublas": ms_c / ms}),
                          flush=True)
                    del Ct
                del A, B, C
    if a.only:
        return
    if not a.skip_elementwise:
        # HBM-bound kernels of the units at the per-rank shapes (bytes = what a
        # kernel must read + write once; GB/s vs the measured 6456 GB/s copy bandwidth)
        rows = s // t
        xs = torch.randn(rows, h, device=dev, dtype=bf)
        rs_ = torch.randn(rows, h, device=dev, dtype=bf)
        g = torch.ones(h, device=dev, dtype=bf)
        y = torch.empty_like(xs)
        xo = torch.empty_like(xs)
        rstd = torch.empty(rows, device=dev, dtype=torch.float32)
        ms = timed(lambda: ops.rmsnorm_fwd(xs, g, 1e-6, y, rstd, resid=rs_, x_out=xo), a.iters)
        print(json.dumps({"kernel": "rmsnorm_fwd_resid", "rows": rows, "h": h, "ms": ms,
                          "gbps": 4 * rows * h * 2 / ms / 1e6}), flush=True)
        dxo = torch.empty_like(xs)
        dg = torch.zeros(h, device=dev, dtype=torch.float32)
        ms = timed(lambda: ops.rmsnorm_bwd(y, xo, g, rstd, dxo, None, dres=rs_), a.iters)
        print(json.dumps({"kernel": "rmsnorm_bwd_resid", "rows": rows, "h": h, "ms": ms,
                          "gbps": 4 * rows * h * 2 / ms / 1e6}), flush=True)
        # ViT LayerNorm (+ residual) at the MLLM shape: cfg5's image rows per
        # rank (4 images x 1024 patches ... here s rows) x hv 1280
        hv = 1280
        xv = torch.randn(s, hv, device=dev, dtype=bf)
        rv = torch.randn(s, hv, device=dev, dtype=bf)
        gv = torch.ones(hv, device=dev, dtype=bf)
        bv = torch.zeros(hv, device=dev, dtype=bf)
        yv, xov, dxv = torch.empty_like(xv), torch.empty_like(xv), torch.empty_like(xv)
        mv = torch.empty(s, device=dev, dtype=torch.float32)
        rsv = torch.empty(s, device=dev, dtype=torch.float32)
        ms = timed(lambda: ops.layernorm_fwd(xv, gv, bv, 1e-6, yv, mv, rsv, resid=rv, x_out=xov), a.iters)
        print(json.dumps({"kernel": "layernorm_fwd_resid", "rows": s, "h": hv, "ms": ms,
                          "gbps": 4 * s * hv * 2 / ms / 1e6}), flush=True)
        ms = timed(lambda: ops.layernorm_bwd(yv, xov, gv, mv, rsv, dxv, dres=rv), a.iters)
        print(json.dumps({"kernel": "layernorm_bwd_resid", "rows": s, "h": hv, "ms": ms,
                          "gbps": 4 * s * hv * 2 / ms / 1e6}), flush=True)
        del xv, rv, yv, xov, dxv
        gu = torch.randn(s, 2 * I, device=dev, dtype=bf)
        H = torch.empty(s, I, device=dev, dtype=bf)
        ms = timed(lambda: ops.swiglu_fwd(gu, H), a.iters)
        print(json.dumps({"kernel": "swiglu_fwd", "s": s, "I": I, "ms": ms, "gbps": 3 * s * I * 2 / ms / 1e6}),
              flush=True)
        dH = torch.randn(s, I, device=dev, dtype=bf)
        dgu = torch.empty_like(gu)
        ms = timed(lambda: ops.swiglu_bwd(dH, gu, dgu), a.iters)
        print(json.dumps({"kernel": "swiglu_bwd", "s": s, "I": I, "ms": ms, "gbps": 5 * s * I * 2 / ms / 1e6}),
              flush=True)
        del gu, H, dH, dgu
    x = torch.randn(s, qkv, device=dev, dtype=bf)
    o = torch.empty(s, nq * d, device=dev, dtype=bf)
    lse = torch.empty(nq, s, device=dev, dtype=torch.float32)
    pairs = s * (s + 1) / 2
    ms = timed(lambda: ops.attn_fwd(x, nq, nkv, d, o, lse), a.iters)
    print(json.dumps({"kernel": "attn_fwd", "s": s, "nq": nq, "nkv": nkv, "ms": ms,
                      "tflops": 4 * pairs * nq * d / ms / 1e9}), flush=True)
    do = torch.randn(s, nq * d, device=dev, dtype=bf)
    dx = torch.empty_like(x)
    ms = timed(lambda: ops.attn_bwd(x, nq, nkv, d, o, do, lse, dx), a.iters)
    print(json.dumps({"kernel": "attn_bwd", "s": s, "nq": nq, "nkv": nkv, "ms": ms,
                      "tflops": 8 * pairs * nq * d / ms / 1e9}), flush=True)
    # ViT-600M bidirectional attention (d = 80, 16 heads / t, 3136 patches)
    sv, nh, dv = 3136, 16 // t, 80
    xv = torch.randn(sv, 3 * nh * dv, device=dev, dtype=bf)
    ov = torch.empty(sv, nh * dv, device=dev, dtype=bf)
    lv = torch.empty(nh, sv, device=dev, dtype=torch.float32)
    ms = timed(lambda: ops.attn_full_fwd(xv, nh, dv, ov, lv), a.iters)
    print(json.dumps({"kernel": "vit_attn_fwd", "s": sv, "nh": nh, "d": dv, "ms": ms,
                      "tflops": 4 * sv * sv * nh * dv / ms / 1e9}), flush=True)
    dov = torch.randn(sv, nh * dv, device=dev, dtype=bf)
    dxv = torch.empty_like(xv)
    ms = timed(lambda: ops.attn_full_bwd(xv, nh, dv, ov, dov, lv, dxv), a.iters)
    print(json.dumps({"kernel": "vit_attn_bwd", "s": sv, "nh": nh, "d": dv, "ms": ms,
                      "tflops": 8 * sv * sv * nh * dv / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
