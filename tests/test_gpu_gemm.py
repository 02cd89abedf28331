"""GEMM kernels (tcgen05 bf16, SIMT fp32) vs the plain definition in fp64.

The three layouts are the linear layer's forward Y = X W^T, dgrad dX = dY W
and wgrad dW = dY^T X (oracle/model.py backward_mb).  Shapes span several
128 x 256 tiles with ragged M / N / K tails, plus the cfg3 TP=4 shapes.
Tolerances: bf16 output => max |err| <= 1e-2 * max |ref| and relative
Frobenius error <= 4e-3 (bf16 rounding of the output, 2^-9 relative, with
fp32 accumulation); fp32 => relative Frobenius error <= 1e-6.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 64), (256, 512, 192), (200, 136, 72), (336, 520, 1000), (1024, 1152, 896),
          (4096, 1152, 3584), (296, 576, 200)]   # N % 192 == 0: the 128 x 192 tiles


def _ops():
    from paper_2510_27257_b200 import ops
    return ops


def _mk(shape, seed, dtype):
    a = np.random.default_rng(seed).standard_normal(shape)
    t = torch.from_numpy(a).to(dtype)
    return t.double().numpy(), t.cuda()


def _ref(layout, A, B):
    if layout == 0:
        return A @ B.T
    if layout == 1:
        return A @ B
    return A.T @ B


def _shapes_for(layout, M, N, K):
    if layout == 0:
        return (M, K), (N, K)
    if layout == 1:
        return (M, K), (K, N)
    return (K, M), (K, N)


@pytest.fixture(params=[int(x) for x in os.environ.get("STP_TEST_GEMM_MODES", "0,1,3").split(",")], ids=lambda m: f"mode{m}")
def gemm_mode(request):
    from paper_2510_27257_b200 import _lib
    _lib.call("stp_set_option", b"gemm_mc", request.param)
    yield request.param
    _lib.call("stp_set_option", b"gemm_mc", 1)


@pytest.mark.parametrize("layout", [0, 1, 2])
@pytest.mark.parametrize("MNK", SHAPES)
def test_gemm_bf16(layout, MNK, gemm_mode):
    ops = _ops()
    M, N, K = MNK
    sa, sb = _shapes_for(layout, M, N, K)
    A, dA = _mk(sa, 1, torch.bfloat16)
    B, dB = _mk(sb, 2, torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ops.gemm(layout, dA, dB, C, M, N, K)
    torch.cuda.synchronize()
    ref = _ref(layout, A, B)
    got = C.double().cpu().numpy()
    err = np.abs(got - ref)
    assert err.max() <= 1e-2 * np.abs(ref).max(), err.max()
    assert np.linalg.norm(got - ref) <= 4e-3 * np.linalg.norm(ref)


@pytest.mark.parametrize("epi", [1, 2, 3])
def test_gemm_bf16_epilogues(epi, gemm_mode):
    ops = _ops()
    M, N, K = 300, 392, 256
    A, dA = _mk((M, K), 3, torch.bfloat16)
    B, dB = _mk((N, K), 4, torch.bfloat16)
    ref = A @ B.T
    bias = R = None
    if epi == 1:
        b, bias = _mk((N,), 5, torch.bfloat16)
        ref = ref + b
    if epi == 3:
        r, R = _mk((M, N), 6, torch.bfloat16)
        ref = ref + r
    if epi == 2:
        c0, _ = _mk((M, N), 7, torch.float32)
        C = torch.from_numpy(c0).float().cuda()
        ref = ref + c0
    else:
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ops.gemm(0, dA, dB, C, M, N, K, epi=epi, bias=bias, R=R, dtype=1)
    torch.cuda.synchronize()
    got = C.double().cpu().numpy()
    tol = 1e-5 if epi == 2 else 4e-3
    assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref)


@pytest.mark.parametrize("layout", [0, 1, 2])
def test_gemm_bf16_max_ctas(layout, gemm_mode):
    ops = _ops()
    M, N, K = 1000, 712, 320
    sa, sb = _shapes_for(layout, M, N, K)
    A, dA = _mk(sa, 8, torch.bfloat16)
    B, dB = _mk(sb, 9, torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ops.gemm(layout, dA, dB, C, M, N, K, max_ctas=7)
    torch.cuda.synchronize()
    ref = _ref(layout, A, B)
    assert np.linalg.norm(C.double().cpu().numpy() - ref) <= 4e-3 * np.linalg.norm(ref)


@pytest.mark.parametrize("layout", [0, 1, 2])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_gemm_fp32(layout, epi):
    ops = _ops()
    M, N, K = 77, 130, 45
    sa, sb = _shapes_for(layout, M, N, K)
    A, dA = _mk(sa, 10, torch.float32)
    B, dB = _mk(sb, 11, torch.float32)
    ref = _ref(layout, A, B)
    bias = R = None
    C = torch.empty(M, N, dtype=torch.float32, device="cuda")
    if epi == 1:
        b, bias = _mk((N,), 12, torch.float32)
        ref = ref + b
    if epi == 2:
        c0, C = _mk((M, N), 13, torch.float32)
        ref = ref + c0
    if epi == 3:
        r, R = _mk((M, N), 14, torch.float32)
        ref = ref + r
    ops.gemm(layout, dA, dB, C, M, N, K, epi=epi, bias=bias, R=R)
    torch.cuda.synchronize()
    assert np.linalg.norm(C.double().cpu().numpy() - ref) <= 1e-6 * np.linalg.norm(ref)


def _swiglu_bwd_ref(dH, G, U):
    sg = 1.0 / (1.0 + np.exp(-G))
    return dH * U * sg * (1.0 + G * (1.0 - sg)), dH * G * sg


@pytest.mark.parametrize("MNK", [(300, 392, 256), (512, 1024, 384), (130, 72, 64)])
def test_gemm_bf16_swiglu_bwd_epilogue(MNK, gemm_mode):
    """STP_EPI_SWIGLU_BWD: the FC2 activation-gradient GEMM dH = dY Wd with the
    SwiGLU backward applied in the epilogue, [G | U] -> [dG | dU] in place."""
    ops = _ops()
    M, N, K = MNK
    A, dA = _mk((M, K), 21, torch.bfloat16)
    B, dB = _mk((K, N), 22, torch.bfloat16)
    gu0, GU = _mk((M, 2 * N), 23, torch.bfloat16)
    ops.gemm(1, dA, dB, GU, M, N, K, epi=4, dtype=1)
    torch.cuda.synchronize()
    dG, dU = _swiglu_bwd_ref(A @ B, gu0[:, :N], gu0[:, N:])
    got = GU.double().cpu().numpy()
    for g, r in ((got[:, :N], dG), (got[:, N:], dU)):
        assert np.linalg.norm(g - r) <= 6e-3 * np.linalg.norm(r)


def test_gemm_fp32_swiglu_bwd_epilogue():
    ops = _ops()
    M, N, K = 77, 130, 45
    A, dA = _mk((M, K), 24, torch.float32)
    B, dB = _mk((K, N), 25, torch.float32)
    gu0, GU = _mk((M, 2 * N), 26, torch.float32)
    ops.gemm(1, dA, dB, GU, M, N, K, epi=4)
    torch.cuda.synchronize()
    dG, dU = _swiglu_bwd_ref(A @ B, gu0[:, :N], gu0[:, N:])
    got = GU.double().cpu().numpy()
    assert np.linalg.norm(got[:, :N] - dG) <= 1e-5 * np.linalg.norm(dG)
    assert np.linalg.norm(got[:, N:] - dU) <= 1e-5 * np.linalg.norm(dU)
