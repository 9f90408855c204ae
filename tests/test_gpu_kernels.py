"""Kernel-level parity of libmfgpu against plain fp32 numpy references,
through the C-ABI test entry points (include/mfgpu_test.h)."""

import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2408_11853_b200 import native
    return native.gpu()


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _gemm(lib, prec, epi, A, W, bias, res=None):
    M, K = A.shape
    N = W.shape[1]
    out = np.zeros((M, N), np.float32)
    rc = lib.mfgt_gemm(prec, epi, M, N, K, _p(A), _p(W), _p(bias),
                       _p(res) if res is not None else None, _p(out))
    if rc != 0:
        from paper_2408_11853_b200 import native
        pytest.fail(native.last_error(None)[1])
    return out


def _ref(epi, A, W, bias, res):
    y = A.astype(np.float64) @ W.astype(np.float64) + bias
    if epi == 1:
        y = y + res
    if epi == 2:
        c = math.sqrt(2 / math.pi)
        y = 0.5 * y * (1 + np.tanh(c * (y + 0.044715 * y ** 3)))
    if epi == 3:
        y = np.tanh(y)
    return y


SHAPES = [(1, 16, 16), (37, 48, 16), (130, 64, 64), (200, 256, 128), (256, 512, 256),
          (300, 1024, 1024), (129, 1152, 192), (64, 3456, 1152), (5, 1, 40)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("prec", [0, 2])
def test_gemm_split_parity(lib, M, N, K, epi, prec):
    rng = np.random.default_rng(M * 1000 + N + K + epi)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float32)
    b = (0.1 * rng.standard_normal(N)).astype(np.float32)
    r = rng.standard_normal((M, N)).astype(np.float32)
    got = _gemm(lib, prec, epi, A, W, b, r)
    want = _ref(epi, A, W, b, r)
    # Operand pieces: fp16 ~22 significant bits, bf16 ~16. The tensor-core fp32
    # accumulator truncates on every partial-sum add, so the error also grows
    # ~linearly in the number of k-steps (measured: tools/diag_gemm_precision.py).
    tol = ((2e-6 if prec == 0 else 6e-5) + 4e-8 * K) * (1 + np.abs(want))
    assert np.all(np.abs(got - want) <= tol), float(np.abs(got - want).max())


@pytest.mark.parametrize("K,epi", [(10240, 0), (4352, 1), (8256, 2)])
@pytest.mark.parametrize("prec", [0, 1, 3])
def test_gemm_k_chunked_accumulation(lib, K, epi, prec):
    """K > 4096: fresh TMEM accumulator every 2048 K, chunks summed round-to-nearest
    (ragged last chunk at K = 4352 / 8256, residual and GELU epilogues). The
    error stays at the K = 1024 level instead of growing with K (unchunked, the
    split GEMM reached rms 6e-5 of the output std at K = 10240)."""
    rng = np.random.default_rng(K + epi + 7 * prec)
    M, N = 300, 512
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float32)
    if prec == 3:  # reference binary16 mode: operands are exact binary16
        A = A.astype(np.float16).astype(np.float32)
        W = W.astype(np.float16).astype(np.float32)
    b = (0.1 * rng.standard_normal(N)).astype(np.float32)
    if prec == 3:
        b = b.astype(np.float16).astype(np.float32)
    r = rng.standard_normal((M, N)).astype(np.float32)
    if prec == 3:
        r = r.astype(np.float16).astype(np.float32)
    got = _gemm(lib, prec, epi, A, W, b, r)
    want = _ref(epi, A, W, b, r)
    rms = float(np.sqrt(np.mean((got - want) ** 2)) / want.std())
    bound = {0: 1.5e-5, 1: 5e-3, 3: 8e-4}[prec]  # bf16 / binary16 output rounding dominate
    assert rms <= bound, rms


@pytest.mark.parametrize("M,N,K", SHAPES[:6])
def test_gemm_bf16_mode(lib, M, N, K):
    rng = np.random.default_rng(7 + M)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float32)
    b = np.zeros(N, np.float32)
    got = _gemm(lib, 1, 0, A, W, b)
    want = _ref(0, A, W, b, None)
    assert np.abs(got - want).max() <= 0.03 * (1 + np.abs(want).max())
    # bf16 inputs exactly reproduce a bf16-rounded fp32 product
    import torch
    Ab = torch.from_numpy(A).bfloat16().double().numpy()
    Wb = torch.from_numpy(W).bfloat16().double().numpy()
    assert np.allclose(got, Ab @ Wb, atol=1e-4, rtol=1e-4)


def _attn_ref(qkv, cu, d, H):
    out = np.zeros((qkv.shape[0], d), np.float64)
    dh = d // H
    for s in range(len(cu) - 1):
        a, b = cu[s], cu[s + 1]
        for h in range(H):
            q = qkv[a:b, h * dh:(h + 1) * dh].astype(np.float64)
            k = qkv[a:b, d + h * dh:d + (h + 1) * dh].astype(np.float64)
            v = qkv[a:b, 2 * d + h * dh:2 * d + (h + 1) * dh].astype(np.float64)
            s_ = q @ k.T / math.sqrt(dh)
            p = np.exp(s_ - s_.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            out[a:b, h * dh:(h + 1) * dh] = p @ v
    return out


@pytest.mark.parametrize("d,H,lens", [(16, 2, [3, 1, 7]), (64, 1, [65, 2, 130, 16, 17]),
                                      (1024, 16, [128, 3, 64, 100, 1, 33, 127, 129]),
                                      (256, 4, [512, 64, 65]), (2560, 32, [70, 9]),
                                      (2560, 32, [300, 9, 129]), (320, 4, [511, 200]),
                                      (1152, 18, [127, 5])])
@pytest.mark.parametrize("prec", [0, 2, 1, 3])
@pytest.mark.parametrize("use_tc", [1, 0])
def test_attention_parity(lib, d, H, lens, prec, use_tc):
    rng = np.random.default_rng(d + len(lens))
    cu = np.zeros(len(lens) + 1, np.int32)
    cu[1:] = np.cumsum(lens)
    T = int(cu[-1])
    qkv = (2 * rng.standard_normal((T, 3 * d))).astype(np.float32)
    out = np.zeros((T, d), np.float32)
    rc = lib.mfgt_attention(prec, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H,
                            _p(qkv), _p(out), use_tc)
    assert rc == 0
    want = _attn_ref(qkv, cu, d, H)
    tol = {0: 1e-5, 2: 1e-4, 1: 3e-2, 3: 5e-3}[prec]
    assert np.abs(out - want).max() <= tol * (1 + np.abs(want).max())


@pytest.mark.parametrize("T,d", [(1, 16), (33, 256), (100, 1024), (7, 1152), (5, 2560)])
def test_layernorm_parity(lib, T, d):
    rng = np.random.default_rng(T + d)
    y = (3 * rng.standard_normal((T, d)) + 1).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    b = (0.1 * rng.standard_normal(d)).astype(np.float32)
    out = np.zeros_like(y)
    assert lib.mfgt_layernorm(T, d, _p(y), _p(g), _p(b), _p(out)) == 0
    y64 = y.astype(np.float64)
    mu = y64.mean(1, keepdims=True)
    var = ((y64 - mu) ** 2).mean(1, keepdims=True)
    want = (y64 - mu) / np.sqrt(var + 1e-5) * g + b
    assert np.abs(out - want).max() <= 2e-5 * (1 + np.abs(want).max())


@pytest.mark.parametrize("M,N,K", [(37, 48, 16), (200, 256, 128), (300, 1024, 1024), (129, 1152, 192)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_fp16_reference_mode(lib, M, N, K, epi):
    """Precision 3 (the reference's fp16 mode): binary16 operands, one MMA per
    k-step, fp16 rounding of the product, fp16 bias add, fp16 residual sum
    (`encoder.py:120-126`). fp16 products are exact in fp32, so the device agrees
    with the reference arithmetic except for rare 1-ulp flips from the fp32
    summation order."""
    rng = np.random.default_rng(M + N + K + 10 * epi)
    h = lambda x: np.asarray(x, np.float32).astype(np.float16)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float32)
    b = (0.1 * rng.standard_normal(N)).astype(np.float32)
    r = h(rng.standard_normal((M, N))).astype(np.float32)
    got = _gemm(lib, 3, epi, A, W, b, r)
    prod = h(h(A).astype(np.float64) @ h(W).astype(np.float64))
    y = h(prod + h(b))                       # numpy float16 + float16 -> float16
    if epi == 1:
        y = h(y.astype(np.float32) + r)
    if epi == 2:
        c = math.sqrt(2 / math.pi)
        y32 = y.astype(np.float32)
        y = h(0.5 * y32 * (1 + np.tanh(c * (y32 + 0.044715 * y32 ** 3))))
    want = y.astype(np.float64)
    # a 1-ulp flip of the rounded product propagates through the fp16 bias /
    # residual adds: bound by the ulp of the largest operand along the chain
    scale = np.abs(prod.astype(np.float64)) + np.abs(h(b).astype(np.float64)) + np.abs(want)
    if epi == 1:
        scale = scale + np.abs(r)
    ulp = np.spacing(scale.astype(np.float16)).astype(np.float64)
    d = np.abs(got - want)
    assert np.all(d <= 3 * ulp + 1e-7), float((d / ulp).max())
    assert np.mean(d == 0) > 0.97


@pytest.mark.parametrize("k", [-14, -7, 17])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_weight_prescale_is_scale_equivariant(lib, k, epi):
    """fp32-parity GEMM: with the per-column power-of-two weight prescale,
    weights and bias times 2^k give exactly 2^k times the output — tiny weights
    (2^-14 ~ 6e-5: unscaled, their fp16 lo pieces would be subnormal) and huge
    ones (2^17: beyond the fp16 range, which used to fail the load) keep the
    unit-scale precision bit for bit."""
    rng = np.random.default_rng(100 + k + epi)
    M, N, K = 300, 384, 1024
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float32)
    b = (0.1 * rng.standard_normal(N)).astype(np.float32)
    r = rng.standard_normal((M, N)).astype(np.float32)
    s = np.float32(2.0 ** k)
    base = _gemm(lib, 0, epi, A, W, b, r)
    scaled = _gemm(lib, 0, epi, A, W * s, b * s, r * s)  # epi 1: residual scaled too
    assert np.array_equal(scaled, base * s)
    rel = float(np.abs(base - _ref(epi, A, W, b, r)).max() / np.abs(base).max())
    assert rel <= 2e-5, rel
