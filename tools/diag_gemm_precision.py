"""Diagnose tcgen05 split-GEMM precision: subnormal handling and accumulator
rounding, via the mfgt_gemm C-ABI test entry point."""
import ctypes as C, math, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_11853_b200 import native
lib = native.gpu()
P = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
def gemm(prec, A, W):
    M, K = A.shape; N = W.shape[1]
    out = np.zeros((M, N), np.float32)
    assert lib.mfgt_gemm(prec, 0, M, N, K, P(A), P(W), P(np.zeros(N, np.float32)), None, P(out)) == 0, native.last_error()
    return out
rng = np.random.default_rng(0)
M, N = 256, 512
for K in [int(k) for k in os.environ.get("KS", "64,1024,4096").split(",")]:
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) * 0.02).astype(np.float32)
    ref = A.astype(np.float64) @ W.astype(np.float64)
    scale = np.abs(ref).std()
    for name, a, w, fac in (("plain", A, W, 1.0), ("W*1024", A, W * 1024, 1024.0),
                            ("A*64,W*1024", A * 64, W * 1024, 65536.0)):
        for prec in (0, 2):
            got = gemm(prec, a, w).astype(np.float64) / fac
            e = np.abs(got - ref)
            print(f"K={K:5d} {name:12s} prec={prec} max_rel={e.max()/scale:.2e} rms_rel={np.sqrt((e**2).mean())/scale:.2e}")
    # exactly representable inputs: isolates accumulation error
    Ah = A.astype(np.float16).astype(np.float32); Wh = (W * 1024).astype(np.float16).astype(np.float32)
    r2 = Ah.astype(np.float64) @ Wh.astype(np.float64)
    got = gemm(1, Ah, Wh).astype(np.float64)  # bf16 mode would round; use prec 0 (lo==0)
    got0 = gemm(0, Ah, Wh).astype(np.float64)
    s2 = np.abs(r2).std()
    print(f"K={K:5d} exact-fp16 inputs prec0 max_rel={np.abs(got0-r2).max()/s2:.2e} rms_rel={np.sqrt(((got0-r2)**2).mean())/s2:.2e}")
    # fp32 reference accumulation error for comparison
    f32 = (A @ W).astype(np.float64)
    print(f"K={K:5d} numpy-fp32 sgemm   max_rel={np.abs(f32-ref).max()/scale:.2e}")
