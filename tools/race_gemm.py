"""The shipped CTA-pair GEMM (gemm2_tc_kernel) on small shapes that take every
code path of the production kernel — K-chunked accumulation with the L2
partial buffer (K > 4096), the relaxed remote accumulator-drained arrive, the
residual and GELU epilogues, both operand formats — for compute-sanitizer:

    compute-sanitizer --tool racecheck python tools/race_gemm.py
    compute-sanitizer --tool memcheck  python tools/race_gemm.py
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_11853_b200 import native  # noqa: E402

lib = native.gpu()
P = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
rng = np.random.default_rng(0)
for prec, epi, M, N, K in [(0, 0, 512, 512, 4352), (0, 1, 300, 1024, 1024), (0, 2, 256, 768, 256),
                           (3, 1, 512, 512, 8256), (1, 4, 384, 256, 128)]:
    A = rng.standard_normal((M, K), dtype=np.float32)
    W = (rng.standard_normal((K, N), dtype=np.float32) * 0.02).astype(np.float32)
    b = rng.standard_normal(N, dtype=np.float32)
    r = rng.standard_normal((M, N), dtype=np.float32)
    out = np.zeros((M, N), np.float32)
    rc = lib.mfgt_gemm(prec, epi, M, N, K, P(A), P(W), P(b), P(r), P(out))
    ref = A.astype(np.float64) @ W + b + (r if epi == 1 else 0)
    err = float(np.abs(out - ref).max()) if epi in (0, 1) else float("nan")
    print(f"prec {prec} epi {epi} {M}x{N}x{K}: rc {rc} max|err| {err:.2e}", flush=True)
