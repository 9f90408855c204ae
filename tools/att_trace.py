"""Per-item timeline of the tcgen05 attention kernel (clock64 trace of the
first 4 CTAs) on a config-2-shaped batch: 3072 sequences ~U{3..128}, d 1024,
16 heads.  python tools/att_trace.py  (GPU box)"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_11853_b200 import native

lib = native.gpu()
rng = np.random.default_rng(0)
lens = rng.integers(3, 129, 3072).astype(np.int32)
cu = np.zeros(len(lens) + 1, np.int32)
cu[1:] = np.cumsum(lens)
T, d, H = int(cu[-1]), 1024, 16
qkv = (0.5 * rng.standard_normal((T, 3 * d))).astype(np.float32)
out = np.zeros((T, d), np.float32)
P = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
lib.mfgt_attention(0, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H, P(qkv), P(out), 1)
buf = np.zeros(4 * 64 * 8, np.int64)
assert lib.mfgt_att_trace(1, None) == 0
assert lib.mfgt_attention(0, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H, P(qkv), P(out), 1) == 0
assert lib.mfgt_att_trace(0, buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
tr = buf.reshape(4, 64, 8)
names = ["S_iss", "O_iss", "S_seen", "P_done", "O_epi", "epi_done"]
for cta in range(2):
    t0 = tr[cta, 0, 0]
    print(f"CTA {cta} (cycles from first S issue)")
    print("  k " + " ".join(f"{n:>8}" for n in names))
    for k in range(40):
        row = tr[cta, k, :6]
        print(f"{k:3d} " + " ".join(f"{(v - t0) if v else -1:8d}" for v in row))
d_ = tr[:, 4:60, :]
print("mean per-item deltas (cycles): S_seen-S_iss %.0f, P_done-S_seen %.0f, O_iss-P_done %.0f, "
      "O_seen-O_iss %.0f, done-O_seen %.0f, item period %.0f" % (
          (d_[..., 2] - d_[..., 0]).mean(), (d_[..., 3] - d_[..., 2]).mean(),
          (d_[..., 1] - d_[..., 3]).mean(), (d_[..., 4] - d_[..., 1]).mean(),
          (d_[..., 5] - d_[..., 4]).mean(), np.diff(tr[:, 4:60, 0], axis=1).mean()))

# wall time of the same launch (CUDA events around mfgt_attention's kernel are not
# exposed; time the whole call minus its H2D by repeating it)
import time
import torch
lib.mfgt_attention(0, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H, P(qkv), P(out), 1)
t0 = time.perf_counter()
for _ in range(5):
    lib.mfgt_attention(0, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H, P(qkv), P(out), 1)
print("mfgt_attention call (incl. H2D/D2H of %.0f MB): %.2f ms" % (qkv.nbytes / 1e6, (time.perf_counter() - t0) / 5 * 1e3))
starts = tr[:, :, 0]
ends = tr[:, :, 5]
for cta in range(4):
    n = int((tr[cta, :, 0] > 0).sum())
    print(f"CTA {cta}: {n} traced items, first S issue -> last epilogue {ends[cta, n-1] - starts[cta, 0]} cycles")
