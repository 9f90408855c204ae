"""Small end-to-end forward passes for compute-sanitizer (memcheck / racecheck /
synccheck): a d256 COMET model (tile attention, d_head 64, 512-K chunked GEMMs),
and the d_head-80 attention kernels (tile + long sequences) through mfgt_attention.

    compute-sanitizer --tool memcheck python tools/memcheck_e2e.py
"""
import ctypes as C
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2408_11853_b200 as mf  # noqa: E402
from oracle import fixtures as fx  # noqa: E402
from oracle import mfrg  # noqa: E402
from paper_2408_11853_b200 import native  # noqa: E402

tmp = tempfile.mkdtemp()
man = fx.tiny_manifest("comet", d_model=256, n_heads=4, n_layers=2, d_ffn=1024, head_hidden=[256])
w = fx.fixture_weights(man, 1234)
path = os.path.join(tmp, "m.mfrg")
mfrg.write(path, mfrg.manifest_dict(**man), [(n, "f32", w[n]) for n, _ in fx.tensor_shapes(man)])
vocab = fx.write_vocab(os.path.join(tmp, "v.txt"), fx.fixture_vocab_lines())
lines = fx.fixture_tsv_lines("comet", 300, seed=3)
for prec in ("fp32", "fp16", "bf16"):
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab, quiet=True, precision=prec)) as ev:
        s = ev.evaluate_lines(lines).segment_scores
    print(prec, len(s), float(np.mean(s)), flush=True)
lib = native.gpu()
P = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
for d, H, lens in [(320, 4, [511, 200, 17]), (2560, 32, [300, 9, 129])]:
    cu = np.zeros(len(lens) + 1, np.int32)
    cu[1:] = np.cumsum(lens)
    qkv = np.random.default_rng(0).standard_normal((int(cu[-1]), 3 * d)).astype(np.float32)
    out = np.zeros((int(cu[-1]), d), np.float32)
    for prec in (0, 3, 1):
        rc = lib.mfgt_attention(prec, len(lens), cu.ctypes.data_as(C.POINTER(C.c_int32)), d, H,
                                P(qkv), P(out), 1)
        print("attention", d, H, lens, prec, rc, flush=True)
