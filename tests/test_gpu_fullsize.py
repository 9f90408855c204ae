"""Parity at BASELINE.json's full model sizes (configs 2-5) against the
REFERENCE itself: `tests/golden/fullsize_cfg<N>.json` holds the scores the
unmodified reference `Evaluator` (`pkg/src/metricforge/evaluate.py:126-241`,
fp32 and its fp16 mode) produced on a length-stratified subset of each
config's synthetic workload (512 records at configs 2-4, 64
at config 5; `tests/golden/make_fullsize_golden.py`). The model and the
records are regenerated here from the committed seeds and checked against the
committed container checksum and pool indices.

Gate: fp32 path max |Δ| <= 1e-3 (north star). Reported (parity log): max /
mean |Δ| and Pearson for fp32, bf16x3, bf16 against the reference fp32, and
the fp16 mode against the reference's own fp16 mode. Plus size-independent
properties on larger samples (bitwise batch-composition invariance,
permutation equivariance, determinism)."""

import json
import os

import numpy as np
import pytest

import bench
import paper_2408_11853_b200 as mf
from oracle import fixtures as fx

from conftest import ROOT, parity_log

pytestmark = pytest.mark.gpu

TOL = 1e-3


def load_golden(c):
    p = ROOT / "tests" / "golden" / f"fullsize_cfg{c}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    with open(p) as f:
        return json.load(f)


@pytest.fixture(scope="module", params=[2, 3, 4, 5])
def cfg(request):
    c = request.param
    g = load_golden(c)
    man, path, vocab = bench.prepare_model(c, 0, 1, lambda: None)
    assert mf.read_manifest(path).checksum == g["checksum"], "regenerated weights differ"
    idx, lines = fx.parity_subset(c, g["n"], g["pool"], g["text_seed"])
    assert idx == g["pool_indices"]
    return c, g, path, vocab, lines


def stats(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    d = np.abs(got - want)
    return {"n": int(len(d)), "max_abs": float(d.max()), "mean_abs": float(d.mean()),
            "pearson": float(np.corrcoef(got, want)[0, 1])}


def score(path, vocab, lines, **kw):
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab, quiet=True, validate=False,
                                         **kw)) as ev:
        rep = ev.evaluate_lines(lines)
        fb = ev.model.stats()["fallback_chunks"]
    return rep, fb


def test_fullsize_parity_vs_reference(cfg):
    c, g, path, vocab, lines = cfg
    rep, fb = score(path, vocab, lines)
    s = stats(rep.segment_scores, g["fp32"])
    s["system_abs"] = abs(rep.system_score - g["fp32_system"])
    parity_log(f"fullsize/config{c}/fp32", fallback_chunks=fb, **s)
    assert s["max_abs"] <= TOL, s


@pytest.mark.parametrize("prec", ["bf16x3", "bf16", "fp16"])
def test_fullsize_other_precisions_reported(cfg, prec):
    c, g, path, vocab, lines = cfg
    if prec == "fp16" and "fp16" not in g:
        pytest.skip("reference fp16 scores not generated")
    rep, _ = score(path, vocab, lines, precision=prec)
    s = stats(rep.segment_scores, g["fp32"])
    if prec == "fp16":
        s["vs_reference_fp16_mode"] = stats(rep.segment_scores, g["fp16"])
    parity_log(f"fullsize/config{c}/{prec}", **s)
    if prec == "bf16x3":
        assert s["max_abs"] <= TOL, s
    elif prec == "fp16":  # the reference's own fp16 bound vs fp32 is 5e-2
        assert s["vs_reference_fp16_mode"]["max_abs"] <= 1e-2, s
    else:
        assert s["pearson"] > 0.99, s


def test_fullsize_invariances(cfg):
    c, g, path, vocab, lines = cfg
    n = 64 if c < 5 else 24
    lines = bench.workload_lines(c, n, fx.TEXT_SEED + 9)
    conf = dict(model=path, vocab=vocab, quiet=True, validate=False)
    with mf.Evaluator(mf.EvaluatorConfig(**conf)) as ev:
        a = ev.evaluate_lines(lines).segment_scores
        again = ev.evaluate_lines(lines).segment_scores
        rev = ev.evaluate_lines(lines[::-1]).segment_scores
    assert a == again and rev == a[::-1]
    with mf.Evaluator(mf.EvaluatorConfig(batch=mf.BatchConfig(mini_batch=3, maxi_batch_factor=2,
                                                              sort_by_length=False),
                                         max_tokens=4096, **conf)) as ev:
        b = ev.evaluate_lines(lines).segment_scores
    assert a == b


def test_fullsize_split_paths_agree_beyond_the_golden_subset(cfg):
    """Size-independent check on records the golden subset does not hold: the
    fp16-pieces parity path and the independent bf16-pieces path (same fp32 math,
    different operand representation) agree far inside the 1e-3 gate
    (profiles/tail_r03.txt: 3.5e-5 over all 100k config-2 records)."""
    c, g, path, vocab, _ = cfg
    n = 4096 if c < 5 else 512
    lines = bench.workload_lines(c, n, fx.TEXT_SEED + 4242)
    got = {}
    for prec in ("fp32", "bf16x3"):
        rep, fb = score(path, vocab, lines, precision=prec)
        assert fb == 0
        got[prec] = np.asarray(rep.segment_scores, np.float64)
    d = np.abs(got["fp32"] - got["bf16x3"])
    parity_log(f"fullsize/config{c}/fp32_vs_bf16x3", n=n, max_abs=float(d.max()),
               mean_abs=float(d.mean()))
    assert d.max() <= 3e-4, d.max()
