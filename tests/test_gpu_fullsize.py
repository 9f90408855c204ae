"""Parity at BASELINE.json's full model sizes (configs 2-5): the device path
vs the CPU oracle on a bounded sample of each config's synthetic workload
(max |Δ| <= 1e-3, the north-star tolerance), plus size-independent
properties on larger samples (bitwise batch-composition invariance,
permutation equivariance, determinism)."""

import numpy as np
import pytest

import bench
import paper_2408_11853_b200 as mf
from oracle import evaluate as oe
from oracle import fixtures as fx

pytestmark = pytest.mark.gpu

SAMPLE = {2: 6, 3: 6, 4: 6, 5: 2}


@pytest.fixture(scope="module", params=[2, 3, 4, 5])
def cfg(request):
    man, path, vocab = bench.prepare_model(request.param, 0, 1, lambda: None)
    return request.param, man, path, vocab


def test_fullsize_parity_vs_oracle(cfg):
    c, man, path, vocab = cfg
    lines = bench.workload_lines(c, SAMPLE[c], fx.TEXT_SEED + 5)
    model, ovocab = bench.oracle_model(c)
    want, _ = oe.score_lines(model, ovocab, lines)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab, quiet=True, validate=False)) as ev:
        got = ev.evaluate_lines(lines).segment_scores
    d = np.abs(np.array(got) - np.array(want))
    assert d.max() <= 1e-3, (c, d.max())


def test_fullsize_invariances(cfg):
    c, man, path, vocab = cfg
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
