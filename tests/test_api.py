"""Drop-in API surface of the Evaluator (`pkg/src/metricforge/evaluate.py`):
config mapping, errors raised before any device work, averages, TSV intake.
Mirrors the reference's tests/test_evaluate.py cases that need no GPU."""

import math

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2408_11853_b200 as mf
from paper_2408_11853_b200.errors import (
    ColumnCountError,
    EmptyReportError,
    KindMismatchError,
    MissingFieldError,
    UnknownMetricError,
    VocabRequiredError,
)


def test_config_parsing():
    c = mf.EvaluatorConfig(model="m", compute_mode="fp16", average_mode="only", like="comet")
    assert c.compute_mode is mf.ComputeMode.FP16 and c.like is mf.Kind.COMET
    assert c.average_mode is mf.AverageMode.ONLY
    with pytest.raises(ValueError, match="max_len"):
        mf.EvaluatorConfig(model="m", max_len=1)
    with pytest.raises(ValueError, match="unknown average mode"):
        mf.EvaluatorConfig(model="m", average_mode="median")
    with pytest.raises(ValueError, match="unknown metric kind"):
        mf.EvaluatorConfig(model="m", like="bert")
    with pytest.raises(ValueError):
        mf.BatchConfig(mini_batch=0)


def test_new_rejects_unknown_keyword_by_name(tiny_qe):
    with pytest.raises(TypeError, match="beam_size"):
        mf.Evaluator.new(model_file=tiny_qe.model, vocab_file=tiny_qe.vocab, beam_size=5)


def test_errors_before_device_work(tiny_qe, tmp_path):
    with pytest.raises(VocabRequiredError):
        mf.Evaluator(mf.EvaluatorConfig(model=tiny_qe.model))
    with pytest.raises(KindMismatchError, match="comet'.*comet-qe'|comet-qe'.*'comet"):
        mf.Evaluator(mf.EvaluatorConfig(model=tiny_qe.model, vocab=tiny_qe.vocab, like="comet"))
    with pytest.raises(UnknownMetricError):
        mf.Evaluator(mf.EvaluatorConfig(model=str(tmp_path / "nope"), vocab=tiny_qe.vocab))


def test_records_from_tsv():
    recs = list(mf.records_from_tsv_lines(["a \t b\n"], mf.Kind.COMET_QE))
    assert recs[0].source == "a " and recs[0].translation == " b"
    assert len(list(mf.records_from_tsv_lines(["t\tr"], mf.Kind.BLEURT))) == 1
    with pytest.raises(ColumnCountError, match="line 1.*expected 2.*got 3"):
        list(mf.records_from_tsv_lines(["ok\tok", "one\ttwo\tthree"], mf.Kind.COMET_QE))
    with pytest.raises(MissingFieldError, match="record 3.*'reference'"):
        mf.EvalRecord(source="a", translation="b").field_values(mf.Kind.COMET, 3)


def test_empty_report_and_modes():
    rep = mf.ScoreReport(segment_scores=[])
    assert rep.system_score is None
    assert mf.apply_average_mode(rep, "skip") == []
    for mode in ("only", "append"):
        with pytest.raises(EmptyReportError):
            mf.apply_average_mode(rep, mode)


@settings(max_examples=80, deadline=None)
@given(st.lists(st.floats(-100, 100, allow_nan=False, allow_infinity=False, width=32),
                min_size=1, max_size=50))
def test_average_identities(scores):
    rep = mf.ScoreReport(segment_scores=list(scores))
    skip = mf.apply_average_mode(rep, "skip")
    append = mf.apply_average_mode(rep, "append")
    only = mf.apply_average_mode(rep, "only")
    assert skip == list(scores) and append[:-1] == skip
    assert append[-1] == only[0] == math.fsum(scores) / len(scores)
