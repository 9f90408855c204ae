"""The CPU oracle is pinned to the reference before anything is checked against
it: every number in tests/golden/reference_vectors.json came from running
metricforge itself (tests/golden/make_golden.py), and eval_qe.txt /
inspect_qe.txt are the reference's own shipped goldens."""

import os
from pathlib import Path

import numpy as np
import pytest

from oracle import batching as obt
from oracle import evaluate as oe
from oracle import fixtures as fx
from oracle import mfrg
from oracle import tokenizer as otk
from oracle.encoder import OracleModel

GOLD = Path(__file__).parent / "golden"


def test_tokenizer_known_answers(golden):
    fixture = otk.OracleVocab(fx.fixture_vocab_lines())
    for case in golden["tokenizer_cases"]:
        v = fixture if case["vocab"] == "fixture" else otk.OracleVocab(fx.SPECIALS + case["vocab"])
        assert v.encode(case["text"]) == case["ids"], case


@pytest.mark.parametrize("kind", ["comet-qe", "comet", "bleurt"])
@pytest.mark.parametrize("max_len", ["128", "8", "5", "3"])
def test_encode_fields_match_reference(golden, kind, max_len):
    d = golden["encode_fields"][kind]
    v = otk.OracleVocab(fx.fixture_vocab_lines())
    assert oe.encode_lines(v, kind, d["lines"], int(max_len)) == d[max_len]


def test_plans_match_reference(golden):
    for p in golden["plans"]:
        batches, order = obt.plan(p["lengths"], p["mini_batch"], p["factor"], p["sort"])
        assert batches == p["batches"] and order == p["order"]


@pytest.mark.parametrize("key", ["comet-qe/post", "comet-qe/pre", "comet/post", "comet/pre",
                                 "bleurt/post", "bleurt/pre"])
@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_tiny_scores_bitwise(golden, key, mode):
    g = golden["tiny"][key]
    kind, style = key.split("/")
    man = fx.tiny_manifest(kind, norm_style=style)
    w = fx.fixture_weights(man, g["seed"])
    scores, system = oe.score_lines(OracleModel(man, w, mode), otk.OracleVocab(fx.fixture_vocab_lines()),
                                    g["lines"])
    assert scores == g[mode]
    assert system == g[mode + "_system"]


def test_reference_cli_golden_eval_qe():
    g = (GOLD / "eval_qe.txt").read_text()
    man = fx.tiny_manifest("comet-qe")
    scores, _ = oe.score_lines(OracleModel(man, fx.fixture_weights(man, 1234)),
                               otk.OracleVocab(fx.fixture_vocab_lines()),
                               fx.fixture_tsv_lines("comet-qe", 20, seed=42))
    assert "".join(f"{s:.4f}\n" for s in scores) == g


def test_container_checksums_match_reference(golden, tmp_path):
    """Our writer is byte-identical to the reference writer (same sha256)."""
    for key, g in golden["tiny"].items():
        kind, style = key.split("/")
        man = fx.tiny_manifest(kind, norm_style=style)
        w = fx.fixture_weights(man, g["seed"])
        ck = mfrg.write(tmp_path / "m.mfrg", mfrg.manifest_dict(**man),
                        [(n, "f32", w[n]) for n, _ in fx.tensor_shapes(man)])
        assert ck == g["checksum"]
    inspect = (GOLD / "inspect_qe.txt").read_text()
    assert f"checksum: {golden['tiny']['comet-qe/post']['checksum']}" in inspect


def test_config1_thousand_records(golden):
    c1 = fx.CONFIGS[1]
    man = fx.tiny_manifest("comet", **{k: c1[k] for k in
                                       ("d_model", "n_heads", "n_layers", "d_ffn", "head_hidden")})
    w = fx.fixture_weights(man, golden["config1"]["seed"])
    scores, system = oe.score_lines(OracleModel(man, w), otk.OracleVocab(fx.fixture_vocab_lines()),
                                    fx.fixture_tsv_lines("comet", 1000, seed=0))
    assert scores == golden["config1"]["scores"]
    assert system == golden["config1"]["system"]


def test_midsize_synthetic_weights(golden):
    g = golden["midsize"]
    man = g["manifest"]
    scores, _ = oe.score_lines(OracleModel(man, dict(fx.synthetic_weights(man))),
                               otk.OracleVocab(fx.synthetic_vocab_lines(man["vocab_size"])),
                               g["lines"])
    assert scores == g["scores"]


def test_synthetic_generator_ids(golden):
    v = otk.OracleVocab(fx.synthetic_vocab_lines(250002))
    got = oe.encode_lines(v, "comet", fx.synthetic_tsv_lines(2, 50), 512)
    assert got == golden["synthetic_ids"]["ids"]


def test_synthetic_lengths_follow_survey_generator():
    lines = fx.synthetic_tsv_lines(2, 2000)
    lens = np.array([[len(c.split()) for c in ln.split("\t")] for ln in lines])
    assert lens.min() >= 1 and lens.max() <= 126 and abs(lens.mean() - 63.5) < 2
    lines5 = fx.synthetic_tsv_lines(5, 2000)
    l5 = np.array([[len(c.split()) for c in ln.split("\t")] for ln in lines5])
    assert l5.max() <= 510 and 20 < np.median(l5) < 30
