"""End-to-end parity of the device path (Evaluator -> libmfhost -> libmfgpu)
against the reference's own numbers (tests/golden/reference_vectors.json,
produced by running metricforge; tests/golden/eval_qe.txt shipped by it) and
against the CPU oracle on the same seeded inputs.

Tolerances (north star): |Δ| <= 1e-3 per segment for the fp32-parity path.
The tiny fixtures are checked much tighter: operands travel as fp16 hi/lo
pairs (~22 significant bits) and the residual stream, LayerNorm, softmax and
pooling stay fp32."""

import math
import os

import numpy as np
import pytest

import paper_2408_11853_b200 as mf
from oracle import evaluate as oe
from oracle import fixtures as fx
from oracle import tokenizer as otk
from oracle.encoder import OracleModel

from conftest import parity_log, write_model

pytestmark = pytest.mark.gpu

PARITY_TOL = 1e-3


def make_ev(fixture, **kw):
    kw.setdefault("quiet", True)
    return mf.Evaluator(mf.EvaluatorConfig(model=fixture.model, vocab=fixture.vocab, **kw))


@pytest.mark.parametrize("key", ["comet-qe/post", "comet-qe/pre", "comet/post", "comet/pre",
                                 "bleurt/post", "bleurt/pre"])
def test_tiny_models_match_reference(golden, tiny_factory, key):
    g = golden["tiny"][key]
    kind, style = key.split("/")
    fix = tiny_factory(kind, style, g["seed"])
    with make_ev(fix) as ev:
        got = ev.evaluate_lines(g["lines"])
    d = np.abs(np.array(got.segment_scores) - np.array(g["fp32"]))
    parity_log(f"tiny/{key}", max_abs=float(d.max()), mean_abs=float(d.mean()))
    assert d.max() <= 1e-5, d.max()  # the reference's ORACLE_TOL (test_acceptance.py:46)
    assert abs(got.system_score - g["fp32_system"]) <= 2e-5


def test_golden_eval_qe_txt(golden, tiny_factory):
    """The reference's byte-stable CLI golden (pkg/tests/golden/eval_qe.txt)."""
    from pathlib import Path
    g = golden["tiny"]["comet-qe/post"]
    fix = tiny_factory("comet-qe", "post", 1234)
    with make_ev(fix) as ev:
        rep = ev.evaluate_lines(g["lines"])
    text = "".join(f"{v:.4f}\n" for v in rep.segment_scores)
    want = (Path(__file__).parent / "golden" / "eval_qe.txt").read_text()
    assert text == want


def test_config1_thousand_triplets(golden, fixture_dir, vocab_path):
    c1 = fx.CONFIGS[1]
    man = fx.tiny_manifest("comet", **{k: c1[k] for k in
                                       ("d_model", "n_heads", "n_layers", "d_ffn", "head_hidden")})
    w = fx.fixture_weights(man, 1234)
    path = write_model(fixture_dir / "config1.mfrg", man, w)
    lines = fx.fixture_tsv_lines("comet", 1000, seed=0)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True)) as ev:
        rep = ev.evaluate_lines(lines)
    ref = np.array(golden["config1"]["scores"])
    d = np.abs(np.array(rep.segment_scores) - ref)
    parity_log("config1/1000", max_abs=float(d.max()), mean_abs=float(d.mean()),
               system_abs=abs(rep.system_score - golden["config1"]["system"]))
    assert d.max() <= PARITY_TOL, d.max()
    assert abs(rep.system_score - golden["config1"]["system"]) <= 1e-4


def test_midsize_xlmr_widths(golden, fixture_dir):
    """d=1024 / 16 heads / d_ffn=4096 widths (2 layers) with BERT-scale weights."""
    g = golden["midsize"]
    man = g["manifest"]
    path = write_model(fixture_dir / "mid.mfrg", man, dict(fx.synthetic_weights(man)))
    vpath = fx.write_vocab(fixture_dir / "mid_vocab.txt", fx.synthetic_vocab_lines(man["vocab_size"]))
    for prec, tol in (("fp32", 5e-5), ("bf16x3", 2e-4), ("bf16", 5e-2)):
        with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vpath, quiet=True,
                                             precision=prec)) as ev:
            rep = ev.evaluate_lines(g["lines"])
        d = np.abs(np.array(rep.segment_scores) - np.array(g["scores"]))
        assert d.max() <= tol, (prec, d.max())


def test_oracle_equivalence_family(tmp_path, vocab_path):
    """The reference's acceptance family (test_acceptance.py:69-126): 50 random
    tiny models (d <= 32, 1-3 layers, pre/post, all kinds), 20 records each."""
    rng = np.random.default_rng(20240917)
    kinds = ["comet-qe", "comet", "bleurt"]
    ov = otk.OracleVocab(fx.fixture_vocab_lines())
    worst = 0.0
    for i in range(50):
        heads = int(rng.choice([1, 2, 4]))
        d = heads * int(rng.choice([4, 8]))
        man = fx.tiny_manifest(kinds[i % 3], d_model=d, n_heads=heads,
                               n_layers=int(rng.integers(1, 4)), d_ffn=2 * d, max_position=64,
                               norm_style=str(rng.choice(["pre", "post"])),
                               head_hidden=[[8], [16], [16, 8]][int(rng.integers(0, 3))])
        w = fx.fixture_weights(man, int(rng.integers(0, 2 ** 31)))
        path = write_model(tmp_path / f"m{i}.mfrg", man, w)
        lines = fx.fixture_tsv_lines(man["like"], 20, seed=i)
        want, _ = oe.score_lines(OracleModel(man, w), ov, lines, max_len=64)
        with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True,
                                             max_len=64)) as ev:
            got = ev.evaluate_lines(lines).segment_scores
        worst = max(worst, float(np.abs(np.array(got) - np.array(want)).max()))
    parity_log("acceptance_family/50", max_abs=worst)
    assert worst <= 1e-5, worst  # the reference's ORACLE_TOL (test_acceptance.py:46)


def test_batch_composition_is_bitwise_invisible(tiny_qe):
    lines = fx.fixture_tsv_lines("comet-qe", 1000, seed=314)
    with make_ev(tiny_qe, batch=mf.BatchConfig(mini_batch=1, maxi_batch_factor=1,
                                               sort_by_length=False)) as ev:
        seq = ev.evaluate_lines(lines).segment_scores
    with make_ev(tiny_qe, batch=mf.BatchConfig(mini_batch=128, maxi_batch_factor=8,
                                               workers=4)) as ev:
        bat = ev.evaluate_lines(lines).segment_scores
    assert seq == bat


def test_small_chunks_are_bitwise_invisible(tiny_comet):
    lines = fx.fixture_tsv_lines("comet", 300, seed=5)
    with make_ev(tiny_comet) as ev:
        a = ev.evaluate_lines(lines).segment_scores
    with make_ev(tiny_comet, max_tokens=256) as ev:  # forces many device chunks
        b = ev.evaluate_lines(lines).segment_scores
    assert a == b


def test_permutation_permutes_scores(tiny_qe):
    lines = fx.fixture_tsv_lines("comet-qe", 20, seed=5)
    with make_ev(tiny_qe) as ev:
        fwd = ev.evaluate_lines(lines).segment_scores
        rev = ev.evaluate_lines(lines[::-1]).segment_scores
    assert rev == fwd[::-1]


def test_zero_head_passes_final_bias(tmp_path, vocab_path, golden):
    man = fx.tiny_manifest("comet-qe")
    w = fx.fixture_weights(man, 3)
    for k in ("head.0.w", "head.0.b", "head.1.w"):
        w[k] = np.zeros_like(w[k])
    w["head.1.b"] = np.full_like(w["head.1.b"], 0.625)
    path = write_model(tmp_path / "zh.mfrg", man, w)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True)) as ev:
        assert ev.evaluate_lines(["north wind\tthe sun"]).segment_scores == [0.625]
    assert golden["zero_head"]["scores"] == [0.625]


def test_zero_weights_give_norm_bias(tmp_path, vocab_path):
    """All-zero weights, unit gains: every state equals the last norm bias, so
    with an identity-like head the score is a known linear function of it."""
    man = fx.tiny_manifest("bleurt", n_layers=1, head_hidden=[])
    w = {n: np.zeros(s, np.float32) for n, s in fx.tensor_shapes(man)}
    for n in w:
        if n.endswith(".g"):
            w[n][:] = 1
    bias = np.linspace(-1, 1, man["d_model"]).astype(np.float32)
    w["layer.0.norm2.b"] = bias
    w["head.0.w"] = np.ones((man["d_model"], 1), np.float32)
    path = write_model(tmp_path / "z.mfrg", man, w)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True)) as ev:
        s = ev.evaluate_lines(["the sun\tnorth"]).segment_scores[0]
    assert abs(s - float(bias.sum())) <= 1e-6


def test_score_records_seam_and_errors(tiny_qe):
    model = mf.GpuScoringModel(tiny_qe.model)
    vocab = mf.load_vocab(tiny_qe.vocab)
    recs = list(mf.records_from_tsv_lines(["north wind\tthe sun", "a\tb"], mf.Kind.COMET_QE))
    enc = [mf.encode_fields(vocab, r, "comet-qe", 128) for r in recs]
    s = model.score_records(enc)
    assert s.dtype == np.float32 and s.shape == (2,)
    bad = [[mf.TokenSequence([2, 64, 3]), mf.TokenSequence([2, 3])]]
    with pytest.raises(ValueError, match="out of range"):
        model.score_records(bad)
    long = [[mf.TokenSequence([2] * 129), mf.TokenSequence([2, 3])]]
    with pytest.raises(ValueError, match="exceeds limit"):
        model.score_records(long)
    model.close()


def test_bf16_path_error_report(golden, tiny_factory):
    g = golden["tiny"]["comet/post"]
    fix = tiny_factory("comet", "post", g["seed"])
    with make_ev(fix, precision="bf16") as ev:
        got = np.array(ev.evaluate_lines(g["lines"]).segment_scores)
    ref = np.array(g["fp32"])
    d = np.abs(got - ref)
    assert d.max() <= 5e-2 and d.mean() <= 1e-2
    assert np.corrcoef(got, ref)[0, 1] > 0.99


def test_fp16_flag_stays_within_reference_bound(golden, tiny_factory):
    """The reference's fp16 guarantee (test_acceptance.py:159-180): segment <= 5e-2,
    system <= 1e-2 vs fp32."""
    g = golden["tiny"]["comet-qe/post"]
    fix = tiny_factory("comet-qe", "post", 1234)
    lines = fx.fixture_tsv_lines("comet-qe", 200, seed=11)
    with make_ev(fix) as ev:
        r32 = ev.evaluate_lines(lines)
    with make_ev(fix, compute_mode="fp16") as ev:
        r16 = ev.evaluate_lines(lines)
    d = np.abs(np.array(r32.segment_scores) - np.array(r16.segment_scores))
    assert d.max() <= 5e-2 and abs(r32.system_score - r16.system_score) <= 1e-2


@pytest.mark.parametrize("key", ["comet-qe/post", "comet-qe/pre", "comet/post", "comet/pre",
                                 "bleurt/post", "bleurt/pre"])
def test_fp16_mode_matches_reference_fp16(golden, tiny_factory, key):
    """`fp16=True` runs the reference's binary16 semantics on the device (fp16
    MMAs, binary16 rounding at every reference rounding point): scores agree with
    the reference's own fp16 path far inside its fp32 bound (5e-2)."""
    g = golden["tiny"][key]
    kind, style = key.split("/")
    fix = tiny_factory(kind, style, g["seed"])
    with make_ev(fix, compute_mode="fp16") as ev:
        assert ev.model.precision == "fp16"
        got = ev.evaluate_lines(g["lines"])
    d = np.abs(np.array(got.segment_scores) - np.array(g["fp16"]))
    assert d.max() <= 2e-3, d.max()
    assert abs(got.system_score - g["fp16_system"]) <= 1e-3


def test_fp16_mode_midsize_vs_oracle_fp16(golden, fixture_dir):
    """XLM-R widths (d 1024, 16 heads, ffn 4096, 2 layers): device fp16 mode vs
    the oracle's fp16 mode (pinned to the reference in test_oracle.py)."""
    g = golden["midsize"]
    man = g["manifest"]
    w = dict(fx.synthetic_weights(man))
    path = write_model(fixture_dir / "mid16.mfrg", man, w)
    vpath = fx.write_vocab(fixture_dir / "mid16_vocab.txt", fx.synthetic_vocab_lines(man["vocab_size"]))
    lines = g["lines"][:24]
    want, _ = oe.score_lines(OracleModel(man, w, mode="fp16"),
                             otk.OracleVocab(fx.synthetic_vocab_lines(man["vocab_size"])), lines)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vpath, quiet=True,
                                         compute_mode="fp16")) as ev:
        got = ev.evaluate_lines(lines).segment_scores
    d = np.abs(np.array(got) - np.array(want))
    assert d.max() <= 2e-3, d.max()


def test_empty_and_degenerate_inputs(tiny_comet):
    """No records -> empty report (system None); empty fields ([BOS EOS] only),
    a single record and one record per window all score like the oracle."""
    with make_ev(tiny_comet) as ev:
        rep = ev.evaluate_lines([])
        assert rep.segment_scores == [] and rep.system_score is None
    lines = ["\t\t", "a\t\t", "\tb\t", "the cat\t\tthe"]
    want, _ = oe.score_lines(OracleModel(tiny_comet.manifest, tiny_comet.weights),
                             otk.OracleVocab(fx.fixture_vocab_lines()), lines)
    with make_ev(tiny_comet) as ev:
        got = ev.evaluate_lines(lines).segment_scores
        one = [ev.evaluate_lines([ln]).segment_scores[0] for ln in lines]
    assert np.abs(np.array(got) - np.array(want)).max() <= 5e-5
    assert got == one  # bitwise: a record's score does not depend on its window


def test_long_and_short_sequences_at_xlmr_width(golden, fixture_dir):
    """d 1024 / 16 heads with sequences of 2..400 tokens in one window: packed
    128-row tiles, the two-pass long-sequence kernel, the BOS-only last layer and
    max_len truncation all against the oracle (fp32 parity path)."""
    man = dict(golden["midsize"]["manifest"], max_position=512)
    w = dict(fx.synthetic_weights(man))
    path = write_model(fixture_dir / "mid_long.mfrg", man, w)
    vlines = fx.synthetic_vocab_lines(man["vocab_size"])
    vpath = fx.write_vocab(fixture_dir / "mid_long_vocab.txt", vlines)
    rng = np.random.default_rng(5)
    n_words = man["vocab_size"] - len(fx.SPECIALS)

    def text(n):
        return " ".join(f"w{i}" for i in rng.integers(0, n_words, n))

    sizes = [0, 1, 30, 126, 127, 128, 200, 300, 398, 600]
    lines = ["\t".join(text(int(rng.choice(sizes))) for _ in range(3)) for _ in range(12)]
    want, _ = oe.score_lines(OracleModel(man, w), otk.OracleVocab(vlines), lines, max_len=512)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vpath, quiet=True)) as ev:
        got = ev.evaluate_lines(lines).segment_scores
    d = np.abs(np.array(got) - np.array(want))
    assert d.max() <= 5e-5, d.max()


def _scaled_tiny(tmp_path, kind, mat_scale, emb_scale, name):
    man = fx.tiny_manifest(kind, d_model=64, n_heads=2, d_ffn=128)
    w = fx.fixture_weights(man, 77)
    for k in w:
        if k.endswith(".w") and not k.startswith("head."):
            w[k] = (w[k] * np.float32(mat_scale)).astype(np.float32)
        elif k == "emb.tok":
            w[k] = (w[k] * np.float32(emb_scale)).astype(np.float32)
    return man, w, write_model(tmp_path / name, man, w)


def test_fp32_path_small_weights_keep_precision(tmp_path, vocab_path):
    """Weights ~1e-4 (the fp16 lo piece of an unscaled weight would be subnormal):
    the per-column power-of-two prescale keeps ~22 bits, no fallback needed."""
    man, w, path = _scaled_tiny(tmp_path, "comet", 4e-4, 1.0, "small.mfrg")
    lines = fx.fixture_tsv_lines("comet", 40, seed=3)
    want, _ = oe.score_lines(OracleModel(man, w), otk.OracleVocab(fx.fixture_vocab_lines()), lines)
    err = {}
    for on in ("1", "0"):  # with / without the prescale (MFG_WEIGHT_PRESCALE: A/B switch)
        os.environ["MFG_WEIGHT_PRESCALE"] = on
        try:
            with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True)) as ev:
                got = ev.evaluate_lines(lines).segment_scores
                st = ev.model.stats()
        finally:
            del os.environ["MFG_WEIGHT_PRESCALE"]
        err[on] = float(np.abs(np.array(got) - np.array(want)).max())
        assert st["fallback_chunks"] == 0
    parity_log("small_weights", max_abs=err["1"], max_abs_unscaled=err["0"])
    assert err["1"] <= 1e-4 and err["1"] < err["0"], err


def test_fp32_path_huge_activations_fall_back_not_fail(tmp_path, vocab_path):
    """Embeddings ~1e5 (beyond the fp16 range of the operand pieces) and weights
    ~1e-4: the default path re-scores the chunk with bf16 hi/lo pieces instead
    of raising (the reference computes in fp32 with no range limit)."""
    man, w, path = _scaled_tiny(tmp_path, "comet", 4e-4, 4e5, "huge.mfrg")
    assert np.abs(w["emb.tok"]).max() >= 1e5
    lines = fx.fixture_tsv_lines("comet", 40, seed=3)
    want, _ = oe.score_lines(OracleModel(man, w), otk.OracleVocab(fx.fixture_vocab_lines()), lines)
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True,
                                         max_tokens=1024)) as ev:
        got = ev.evaluate_lines(lines).segment_scores
        st = ev.model.stats()
    d = float(np.abs(np.array(got) - np.array(want)).max())
    parity_log("huge_activations", max_abs=d, fallback_chunks=st["fallback_chunks"])
    assert st["fallback_chunks"] >= 1 and st["fallback_records"] >= 1
    assert d <= 1e-3, d
