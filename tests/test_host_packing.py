"""libmfhost (C++ tokenizer, planner, packer) is bit-exact against the
reference's goldens and the oracle, including the reference's own property
tests (`pkg/tests/test_vocab.py:110-248`, `test_batching.py:41-72`)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2408_11853_b200 as mf
from oracle import batching as obt
from oracle import evaluate as oe
from oracle import fixtures as fx
from oracle import tokenizer as otk
from paper_2408_11853_b200.batching import pack_roles, plan_order
from paper_2408_11853_b200.errors import ColumnCountError, MissingFieldError, VocabularyError

MARK = "▁"
WHITESPACE = [0x9, 0xA, 0xB, 0xC, 0xD, 0x1C, 0x1D, 0x1E, 0x1F, 0x20, 0x85, 0xA0, 0x1680,
              *range(0x2000, 0x200B), 0x2028, 0x2029, 0x202F, 0x205F, 0x3000]


def test_golden_tokenizer_cases(golden):
    fixture = mf.Vocabulary(fx.fixture_vocab_lines())
    for case in golden["tokenizer_cases"]:
        v = fixture if case["vocab"] == "fixture" else mf.Vocabulary(fx.SPECIALS + case["vocab"])
        assert v.encode(case["text"]) == case["ids"], case


@pytest.mark.parametrize("kind", ["comet-qe", "comet", "bleurt"])
@pytest.mark.parametrize("max_len", [128, 8, 5, 3])
def test_golden_encode_fields(golden, kind, max_len):
    d = golden["encode_fields"][kind]
    v = mf.Vocabulary(fx.fixture_vocab_lines())
    k = mf.Kind.parse(kind)
    recs = list(mf.records_from_tsv_lines(d["lines"], k))
    ids, off = v.encode_batch(k, [r.field_values(k) for r in recs], max_len, n_threads=3)
    ns = (len(off) - 1) // len(recs)
    got = [[ids[off[i * ns + j]:off[i * ns + j + 1]].tolist() for j in range(ns)]
           for i in range(len(recs))]
    assert got == d[str(max_len)]
    # the single-record seam gives the same
    assert [s.ids for s in mf.encode_fields(v, recs[0], kind, max_len)] == d[str(max_len)][0]


def test_golden_synthetic_250k_vocab(golden):
    v = mf.Vocabulary(fx.synthetic_vocab_lines(250002))
    lines = fx.synthetic_tsv_lines(2, 50)
    recs = list(mf.records_from_tsv_lines(lines, mf.Kind.COMET))
    ids, off = v.encode_batch(mf.Kind.COMET, [r.field_values(mf.Kind.COMET) for r in recs], 512)
    got = [[ids[off[i * 3 + j]:off[i * 3 + j + 1]].tolist() for j in range(3)] for i in range(50)]
    assert got == golden["synthetic_ids"]["ids"]


@st.composite
def vocab_and_text(draw):
    pieces = draw(st.lists(st.text(alphabet="abcde" + MARK + "é北", min_size=1, max_size=4)
                           .filter(lambda t: t not in fx.SPECIALS), min_size=1, max_size=12,
                           unique=True))
    words = draw(st.lists(st.text(alphabet="abcdef北é", min_size=1, max_size=6), max_size=6))
    seps = draw(st.lists(st.sampled_from([" ", "\t", "  ", "　", " ", "\x1c", "\xa0"]),
                         min_size=len(words) + 1, max_size=len(words) + 1))
    text = seps[0] + "".join(w + s for w, s in zip(words, seps[1:]))
    return pieces, text


def _brute(stream, tokens):
    ids, i = [], 0
    while i < len(stream):
        best = None
        for t in tokens:
            if stream.startswith(t, i) and (best is None or len(t) > len(best)):
                best = t
        if best is None:
            ids.append(1)
            i += 1
        else:
            ids.append(tokens[best])
            i += len(best)
    return ids


@settings(max_examples=300, deadline=None)
@given(data=vocab_and_text())
def test_matches_brute_force_segmenter(data):
    pieces, text = data
    v = mf.Vocabulary(fx.SPECIALS + pieces)
    words = text.split()
    stream = MARK + MARK.join(words) if words else ""
    tokens = {p: i + 5 for i, p in enumerate(pieces)}
    assert v.encode(text) == _brute(stream, tokens) == otk.OracleVocab(fx.SPECIALS + pieces).encode(text)


@st.composite
def closed_vocab_and_text(draw):
    """Pieces with the marker only in front (the C++ whole-word fast path), long
    pieces (> 16 UTF-8 bytes) included, words that are / are not whole pieces."""
    body = st.text(alphabet="abcdé北", min_size=1, max_size=7)
    pieces = draw(st.lists(st.tuples(st.booleans(), body).map(lambda t: (MARK if t[0] else "") + t[1]),
                           min_size=1, max_size=14, unique=True))
    pieces = [p for p in pieces if p not in fx.SPECIALS]
    words = draw(st.lists(st.one_of(st.sampled_from([p.lstrip(MARK) for p in pieces] or ["a"]),
                                    st.text(alphabet="abcdé北", min_size=1, max_size=9)),
                          max_size=8))
    return pieces, " ".join(words)


@settings(max_examples=300, deadline=None)
@given(data=closed_vocab_and_text())
def test_whole_word_fast_path_matches_brute_force(data):
    pieces, text = data
    if not pieces:
        return
    v = mf.Vocabulary(fx.SPECIALS + pieces)
    words = text.split()
    stream = MARK + MARK.join(words) if words else ""
    tokens = {p: i + 5 for i, p in enumerate(pieces)}
    assert v.encode(text) == _brute(stream, tokens)


def test_python_whitespace_set_exactly():
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "a", MARK + "b"])
    a, b = 5, 6
    for cp in WHITESPACE:
        assert v.encode("a" + chr(cp) + "b") == [a, b], hex(cp)
    for cp in (0x200B, 0x180E, 0xFEFF, 0x2060, 0x00AD):  # not str.isspace()
        got = v.encode("a" + chr(cp) + "b")
        assert got == otk.OracleVocab(fx.SPECIALS + [MARK + "a", MARK + "b"]).encode("a" + chr(cp) + "b")
        assert len(got) == 3, hex(cp)
    assert sorted(c for c in range(0x110000) if chr(c).isspace()) == sorted(WHITESPACE)


def test_unk_consumes_one_code_point_and_specials_never_match():
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "a"])
    assert v.encode("a§b") == [5, 1, 1]
    v2 = mf.Vocabulary(fx.SPECIALS + ["<", "pad", ">"])
    assert v2.encode("<pad>") == [1, 5, 6, 7]
    assert v2.encode("\ud800x") == otk.OracleVocab(fx.SPECIALS + ["<", "pad", ">"]).encode("\ud800x")


@settings(max_examples=200, deadline=None)
@given(n_first=st.integers(0, 30), n_second=st.integers(0, 30), max_len=st.integers(3, 40))
def test_joint_truncation_matches_stepwise_rule(n_first, n_second, max_len):
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "w"])
    rec = mf.EvalRecord(translation="w " * n_first, reference="w " * n_second)
    (seq,) = mf.encode_fields(v, rec, "bleurt", max_len)
    a, b = [5] * n_first, [5] * n_second
    while 3 + len(a) + len(b) > max_len:  # the reference's loop (vocab.py:124-128)
        if len(b) >= len(a):
            b.pop()
        else:
            a.pop()
    assert seq.ids == [2] + a + [4] + b + [3]


@settings(max_examples=150, deadline=None)
@given(kind=st.sampled_from(["comet-qe", "comet", "bleurt"]), words=st.integers(0, 40),
       max_len=st.integers(3, 64))
def test_length_bound_and_structure(kind, words, max_len):
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "w"])
    text = "w " * words
    rec = mf.EvalRecord(source=text, translation=text, reference=text)
    seqs = mf.encode_fields(v, rec, kind, max_len)
    for s in seqs:
        assert 2 <= len(s) <= max_len and s.ids[0] == 2 and s.ids[-1] == 3
    assert sum(s.ids.count(4) for s in seqs) == (1 if kind == "bleurt" else 0)


def test_max_len_errors_and_missing_field():
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "x"])
    with pytest.raises(ValueError, match="BOS, SEP and EOS"):
        mf.encode_fields(v, mf.EvalRecord(translation="x", reference="x"), "bleurt", 2)
    with pytest.raises(ValueError, match="BOS and EOS"):
        mf.encode_fields(v, mf.EvalRecord(source="x", translation="x"), "comet-qe", 1)
    with pytest.raises(MissingFieldError, match=r"record 7.*'reference'.*'comet'"):
        mf.encode_fields(v, mf.EvalRecord(source="x", translation="x", index=7), "comet", 128)


def test_load_vocab_semantics(tmp_path):
    p = tmp_path / "v.txt"
    p.write_bytes("\r\n".join(fx.SPECIALS + [MARK + "a"]).encode() + b"\r\n")  # universal newlines
    assert mf.load_vocab(str(p)).encode("a") == [5]
    p.write_text("\n".join(fx.SPECIALS + ["abc", "abc"]) + "\n", encoding="utf-8")
    with pytest.raises(VocabularyError, match="'abc'"):
        mf.load_vocab(str(p))
    p.write_text("\n".join(["<unk>", "<pad>", "<s>", "</s>", "<sep>"]) + "\n", encoding="utf-8")
    with pytest.raises(VocabularyError, match="first five"):
        mf.load_vocab(str(p))
    p.write_text("", encoding="utf-8")
    with pytest.raises(VocabularyError, match="empty"):
        mf.load_vocab(str(p))


@settings(max_examples=150, deadline=None)
@given(lengths=st.lists(st.integers(0, 50), max_size=60), mini_batch=st.integers(1, 9),
       factor=st.integers(1, 4), sort=st.booleans())
def test_plan_matches_oracle(lengths, mini_batch, factor, sort):
    cfg = mf.BatchConfig(mini_batch=mini_batch, maxi_batch_factor=factor, sort_by_length=sort)
    plan = mf.plan_batches(lengths, cfg)
    batches, order = obt.plan(lengths, mini_batch, factor, sort)
    assert plan.batches == batches and plan.order == order
    assert mf.restore_order([float(i) for i in order], plan) == [float(i) for i in range(len(lengths))]


def test_plan_known_answers():
    assert mf.plan_batches([3, 9, 9, 1], mf.BatchConfig(mini_batch=4, maxi_batch_factor=1)).order == [1, 2, 0, 3]
    assert mf.plan_batches([1, 9, 2, 8], mf.BatchConfig(mini_batch=1, maxi_batch_factor=2)).order == [1, 0, 3, 2]
    plan = mf.plan_batches([3, 9, 9, 1], mf.BatchConfig(mini_batch=4))
    assert mf.restore_order(["a", "b", "c", "d"], plan) == ["c", "a", "b", "d"]
    with pytest.raises(ValueError, match="3 scores for 2"):
        mf.restore_order([1.0, 2.0, 3.0], mf.plan_batches([1, 2], mf.BatchConfig()))


def test_pack_roles_layout():
    v = mf.Vocabulary(fx.fixture_vocab_lines())
    lines = fx.fixture_tsv_lines("comet", 37, seed=3)
    recs = list(mf.records_from_tsv_lines(lines, mf.Kind.COMET))
    ids, off = v.encode_batch(mf.Kind.COMET, [r.field_values(mf.Kind.COMET) for r in recs], 128)
    order = plan_order(np.diff(off).reshape(37, 3).sum(1), mf.BatchConfig(mini_batch=8))
    packed, cu = pack_roles(ids, off, 3, order)
    ref = oe.encode_lines(otk.OracleVocab(fx.fixture_vocab_lines()), "comet", lines, 128)
    for k in range(3):
        for i, rec in enumerate(order):
            s = k * 37 + i
            assert packed[cu[s]:cu[s + 1]].tolist() == ref[rec][k]
    assert cu[-1] == len(packed)


def test_multithreaded_encoding_is_identical():
    v = mf.Vocabulary(fx.synthetic_vocab_lines(5000))
    lines = [" ".join(f"w{(i * 7 + j) % 4995}" for j in range(i % 50)) + "\t" + "x y" for i in range(3000)]
    recs = list(mf.records_from_tsv_lines(lines, mf.Kind.COMET_QE))
    fields = [r.field_values(mf.Kind.COMET_QE) for r in recs]
    a = v.encode_batch(mf.Kind.COMET_QE, fields, 40, n_threads=1)
    b = v.encode_batch(mf.Kind.COMET_QE, fields, 40, n_threads=8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---------------------------------------------------------------- native TSV intake
_FIELD = st.text(alphabet="ab é北\r\x0b" + MARK, max_size=12)


@settings(max_examples=200, deadline=None)
@given(kind=st.sampled_from([mf.Kind.COMET_QE, mf.Kind.COMET, mf.Kind.BLEURT]),
       rows=st.lists(st.tuples(st.lists(_FIELD, min_size=1, max_size=4),
                               st.sampled_from(["", "\n", "\n\n", "\r\n"])), max_size=12),
       max_len=st.sampled_from([3, 5, 64]), threads=st.sampled_from([1, 4]))
def test_encode_tsv_matches_python_intake(kind, rows, max_len, threads):
    """mfh_encode_tsv == records_from_tsv_lines -> field_values -> encode_batch,
    including the ColumnCountError of the first bad line (`evaluate.py:117-123`)."""
    v = mf.Vocabulary(fx.SPECIALS + [MARK + "a", "b", MARK + "é北", "北", MARK + "ab"])
    lines = ["\t".join(cols) + end for cols, end in rows]
    try:
        recs = list(mf.records_from_tsv_lines(lines, kind))
        want_err = None
    except ColumnCountError as e:
        want_err = (e.line_index, e.expected, e.got)
    if want_err is not None:
        with pytest.raises(ColumnCountError) as ei:
            v.encode_tsv(kind, lines, max_len, threads, first_index=0)
        assert (ei.value.line_index, ei.value.expected, ei.value.got) == want_err
        return
    fields = [r.field_values(kind) for r in recs]
    want = v.encode_batch(kind, fields, max_len, threads)
    got = v.encode_tsv(kind, lines, max_len, threads)
    assert np.array_equal(want[0], got[0]) and np.array_equal(want[1], got[1])


def test_encode_tsv_error_index_is_global_and_first():
    v = mf.Vocabulary(fx.synthetic_vocab_lines(100))
    lines = ["w1\tw2\n"] * 5000
    lines[3100] = "w1\n"
    lines[4000] = "w1\tw2\tw3\n"
    with pytest.raises(ColumnCountError) as ei:
        v.encode_tsv(mf.Kind.COMET_QE, lines, 16, 8, first_index=2048)
    assert (ei.value.line_index, ei.value.got) == (2048 + 3100, 1)


def test_encode_tsv_large_window_matches_encode_batch():
    v = mf.Vocabulary(fx.synthetic_vocab_lines(5000))
    lines = ["\t".join(" ".join(f"w{(i * 13 + j * k) % 4995}" for j in range(1 + (i * k) % 70))
                   for k in (1, 2, 3)) + "\n" for i in range(3000)]
    recs = [r.field_values(mf.Kind.COMET) for r in mf.records_from_tsv_lines(lines, mf.Kind.COMET)]
    a = v.encode_batch(mf.Kind.COMET, recs, 48, n_threads=8)
    b = v.encode_tsv(mf.Kind.COMET, lines, 48, n_threads=8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
