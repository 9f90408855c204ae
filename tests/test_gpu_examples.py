"""examples/mfeval.cpp (lib/mfeval): the scoring path driven from C++ only through
the two C-ABIs (include/mfhost.h, include/mfgpu.h), as a non-Python host would
bind them. Its stdout must be byte-identical to the reference's CLI golden and
to the Python Evaluator's scores."""

import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2408_11853_b200 as mf

pytestmark = pytest.mark.gpu

EXE = Path(mf.__file__).resolve().parent / "lib" / "mfeval"


def run(args, tmp_path):
    if not EXE.exists():
        pytest.fail(f"{EXE} missing: run __graft_entry__.build()")
    return subprocess.run([str(EXE), *map(str, args)], capture_output=True, text=True, timeout=300)


def write_tsv(path, lines):
    path.write_text("".join(l + "\n" for l in lines), encoding="utf-8")
    return path


def test_reference_cli_golden_byte_identical(golden, tiny_factory, tmp_path):
    """pkg/tests/golden/eval_qe.txt, produced by the reference's own CLI."""
    g = golden["tiny"]["comet-qe/post"]
    fix = tiny_factory("comet-qe", "post", 1234)
    tsv = write_tsv(tmp_path / "in.tsv", g["lines"])
    r = run([fix.model, fix.vocab, tsv], tmp_path)
    assert r.returncode == 0, r.stderr
    want = (Path(__file__).parent / "golden" / "eval_qe.txt").read_text()
    assert r.stdout == want


@pytest.mark.parametrize("kind", ["comet", "bleurt", "comet-qe"])
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_matches_python_evaluator_bitwise(golden, tiny_factory, tmp_path, kind, prec):
    key = f"{kind}/post"
    g = golden["tiny"][key]
    fix = tiny_factory(kind, "post", g["seed"])
    # more than one window (mini-batch 4 x factor 2) and CRLF line ends
    lines = list(g["lines"]) * 3
    tsv = tmp_path / "in.tsv"
    tsv.write_bytes("".join(l + "\r\n" for l in lines).encode("utf-8"))
    r = run([fix.model, fix.vocab, tsv, "--precision", "9", "--gpu-precision", prec,
             "--mini-batch", "4", "--maxi-batch", "2"], tmp_path)
    assert r.returncode == 0, r.stderr
    cfg = mf.EvaluatorConfig(model=fix.model, vocab=fix.vocab, quiet=True, precision=prec,
                             batch=mf.BatchConfig(mini_batch=4, maxi_batch_factor=2))
    with mf.Evaluator(cfg) as ev:
        want = ev.evaluate_lines([l + "\n" for l in lines]).segment_scores
    assert r.stdout == "".join(f"{v:.9f}\n" for v in want)


def test_column_error_exit_code_and_global_index(tiny_factory, tmp_path):
    fix = tiny_factory("comet-qe", "post", 1234)
    lines = ["a b\tc d"] * 20
    lines[13] = "only one column"
    tsv = write_tsv(tmp_path / "bad.tsv", lines)
    r = run([fix.model, fix.vocab, tsv, "--mini-batch", "2", "--maxi-batch", "2"], tmp_path)
    assert r.returncode == 2
    assert "line 13: expected 2 tab-separated columns, got 1" in r.stderr
    assert r.stdout == ""


def test_empty_input_prints_nothing(tiny_factory, tmp_path):
    fix = tiny_factory("comet", "post", 1234)
    tsv = tmp_path / "empty.tsv"
    tsv.write_text("")
    r = run([fix.model, fix.vocab, tsv], tmp_path)
    assert r.returncode == 0 and r.stdout == ""
