"""CLI drop-in (`pkg/src/metricforge/cli.py` semantics): golden outputs, exit codes."""

import subprocess
import sys
from pathlib import Path

import pytest

from oracle import fixtures as fx

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"


def cli(*args, stdin=None):
    return subprocess.run([sys.executable, "-m", "paper_2408_11853_b200.cli", *args], cwd=ROOT,
                          input=stdin, capture_output=True, text=True, timeout=300)


def test_inspect_golden_byte_identical(tiny_qe):
    r = cli("inspect", tiny_qe.model)
    assert r.returncode == 0
    assert r.stdout == (GOLD / "inspect_qe.txt").read_text()


def test_usage_errors_exit_2(tiny_qe, tmp_path):
    r = cli("-m", tiny_qe.model, "-v", tiny_qe.vocab, "--stdin", "-s", "x.txt")
    assert r.returncode == 2 and "--stdin excludes" in r.stderr
    r = cli("-m", str(tmp_path / "nope"), "-v", tiny_qe.vocab, "--stdin", stdin="")
    assert r.returncode == 2
    r = cli("-m", tiny_qe.model, "--stdin", stdin="")
    assert r.returncode == 2 and "vocabulary" in r.stderr


@pytest.mark.gpu
def test_eval_golden_and_average(tiny_qe, tmp_path):
    lines = fx.fixture_tsv_lines("comet-qe", 20, seed=42)
    tsv = "".join(l + "\n" for l in lines)
    outs = [cli("-m", tiny_qe.model, "-v", tiny_qe.vocab, "--stdin", "--quiet", stdin=tsv) for _ in range(2)]
    assert all(o.returncode == 0 for o in outs)
    assert outs[0].stdout == outs[1].stdout == (GOLD / "eval_qe.txt").read_text()
    src, mt = tmp_path / "s.txt", tmp_path / "t.txt"
    src.write_text("".join(l.split("\t")[0] + "\n" for l in lines))
    mt.write_text("".join(l.split("\t")[1] + "\n" for l in lines))
    r = cli("-m", tiny_qe.model, "-v", tiny_qe.vocab, "-s", str(src), "-t", str(mt), "-a", "only", "--quiet")
    assert r.returncode == 0 and len(r.stdout.splitlines()) == 1
    mt.write_text("just one line\n")
    r = cli("-m", tiny_qe.model, "-v", tiny_qe.vocab, "-s", str(src), "-t", str(mt))
    assert r.returncode == 2 and "disagree at line 2" in r.stderr
    r = cli("-m", tiny_qe.model, "-v", tiny_qe.vocab, "--stdin", stdin="a\tb\tc\n")
    assert r.returncode == 2 and "line 0" in r.stderr
