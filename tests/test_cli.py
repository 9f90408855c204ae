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


@pytest.mark.gpu
def test_bench_table_shape_matches_reference_golden(tiny_qe):
    """`bench` prints the reference's byte-stable table (pkg/tests/golden/bench_qe.txt,
    checked by test_acceptance.py:400-420 with the value column normalised)."""
    r = cli("bench", "-m", tiny_qe.model, "-v", tiny_qe.vocab, "-n", "16", "--repeats", "1", "--fp16")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    rows = [ln.split("\t") for ln in lines[1:]]
    norm = "\n".join([lines[0]] + ["\t".join([x[0], x[1], "<value>", x[3]]) for x in rows]) + "\n"
    assert norm == (GOLD / "bench_qe.txt").read_text()
    assert all(float(x[2]) > 0 for x in rows)
    r = cli("bench", "-m", tiny_qe.model, "-v", tiny_qe.vocab, "-n", "16", "--repeats", "1",
            "--all-precisions")
    modes = [ln.split("\t")[:2] for ln in r.stdout.splitlines()[1:]]
    assert modes == [["warmup", "mmap"], ["warmup", "eager"], ["throughput", "fp32"],
                     ["throughput", "bf16x3"], ["throughput", "bf16"], ["memory", "rss"],
                     ["memory", "device"]]


def _multi(*args, stdin=None):
    import os
    env = dict(os.environ, MFG_SHARE_DEVICES="1")  # 2 ranks on the test box's GPU(s)
    return subprocess.run([sys.executable, "-m", "paper_2408_11853_b200.cli", *args], cwd=ROOT,
                          input=stdin, capture_output=True, text=True, timeout=600, env=env)


@pytest.mark.gpu
def test_multi_rank_cli_streams_stdin_like_one_gpu(tiny_factory, tmp_path):
    """--gpus 2: rank 0 streams stdin to the ranks (no spool file); the output is
    byte-identical to the single-GPU run, including a lone '\\r' inside a field
    (stdin splits only on '\\n') and a field file holding a TAB inside a field."""
    fix = tiny_factory("comet", "post", 1234)
    lines = fx.fixture_tsv_lines("comet", 700, seed=21)
    lines[5] = "the\rnorth\twind\tsun"
    tsv = "".join(l + "\n" for l in lines)
    base = ["-m", fix.model, "-v", fix.vocab, "--quiet", "--precision", "8",
            "--mini-batch", "16", "--maxi-batch", "4"]
    one = cli(*base, "--stdin", stdin=tsv)
    two = _multi(*base, "--stdin", "--gpus", "2", stdin=tsv)
    assert one.returncode == 0 and two.returncode == 0, two.stderr
    assert len(one.stdout.splitlines()) == 700 and two.stdout == one.stdout
    cols = [[l.split("\t")[k] for l in lines] for k in range(3)]
    cols[1][3] = "north\twind"  # legal in a field file: only line ends separate records
    cols[0][5] = "the north"  # field files use splitlines() (cli.py:129): no lone '\r' here
    paths = []
    for k, name in enumerate(("s", "t", "r")):
        p = tmp_path / f"{name}.txt"
        p.write_text("".join(c + "\n" for c in cols[k]))
        paths += [f"-{name}", str(p)]
    one = cli(*base, *paths)
    two = _multi(*base, *paths, "--gpus", "2")
    assert one.returncode == 0 and two.returncode == 0, two.stderr
    assert two.stdout == one.stdout
    bad = tsv.replace(lines[650] + "\n", "only\ttwo\n")
    r = _multi(*base, "--stdin", "--gpus", "2", stdin=bad)
    assert r.returncode == 2 and "line 650: expected 3 tab-separated columns, got 2" in r.stderr
    assert r.stdout == "" and r.stderr.count("error:") == 1


@pytest.mark.gpu
def test_stdin_stream_bad_line_index_matches_list_path(tiny_factory):
    """A bad line deep in a long stdin stream (many windows in) reports the same
    global index as the list path (`evaluate.py:117-123`), and nothing reaches stdout."""
    import paper_2408_11853_b200 as mf
    fix = tiny_factory("comet-qe", "post", 1234)
    lines = fx.fixture_tsv_lines("comet-qe", 30000, seed=5)
    lines[29876] = "one column only"
    with mf.Evaluator(mf.EvaluatorConfig(model=fix.model, vocab=fix.vocab, quiet=True)) as ev:
        with pytest.raises(mf.errors.ColumnCountError) as ei:
            ev.evaluate_lines(lines)
    assert ei.value.line_index == 29876
    r = cli("-m", fix.model, "-v", fix.vocab, "--stdin", stdin="".join(l + "\n" for l in lines))
    assert r.returncode == 2 and r.stdout == ""
    assert "line 29876: expected 2 tab-separated columns, got 1" in r.stderr


@pytest.mark.gpu
def test_eight_ranks_score_bitwise_like_one(tiny_factory):
    """scores at 1 and 8 ranks are identical (here 8 ranks share the
    test box's GPU; whole mini-batches are LPT-assigned, no collective on the data
    path). 3000 records = 3 windows of 128 x 8, more mini-batches than ranks."""
    fix = tiny_factory("comet-qe", "pre", 77)
    lines = fx.fixture_tsv_lines("comet-qe", 3000, seed=8)
    tsv = "".join(l + "\n" for l in lines)
    base = ["-m", fix.model, "-v", fix.vocab, "--quiet", "--precision", "9", "--max-tokens", "32768"]
    one = cli(*base, "--stdin", stdin=tsv)
    eight = _multi(*base, "--stdin", "--gpus", "8", stdin=tsv)
    assert one.returncode == 0 and eight.returncode == 0, eight.stderr[-2000:]
    assert len(one.stdout.splitlines()) == 3000 and eight.stdout == one.stdout
