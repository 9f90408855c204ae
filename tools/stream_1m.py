"""The f3 acceptance run: a 1M-line config-5 file scored through the CLI's
`--stdin` stream (peak / steady RSS sampled) and through the list path
(`Evaluator.evaluate_lines(list)`), scores compared line by line at 9 digits;
then a bad line near the end: same ColumnCountError index on both paths.

    python tools/stream_1m.py [--lines 1000000]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import stream_rss  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lines", type=int, default=1000000)
    a = ap.parse_args()
    res = stream_rss.run(5, a.lines, ["--precision", "9"])
    import bench
    import paper_2408_11853_b200 as mf
    _, model, vocab = bench.prepare_model(5, 0, 1, lambda: None)
    path = os.path.join(bench.BENCH_DIR, f"stream_cfg5_{a.lines}.tsv")
    with open(path, encoding="utf-8") as f:
        lines = f.read().split("\n")[:-1]
    t0 = time.perf_counter()
    with mf.Evaluator(mf.EvaluatorConfig(model=model, vocab=vocab, quiet=True)) as ev:
        scores = ev.evaluate_lines(lines).segment_scores
        list_s = time.perf_counter() - t0
        listed = [f"{v:.9f}" for v in scores]
        streamed = open(path + ".scores").read().split("\n")[:-1]
        res["list_path_s"] = list_s
        res["same_scores_as_list_path"] = streamed == listed
        # a bad line a quarter of the way in (many windows deep; both paths score
        # everything before it): same global index on both paths
        bad = len(lines) // 4 + 37
        lines[bad] = "only one column"
        try:
            ev.evaluate_lines(lines)
            res["list_error"] = None
        except mf.errors.ColumnCountError as e:
            res["list_error"] = e.line_index
    with open(path + ".bad", "w", encoding="utf-8") as f:
        f.write("".join(ln + "\n" for ln in lines))
    with open(path + ".bad", "rb") as fin:
        r = subprocess.run([sys.executable, "-m", "paper_2408_11853_b200.cli", "-m", model, "-v",
                            vocab, "--stdin", "--quiet"], stdin=fin, capture_output=True, text=True,
                           cwd=ROOT)
    res["stream_error"] = {"rc": r.returncode, "stderr": r.stderr.strip()[-200:],
                           "stdout_bytes": len(r.stdout)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
