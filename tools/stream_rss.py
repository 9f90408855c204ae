"""Bounded-memory evidence for the streamed CLI intake: score an
N-line TSV file through `--stdin` and record the CLI process's peak RSS
(VmHWM) and wall time; run it for two sizes — RSS must not grow with N.

    python tools/stream_rss.py --config 5 --lines 20000 200000
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def write_lines(cfg, n, path, chunk=50000):
    from oracle import fixtures as fx
    with open(path, "w", encoding="utf-8") as f:
        for s in range(0, n, chunk):  # generated and written in chunks (seeded per chunk)
            f.write("".join(ln + "\n" for ln in fx.synthetic_tsv_lines(cfg, min(chunk, n - s),
                                                                      seed=fx.TEXT_SEED + s)))


def run(cfg, n, extra):
    import bench
    _, model, vocab = bench.prepare_model(cfg, 0, 1, lambda: None)
    path = os.path.join(bench.BENCH_DIR, f"stream_cfg{cfg}_{n}.tsv")
    if not os.path.exists(path):
        write_lines(cfg, n, path)
    out = path + ".scores"
    t0 = time.perf_counter()
    with open(path, "rb") as fin:
        p = subprocess.Popen([sys.executable, "-m", "paper_2408_11853_b200.cli", "-m", model,
                              "-v", vocab, "--stdin", "--quiet", "-o", out, *extra],
                             stdin=fin, cwd=ROOT)
        hwm = last = 0
        while p.poll() is None:
            try:
                with open(f"/proc/{p.pid}/status") as st:
                    for line in st:
                        if line.startswith("VmHWM:"):
                            hwm = max(hwm, int(line.split()[1]))
                        elif line.startswith("VmRSS:"):
                            last = int(line.split()[1])  # steady state while scoring
            except OSError:
                pass
            time.sleep(0.2)
    dt = time.perf_counter() - t0
    digest = hashlib.sha256(open(out, "rb").read()).hexdigest()[:16]
    n_out = sum(1 for _ in open(out))
    return {"config": cfg, "lines": n, "rc": p.returncode, "scores": n_out,
            "input_mb": os.path.getsize(path) / 2 ** 20, "peak_rss_mb": hwm / 1024,
            "wall_s": dt, "records_per_s": n / dt, "final_rss_mb": last / 1024,
            "scores_sha256_16": digest}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--lines", type=int, nargs="+", default=[20000, 200000])
    a, extra = ap.parse_known_args()
    for n in a.lines:
        print(json.dumps(run(a.config, n, extra)), flush=True)
