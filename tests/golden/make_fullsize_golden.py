"""Full-size parity goldens: the REFERENCE `Evaluator` itself on configs 2-5.

Run in the development container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py [cfg ...]

For each config (512 length-stratified records at configs
2-4, 64 at config 5) it writes the synthetic random-init model (seeded,
`oracle.fixtures.synthetic_weights`) and vocabulary, scores the
`oracle.fixtures.parity_subset` records through the unmodified reference
`metricforge.Evaluator` (default BatchConfig, fp32 and the reference fp16
mode), and commits only the seeds, the container checksum and the scores to
`tests/golden/fullsize_cfg<N>.json`. The GPU tests and bench.py regenerate the
same model and records on the box (checked against the checksum) and compare.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import metricforge as mf  # noqa: E402

from oracle import fixtures as ofx  # noqa: E402

WORK = os.environ.get("MFG_GOLDEN_DIR", "/tmp/mfg_golden")


def build_model(cfg):
    man = dict(ofx.CONFIGS[cfg])
    path = os.path.join(WORK, f"config{cfg}.mfrg")
    vocab = os.path.join(WORK, f"config{cfg}.vocab.txt")
    if not os.path.exists(path + ".ok"):
        tensors = ((n, "f32", a.shape, a.tobytes()) for n, a in ofx.synthetic_weights(man))
        mf.write_container(mf.ModelManifest(**man), tensors, path)
        ofx.write_vocab(vocab, ofx.synthetic_vocab_lines(man["vocab_size"]))
        open(path + ".ok", "w").close()
    return man, path, vocab


def score(path, vocab, lines, mode):
    cfg = mf.EvaluatorConfig(model=path, vocab=vocab, compute_mode=mode, quiet=True,
                             validate=False)
    t0 = time.time()
    with mf.Evaluator(cfg) as ev:
        rep = ev.evaluate_lines(lines)
    return [float(s) for s in rep.segment_scores], rep.system_score, time.time() - t0


def main(cfgs):
    os.makedirs(WORK, exist_ok=True)
    modes = os.environ.get("MFG_GOLDEN_MODES", "fp32,fp16").split(",")
    for mode in modes:
        for cfg in cfgs:
            dst = os.path.join(HERE, f"fullsize_cfg{cfg}.json")
            out = json.load(open(dst)) if os.path.exists(dst) else {}
            if mode in out:
                continue
            man, path, vocab = build_model(cfg)
            idx, lines = ofx.parity_subset(cfg)
            scores, system, secs = score(path, vocab, lines, mode)
            out.update({
                "generator": "tests/golden/make_fullsize_golden.py",
                "reference": "metricforge 0.1.0 Evaluator (pkg/src/metricforge/evaluate.py:126-241)",
                "config": cfg, "manifest": man, "checksum": mf.read_manifest(path).checksum,
                "weight_seed": ofx.WEIGHT_SEED, "pool": ofx.PARITY_POOL,
                "text_seed": ofx.PARITY_SEED, "n": len(lines), "pool_indices": idx,
                "lengths": [sum(len(c.split()) for c in ln.split("\t")) for ln in lines],
            })
            out[mode] = scores
            out[mode + "_system"] = system
            out.setdefault("seconds", {})[mode] = secs
            out["host"] = {"cpu": platform.processor() or platform.machine(),
                           "cores": os.cpu_count()}
            with open(dst, "w") as f:
                json.dump(out, f)
            print(f"config {cfg} {mode}: {len(lines)} records in {secs:.0f} s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2, 3, 4, 5])
