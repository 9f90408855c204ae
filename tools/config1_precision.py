"""Config-1 (reference fixture weights, std 0.25) fp32-path error vs the
reference's scores under accumulation variants (env MFG_KCHUNK / MFG_WEIGHT_PRESCALE
are read once per process, so each variant runs in its own process).

    python tools/config1_precision.py            # all variants, one line each
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import numpy as np

    import paper_2408_11853_b200 as mf
    from oracle import fixtures as fx
    from oracle import mfrg
    with open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")) as f:
        g = json.load(f)["config1"]
    c1 = fx.CONFIGS[1]
    man = fx.tiny_manifest("comet", **{k: c1[k] for k in
                                       ("d_model", "n_heads", "n_layers", "d_ffn", "head_hidden")})
    w = fx.fixture_weights(man, 1234)
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "c1.mfrg")
    mfrg.write(path, mfrg.manifest_dict(**man), [(n, "f32", w[n]) for n, _ in fx.tensor_shapes(man)])
    vocab = fx.write_vocab(os.path.join(tmp, "v.txt"), fx.fixture_vocab_lines())
    lines = fx.fixture_tsv_lines("comet", 1000, seed=0)
    out = {}
    for prec in ("fp32", "bf16x3"):
        with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab, quiet=True, precision=prec)) as ev:
            s = np.array(ev.evaluate_lines(lines).segment_scores)
        d = np.abs(s - np.array(g["scores"]))
        out[prec] = {"max": float(d.max()), "mean": float(d.mean())}
    print(json.dumps({"env": {k: os.environ.get(k) for k in ("MFG_KCHUNK", "MFG_WEIGHT_PRESCALE")},
                      **out}), flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
    else:
        for env in ({}, {"MFG_WEIGHT_PRESCALE": "0"}, {"MFG_KCHUNK": "512"}, {"MFG_KCHUNK": "256"},
                    {"MFG_KCHUNK": "128"}):
            subprocess.run([sys.executable, __file__, "--one"], env=dict(os.environ, **env))
