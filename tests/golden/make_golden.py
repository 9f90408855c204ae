"""Generate golden vectors by running the REFERENCE implementation.

Run in the development container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

It imports `metricforge` read-only, builds the reference's own fixtures with
its own `fixturegen`, and records token ids, batch plans, container checksums
and scores (fp32 and fp16) to `tests/golden/reference_vectors.json`. Tests
compare the oracle and the CUDA path against these numbers; nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import fixturegen  # noqa: E402  (reference tests dir)
import metricforge as mf  # noqa: E402
from metricforge import vocab as mfv  # noqa: E402

from oracle import fixtures as ofx  # noqa: E402


def ref_scores(model, vocab, lines, mode="fp32", **batch):
    cfg = mf.EvaluatorConfig(model=model, vocab=vocab, compute_mode=mode, quiet=True,
                             batch=mf.BatchConfig(**batch) if batch else mf.BatchConfig())
    with mf.Evaluator(cfg) as ev:
        rep = ev.evaluate_lines(lines)
    return [float(s) for s in rep.segment_scores], rep.system_score


def encoded_ids(vocab_path, kind, lines, max_len):
    v = mf.load_vocab(vocab_path)
    recs = list(mf.records_from_tsv_lines(lines, mf.Kind.parse(kind)))
    return [[s.ids for s in mf.encode_fields(v, r, kind, max_len)] for r in recs]


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "metricforge 0.1.0"}
    tmp = tempfile.mkdtemp(prefix="golden")
    vocab = fixturegen.write_vocab(os.path.join(tmp, "vocab.txt"))

    # ---- tokenizer known answers ------------------------------------------
    cases = []
    fixture_tokens = fixturegen.vocab_lines()
    texts = [
        "", "   ", "the north wind", "  the\t\tnorth\nwind  ", "Zq!7 sun",
        "traveling wrapped cloaked", "the north wind　sun", "a​b",
        "xy z w", "<pad> <s>", "stronger" * 5, "é北風 ing ed er",
        "ab\x1cc\x1dd\x1ee\x1ff", "the᠎north", "﻿the",
    ]
    v = mf.Vocabulary(fixture_tokens)
    for t in texts:
        cases.append({"vocab": "fixture", "text": t, "ids": v.encode(t)})
    small_vocabs = [
        ["▁he", "llo", "▁hello"], ["▁a"], ["<", "pad", ">"], ["▁hi"],
        ["a", "ab", "abc", "▁", "▁ab", "bca", "cab"],
        ["▁é", "é", "北", "風北", "▁北風"],
    ]
    small_texts = ["hello", "a§b", "<pad>", "hi hi", "  hi\t\thi  ", "abcabcab ab cab",
                   "é北風北 北風", "北風北風"]
    for sv in small_vocabs:
        vv = mf.Vocabulary(list(mfv.SPECIAL_TOKENS) + sv)
        for t in small_texts:
            cases.append({"vocab": sv, "text": t, "ids": vv.encode(t)})
    out["tokenizer_cases"] = cases

    # ---- encode_fields per kind, several max_len --------------------------
    ef = {}
    for kind in ("comet-qe", "comet", "bleurt"):
        lines = fixturegen.random_tsv_lines(kind, 40, seed=5)
        ef[kind] = {str(ml): encoded_ids(vocab, kind, lines, ml) for ml in (128, 8, 5, 3)}
        ef[kind]["lines"] = lines
    out["encode_fields"] = ef

    # ---- plans ----------------------------------------------------------------
    rng = np.random.default_rng(3)
    plans = []
    for _ in range(30):
        n = int(rng.integers(0, 60))
        lengths = [int(x) for x in rng.integers(0, 50, size=n)]
        mb, fac, srt = int(rng.integers(1, 9)), int(rng.integers(1, 4)), bool(rng.integers(0, 2))
        p = mf.plan_batches(lengths, mf.BatchConfig(mini_batch=mb, maxi_batch_factor=fac,
                                                     sort_by_length=srt))
        plans.append({"lengths": lengths, "mini_batch": mb, "factor": fac, "sort": srt,
                      "batches": p.batches, "order": p.order})
    out["plans"] = plans

    # ---- tiny models per kind / norm style: scores fp32 + fp16 -------------
    tiny = {}
    for kind in ("comet-qe", "comet", "bleurt"):
        for style, seed in (("post", 1234), ("pre", 11)):
            path = os.path.join(tmp, f"{kind}-{style}.mfrg")
            fixturegen.write_tiny_model(path, kind, seed=seed, norm_style=style)
            lines = fixturegen.random_tsv_lines(kind, 20, seed=42)
            s32, sys32 = ref_scores(path, vocab, lines, "fp32")
            s16, sys16 = ref_scores(path, vocab, lines, "fp16")
            man = mf.read_manifest(path)
            tiny[f"{kind}/{style}"] = {
                "seed": seed, "lines": lines, "checksum": man.checksum,
                "fp32": s32, "fp32_system": sys32, "fp16": s16, "fp16_system": sys16,
                "ids": encoded_ids(vocab, kind, lines, 128),
            }
    out["tiny"] = tiny

    # ---- degenerate known answer: zero head passes the final bias ----------
    man = fixturegen.tiny_manifest(mf.Kind.COMET_QE)
    w = fixturegen.make_weights(man, seed=3)
    for k in ("head.0.w", "head.0.b", "head.1.w"):
        w[k] = np.zeros_like(w[k])
    w["head.1.b"] = np.full_like(w["head.1.b"], 0.625)
    zpath = os.path.join(tmp, "zerohead.mfrg")
    mf.write_container(man, fixturegen.weights_to_tensors(w), zpath)
    out["zero_head"] = {"checksum": mf.read_manifest(zpath).checksum,
                        "scores": ref_scores(zpath, vocab, ["north wind\tthe sun"])[0]}

    # ---- config 1: d256 COMET, 1k fixture triplets ---------------------------
    t0 = time.time()
    c1 = ofx.CONFIGS[1]
    p1 = os.path.join(tmp, "config1.mfrg")
    fixturegen.write_tiny_model(p1, "comet", seed=1234, d_model=c1["d_model"],
                                n_heads=c1["n_heads"], n_layers=c1["n_layers"],
                                d_ffn=c1["d_ffn"], head_hidden=c1["head_hidden"])
    lines1 = fixturegen.random_tsv_lines("comet", 1000, seed=0)
    s1, sys1 = ref_scores(p1, vocab, lines1)
    out["config1"] = {"seed": 1234, "checksum": mf.read_manifest(p1).checksum,
                      "scores": s1, "system": sys1, "seconds": time.time() - t0}

    # ---- midsize: XLM-R-large widths, 2 layers, synthetic weights -----------
    mid_man = dict(ofx.CONFIGS[2], vocab_size=2000, n_layers=2)
    mid_path = os.path.join(tmp, "mid.mfrg")
    mtensors = [(n, "f32", a.shape, a.tobytes()) for n, a in ofx.synthetic_weights(mid_man)]
    mf.write_container(mf.ModelManifest(**mid_man), mtensors, mid_path)
    vpath = ofx.write_vocab(os.path.join(tmp, "synvocab.txt"),
                            ofx.synthetic_vocab_lines(mid_man["vocab_size"]))
    mid_lines = [ln for ln in ofx.synthetic_tsv_lines(2, 400)
                 if max(len(c.split()) for c in ln.split("\t")) < 30][:24]
    # remap words into the smaller vocab (w<i> with i < 1995)
    mid_lines = ["\t".join(" ".join(f"w{int(w[1:]) % 1995}" for w in c.split())
                           for c in ln.split("\t")) for ln in mid_lines]
    sm, ssys = ref_scores(mid_path, vpath, mid_lines)
    out["midsize"] = {"manifest": mid_man, "checksum": mf.read_manifest(mid_path).checksum,
                      "lines": mid_lines, "scores": sm, "system": ssys}

    # ---- synthetic 250k vocab tokenisation sample -----------------------------
    big_lines = ofx.synthetic_tsv_lines(2, 50)
    bv = ofx.write_vocab(os.path.join(tmp, "bigvocab.txt"), ofx.synthetic_vocab_lines(250002))
    out["synthetic_ids"] = {"cfg": 2, "count": 50,
                            "ids": encoded_ids(bv, "comet", big_lines, 512)}

    dst = os.path.join(HERE, "reference_vectors.json")
    with open(dst, "w", encoding="utf-8") as f:
        json.dump(out, f, ensure_ascii=False)
    print("wrote", dst, os.path.getsize(dst), "bytes")


if __name__ == "__main__":
    main()
