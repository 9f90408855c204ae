"""End-to-end oracle pipeline mirroring `Evaluator.evaluate_lines`
(`pkg/src/metricforge/evaluate.py:112-123, 168-200`): TSV split, per-kind
encode, window plan, per-mini-batch scoring, order restore, fsum mean."""

from __future__ import annotations

import math

from . import batching, tokenizer
from .encoder import OracleModel
from .fixtures import FIELDS


def encode_lines(vocab, kind, lines, max_len):
    n_cols = len(FIELDS[kind])
    out = []
    for i, line in enumerate(lines):
        cols = line.rstrip("\n").split("\t")
        if len(cols) != n_cols:
            raise ValueError(f"line {i}: expected {n_cols} tab-separated columns, got {len(cols)}")
        out.append(tokenizer.encode_record(vocab, kind, cols, max_len))
    return out


def score_lines(model: OracleModel, vocab, lines, mini_batch=128, factor=8, sort=True,
                max_len=512):
    kind = model.kind
    max_len = min(max_len, model.m["max_position"])
    enc = encode_lines(vocab, kind, lines, max_len)
    win = mini_batch * factor
    scores = []
    for s in range(0, len(enc), win):
        window = enc[s:s + win]
        lengths = [sum(len(q) for q in rec) for rec in window]
        batches, order = batching.plan(lengths, mini_batch, factor, sort)
        flat = []
        for b in batches:
            flat += [float(v) for v in model.score([window[i] for i in b])]
        scores += batching.restore(flat, order)
    system = math.fsum(scores) / len(scores) if scores else None
    return scores, system
