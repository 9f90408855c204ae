"""Batch-plan oracle, restating `pkg/src/metricforge/batching.py:61-101`.

Records are cut into windows of `mini_batch * factor`; inside a window
they are (optionally) stably ordered by descending length with the record
index as tie-break; the concatenated order is chunked into mini-batches.
`order[scoring_position] = original_index`.
"""

from __future__ import annotations


def plan(lengths, mini_batch=128, factor=8, sort=True):
    n = len(lengths)
    win = mini_batch * factor
    order = []
    for s in range(0, n, win):
        idx = list(range(s, min(n, s + win)))
        if sort:
            idx.sort(key=lambda i: (-lengths[i], i))
        order += idx
    batches = [order[s:s + mini_batch] for s in range(0, len(order), mini_batch)]
    return batches, order


def restore(scores, order):
    if len(scores) != len(order):
        raise ValueError(f"got {len(scores)} scores for {len(order)} planned records")
    out = [None] * len(order)
    for pos, orig in enumerate(order):
        out[orig] = scores[pos]
    return out
