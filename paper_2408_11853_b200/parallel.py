"""Segment-level data parallelism across the GPUs of one box.

The reference's only parallelism is a thread pool mapping `score_records`
over the mini-batches of a window (`pkg/src/metricforge/evaluate.py:154-158,
171-175`); results are bitwise independent of the worker count
(`tests/test_evaluate.py:92-98`). Here the workers are processes, one per GPU
(`torchrun`, RANK / WORLD_SIZE / LOCAL_RANK):

  * every rank computes the same global plan (windows -> bit-exact length
    sort -> mini-batches); with TSV lines the tokenisation is sharded too
    (lengths of 1/w of the lines per rank, all-gathered; then each rank encodes
    only its own mini-batches' records — `score_sharded_lines`);
  * mini-batches are assigned to ranks longest-processing-time-first on the
    cost  sum_seq (L * c_gemm + L^2 * c_attn)  (round-robin per window would
    always give the longest, sorted-first batch to rank 0);
  * each rank scores its batches in one device call per window, the
    (plan position, score) pairs are all-gathered, and the plan's inverse
    permutation restores input order.

There is no collective on the data path: records are independent, the only
exchange is the final gather of float32 scores. Scores are bitwise identical
at any world size because no kernel's reduction order depends on batch
composition.
"""

from __future__ import annotations

import heapq
import math
import os
from typing import Callable, Optional

import numpy as np

from .batching import BatchConfig, pack_roles, plan_order
from .evaluate import ScoreReport, records_from_tsv_lines
from .kinds import N_SEQUENCES, Kind

# relative per-token GEMM cost vs per-token-pair attention cost (config-2 scale:
# 2*(4d^2 + 2 d f) per token, 4 d per token pair)
C_GEMM = 2.0 * (4 * 1024 ** 2 + 2 * 1024 * 4096)
C_ATTN = 4.0 * 1024


def batch_cost(seq_lens) -> float:
    L = np.asarray(seq_lens, dtype=np.float64)
    return float((L * C_GEMM + L * L * C_ATTN).sum())


def lpt_assign(costs, world: int):
    """Longest-processing-time-first: returns one list of batch indices per rank.
    Deterministic (ties broken by batch index, then rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(b) for b in out]


def shard_plan(seq_off, n_seq, n_records, config: BatchConfig, world: int):
    """Global plan of a record-major encoding and its LPT assignment.

    Returns (order, batches, assignment): order[pos] = record index; batches =
    list of (start, stop) plan-position ranges (one mini-batch each); assignment
    = per rank list of batch indices."""
    lens = np.diff(seq_off).reshape(n_records, n_seq)
    order = plan_order(lens.sum(axis=1), config)
    mb = config.mini_batch
    batches = [(s, min(n_records, s + mb)) for s in range(0, n_records, mb)]
    costs = [batch_cost(lens[order[a:b]].ravel()) for a, b in batches]
    return order, batches, lpt_assign(costs, world)


def score_sharded(model_score: Callable, vocab, kind, field_texts, max_len, config: BatchConfig,
                  rank: int, world: int, gather: Optional[Callable] = None, n_threads: int = 0,
                  encoded=None):
    """Score `field_texts` (per-record field lists) across `world` ranks.

    model_score(ids, cu, n) -> float32[n] scores role-major packed records (e.g.
    GpuScoringModel.score_packed); gather(obj) -> list of obj from all ranks
    (e.g. torch.distributed.all_gather_object). Returns scores in input order
    (on every rank). encoded = ((ids, seq_off), n) skips the tokenisation (records
    already encoded, e.g. by Vocabulary.encode_tsv)."""
    kind = Kind.parse(kind)
    ns = N_SEQUENCES[kind]
    if encoded is not None:
        (ids, seq_off), n = encoded
    else:
        n = len(field_texts)
        ids, seq_off = vocab.encode_batch(kind, field_texts, max_len, n_threads)
    order, batches, assign = shard_plan(seq_off, ns, n, config, world)
    mine = assign[rank]
    pos = np.concatenate([np.arange(*batches[b]) for b in mine]) if mine else np.zeros(0, np.int64)
    if len(pos):
        packed, cu = pack_roles(ids, seq_off, ns, order[pos])
        scores = np.asarray(model_score(packed, cu, len(pos)), dtype=np.float32)
    else:
        scores = np.zeros(0, np.float32)
    parts = gather((pos, scores)) if gather is not None else [(pos, scores)]
    flat = np.empty(n, dtype=np.float32)
    seen = 0
    for p, s in parts:
        flat[order[p]] = s
        seen += len(p)
    if seen != n:
        raise RuntimeError(f"gathered {seen} scores for {n} records")
    return flat


def score_sharded_lines(model_score: Callable, vocab, kind, lines, max_len, config: BatchConfig,
                        rank: int, world: int, gather: Optional[Callable] = None,
                        n_threads: int = 0):
    """score_sharded for TSV lines with the tokenisation sharded too: rank r
    encodes lines [n r / w, n (r+1) / w) natively (Vocabulary.encode_tsv) only
    for their sequence lengths, the lengths are all-gathered, every rank builds
    the same global plan and LPT assignment, then encodes just the records of
    its own mini-batches (about 2/w of the host work instead of all of it).
    The records reach model_score in exactly the order score_sharded uses, so
    the scores are bitwise the same. Errors: the reference raises the first
    bad line (ColumnCountError) unless a max_len ValueError comes first, i.e.
    in an earlier window (`evaluate.py:179-196`); every rank raises the same."""
    from .errors import ColumnCountError

    kind = Kind.parse(kind)
    ns = N_SEQUENCES[kind]
    n = len(lines)
    if gather is None or world == 1:
        enc = vocab.encode_tsv(kind, lines, max_len, n_threads)
        return score_sharded(model_score, vocab, kind, None, max_len, config, rank, world, gather,
                             n_threads, encoded=(enc, n))
    a, b = n * rank // world, n * (rank + 1) // world
    need = 3 if kind is Kind.BLEURT else 2
    len_err = n > 0 and max_len < need  # raised at window 0's encode by the reference
    lens, col_err = np.zeros(0, np.int64), None
    try:
        _, off = vocab.encode_tsv(kind, lines[a:b], max_len, n_threads, first_index=a)
        lens = np.diff(off)
    except ColumnCountError as e:
        col_err = (e.line_index, e.expected, e.got)
    except ValueError:
        if not len_err:
            raise
    parts = gather((lens, col_err))
    cols = [p[1] for p in parts if p[1] is not None]
    first_col = min(cols) if cols else None
    if len_err and (first_col is None or first_col[0] >= config.window):
        what = "BOS, SEP and EOS" if kind is Kind.BLEURT else "BOS and EOS"
        raise ValueError(f"max_len {max_len} cannot hold {what}")
    if first_col is not None:
        raise ColumnCountError(*first_col)
    seq_lens = np.concatenate([p[0] for p in parts])
    seq_off = np.zeros(len(seq_lens) + 1, dtype=np.int64)
    np.cumsum(seq_lens, out=seq_off[1:])
    order, batches, assign = shard_plan(seq_off, ns, n, config, world)
    mine = assign[rank]
    pos = np.concatenate([np.arange(*batches[i]) for i in mine]) if mine else np.zeros(0, np.int64)
    if len(pos):
        ids, off = vocab.encode_tsv(kind, [lines[i] for i in order[pos]], max_len, n_threads)
        packed, cu = pack_roles(ids, off, ns, np.arange(len(pos)))
        scores = np.asarray(model_score(packed, cu, len(pos)), dtype=np.float32)
    else:
        scores = np.zeros(0, np.float32)
    flat = np.empty(n, dtype=np.float32)
    seen = 0
    for p, sc in gather((pos, scores)):
        flat[order[p]] = sc
        seen += len(p)
    if seen != n:
        raise RuntimeError(f"gathered {seen} scores for {n} records")
    return flat


class DistributedEvaluator:
    """`Evaluator` over all ranks of an initialised torch.distributed group.

    Every rank passes the same lines; every rank gets the full report."""

    def __init__(self, config, group=None):
        import torch.distributed as dist

        from .evaluate import Evaluator

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if config.device is None:
            config.device = int(os.environ.get("LOCAL_RANK", "0"))
        self.ev = Evaluator(config)
        self.config = config
        self._group = group

    def _gather(self, obj):
        import torch.distributed as dist

        if self.world == 1:
            return [obj]
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self._group)
        return out

    def evaluate_lines(self, lines) -> ScoreReport:
        kind = self.ev.kind
        if isinstance(lines, (list, tuple)) and all(type(l) is str for l in lines):
            scores = score_sharded_lines(self.ev.model.score_packed, self.ev.vocab, kind, lines,
                                         self.ev.max_len, self.config.batch, self.rank, self.world,
                                         self._gather, self.config.tokenizer_threads)
            return ScoreReport(segment_scores=scores.tolist())
        else:
            recs = [r.field_values(kind, i)
                    for i, r in enumerate(records_from_tsv_lines(lines, kind))]
            encoded = self.ev.vocab.encode_batch(kind, recs, self.ev.max_len,
                                                 self.config.tokenizer_threads)
            n = len(recs)
        scores = score_sharded(self.ev.model.score_packed, self.ev.vocab, kind, None,
                               self.ev.max_len, self.config.batch, self.rank, self.world,
                               self._gather, self.config.tokenizer_threads,
                               encoded=(encoded, n))
        return ScoreReport(segment_scores=scores.tolist())

    def close(self):
        self.ev.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
