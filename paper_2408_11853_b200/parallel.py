"""Segment-level data parallelism across the GPUs of one box.

The reference's only parallelism is a thread pool mapping `score_records`
over the mini-batches of a window (`pkg/src/metricforge/evaluate.py:154-158,
171-175`); results are bitwise independent of the worker count
(`tests/test_evaluate.py:92-98`). Here the workers are processes, one per GPU
(RANK / WORLD_SIZE / LOCAL_RANK), and the input is STREAMED:

  * rank 0 (the coordinator) reads the input lazily — any iterable of TSV
    lines or EvalRecords, e.g. stdin — one *round* of `stream_windows`
    reference windows (mini_batch x maxi_batch_factor records each) at a time,
    tokenising the next round in a producer thread (bounded queue: at most one
    round ahead, so memory stays bounded for any input size);
  * per round it computes the reference plan of every window (bit-exact
    length sort, `batching.py:61-73`), assigns whole mini-batches to ranks
    longest-processing-time-first on the cost
    sum_seq (L * c_gemm + L^2 * c_attn) derived from the model's d, d_ffn and
    layer count, and scatters each rank its role-major packed token ids;
  * every rank scores its share in one device call per round on a worker
    thread, so round k+1's scatter overlaps round k's GPU work; the float32
    scores come back to rank 0, which restores input order.

There is no collective on the data path: records are independent; the only
exchanges are host-side (token ids out, scores back) over a gloo group. Any
error — a bad TSV line on rank 0, a device error on any rank — ends the
stream on every rank with the same exception, and scores are bitwise identical
at any world size because no kernel's reduction order depends on batch
composition.
"""

from __future__ import annotations

import heapq
import os
import queue
import threading
from concurrent.futures import ThreadPoolExecutor
from itertools import islice
from typing import Callable, Optional

import numpy as np

from .batching import BatchConfig, pack_roles, plan_order
from .evaluate import ScoreReport
from .kinds import FIELDS_REQUIRED, N_SEQUENCES, Kind, record_from_columns


class CostModel:
    """Relative device cost of a sequence of L tokens: GEMMs 2(4d^2 + 2 d f) per
    token per layer, attention 4 d per token pair per layer (SURVEY.md §8 cfg table)."""

    def __init__(self, d_model=1024, d_ffn=4096, n_layers=24):
        self.c_gemm = 2.0 * (4 * d_model ** 2 + 2 * d_model * d_ffn) * n_layers
        self.c_attn = 4.0 * d_model * n_layers

    @classmethod
    def from_info(cls, info):
        return cls(int(info.d_model), int(info.d_ffn), max(1, int(info.n_layers)))

    def __call__(self, seq_lens) -> float:
        L = np.asarray(seq_lens, dtype=np.float64)
        return float((L * self.c_gemm + L * L * self.c_attn).sum())


def batch_cost(seq_lens, cost: Optional[CostModel] = None) -> float:
    return (cost or CostModel())(seq_lens)


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


def shard_plan(seq_off, n_seq, n_records, config: BatchConfig, world: int,
               cost: Optional[CostModel] = None):
    """Plan of a record-major encoding (starting at a window boundary) and its
    LPT assignment. Returns (order, batches, assignment): order[pos] = record
    index; batches = (start, stop) plan-position ranges, one mini-batch each;
    assignment = per rank list of batch indices."""
    lens = np.diff(seq_off).reshape(n_records, n_seq)
    order = plan_order(lens.sum(axis=1), config)
    mb = config.mini_batch
    batches = [(s, min(n_records, s + mb)) for s in range(0, n_records, mb)]
    costs = [batch_cost(lens[order[a:b]].ravel(), cost) for a, b in batches]
    return order, batches, lpt_assign(costs, world)


def score_sharded(model_score: Callable, vocab, kind, field_texts, max_len, config: BatchConfig,
                  rank: int, world: int, gather: Optional[Callable] = None, n_threads: int = 0,
                  encoded=None, cost: Optional[CostModel] = None):
    """Score an in-memory set of records across `world` ranks (every rank holds
    the same input). model_score(ids, cu, n) -> float32[n]; gather(obj) -> list
    of obj from all ranks. Returns scores in input order on every rank.
    Errors inside the local scoring are gathered and re-raised on every rank."""
    kind = Kind.parse(kind)
    ns = N_SEQUENCES[kind]
    if encoded is not None:
        (ids, seq_off), n = encoded
    else:
        n = len(field_texts)
        ids, seq_off = vocab.encode_batch(kind, field_texts, max_len, n_threads)
    order, batches, assign = shard_plan(seq_off, ns, n, config, world, cost)
    mine = assign[rank]
    pos = np.concatenate([np.arange(*batches[b]) for b in mine]) if mine else np.zeros(0, np.int64)
    err = None
    scores = np.zeros(0, np.float32)
    try:
        if len(pos):
            packed, cu = pack_roles(ids, seq_off, ns, order[pos])
            scores = np.asarray(model_score(packed, cu, len(pos)), dtype=np.float32)
    except Exception as e:  # noqa: BLE001 - re-raised on every rank below
        err = e
    parts = gather((pos, scores, err)) if gather is not None else [(pos, scores, err)]
    for _, _, e in parts:
        if e is not None:
            raise e
    flat = np.empty(n, dtype=np.float32)
    seen = 0
    for p, s, _ in parts:
        flat[order[p]] = s
        seen += len(p)
    if seen != n:
        raise RuntimeError(f"gathered {seen} scores for {n} records")
    return flat


# --------------------------------------------------------------------------- streaming
class Comm:
    """Host-side object exchange between the ranks of one gloo group."""

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group

    def scatter(self, objs):
        """Rank 0 passes one object per rank; every rank returns its own."""
        if self.world == 1:
            return objs[0]
        import torch.distributed as dist
        out = [None]
        dist.scatter_object_list(out, objs if self.rank == 0 else None, src=0, group=self.group)
        return out[0]

    def gather(self, obj):
        """List of every rank's obj on rank 0, None elsewhere."""
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world if self.rank == 0 else None
        dist.gather_object(obj, out, dst=0, group=self.group)
        return out

    def bcast(self, obj):
        if self.world == 1:
            return obj
        import torch.distributed as dist
        box = [obj]
        dist.broadcast_object_list(box, src=0, group=self.group)
        return box[0]


_END = ("end",)


def _rounds_from_lines(vocab, kind, lines, max_len, per_round, n_threads):
    """Yield (ids, seq_off, n) per round of up to per_round TSV lines (native
    intake; ColumnCountError carries the global line index)."""
    it = iter(lines)
    base = 0
    while True:
        chunk = list(islice(it, per_round))
        if not chunk:
            return
        if all(type(ln) is str for ln in chunk):
            ids, off = vocab.encode_tsv(kind, chunk, max_len, n_threads, base)
        else:
            want = len(FIELDS_REQUIRED[kind])
            fields = []
            for i, ln in enumerate(chunk):
                cols = ln.rstrip("\n").split("\t")
                if len(cols) != want:
                    from .errors import ColumnCountError
                    raise ColumnCountError(base + i, want, len(cols))
                fields.append(record_from_columns(cols, kind, base + i).field_values(kind, base + i))
            ids, off = vocab.encode_batch(kind, fields, max_len, n_threads)
        yield ids, off, len(chunk)
        base += len(chunk)


def _rounds_from_records(vocab, kind, records, max_len, per_round, n_threads):
    it = iter(records)
    base = 0
    while True:
        chunk = list(islice(it, per_round))
        if not chunk:
            return
        fields = [r.field_values(kind, base + i) for i, r in enumerate(chunk)]
        ids, off = vocab.encode_batch(kind, fields, max_len, n_threads)
        yield ids, off, len(chunk)
        base += len(chunk)


def _portable(e):
    """The exception itself when it survives pickling (so other ranks can re-raise
    it), else a RuntimeError carrying its type and message."""
    import pickle
    try:
        pickle.loads(pickle.dumps(e))
        return e
    except Exception:  # noqa: BLE001
        return RuntimeError(f"{type(e).__name__}: {e}")


def _assign_round(item, ns, config, world, cost, base):
    """Rank 0: plan one round, LPT its mini-batches and pack each rank's share."""
    ids, off, n = item
    order, batches, assign = shard_plan(off, ns, n, config, world, cost)
    pos = [np.concatenate([np.arange(*batches[b]) for b in a]) if a else np.zeros(0, np.int64)
           for a in assign]
    objs = []
    for r in range(world):
        if len(pos[r]):
            packed, cu = pack_roles(ids, off, ns, order[pos[r]])
            objs.append(("work", packed, cu, len(pos[r])))
        else:
            objs.append(("work", np.zeros(0, np.int32), np.zeros(1, np.int64), 0))
    return objs, (base, order, pos)


def stream_sharded(model_score: Callable, rounds, kind, config: BatchConfig, comm: Comm,
                   cost: Optional[CostModel] = None, prefetch: int = 1):
    """Score a stream of encoded rounds (rank 0's `rounds` iterable yields
    (ids, seq_off, n) record-major, each round starting at a window boundary;
    other ranks pass None) across the ranks of `comm`. Returns float32 scores in
    input order on every rank; raises the stream's first error on every rank.

    Per round i (all ranks, same collective sequence):
        scatter(work_i)  ->  gather(scores_{i-1})  ->  submit(score work_i)
    so round i's transfer overlaps round i-1's device work."""
    kind = Kind.parse(kind)
    ns = N_SEQUENCES[kind]
    rank, world = comm.rank, comm.world
    pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="mfg-rank-score")
    out_parts = []       # rank 0: per round (base, order, per-rank positions)
    results = {}         # rank 0: round -> per-rank scores
    first_err = None
    q = None
    stop = threading.Event()

    if rank == 0:
        q = queue.Queue(maxsize=max(1, prefetch))

        def producer():
            try:
                for item in rounds:
                    while not stop.is_set():
                        try:
                            q.put(("work_ready", item), timeout=0.1)
                            break
                        except queue.Full:
                            continue
                    if stop.is_set():
                        return
                q.put(_END)
            except BaseException as e:  # noqa: BLE001 - forwarded to every rank
                q.put(("error", e))

        threading.Thread(target=producer, daemon=True, name="mfg-intake").start()

    def score_local(work):
        packed, cu, m = work
        try:
            if m == 0:
                return np.zeros(0, np.float32), None
            return np.asarray(model_score(packed, cu, m), dtype=np.float32), None
        except Exception as e:  # noqa: BLE001 - gathered and re-raised everywhere
            return None, _portable(e)

    fut = None
    base = 0
    i = 0
    try:
        while True:
            # ---- rank 0: next round's assignment (or the terminal message)
            objs = None
            if rank == 0:
                item = q.get() if first_err is None else ("error", first_err)
                if item[0] == "work_ready":
                    try:
                        objs, part = _assign_round(item[1], ns, config, world, cost, base)
                        out_parts.append(part)
                        base += item[1][2]
                    except Exception as e:  # noqa: BLE001
                        item = ("error", e)
                if item[0] in ("end", "error"):
                    if item[0] == "error" and first_err is None:
                        first_err = _portable(item[1])
                    objs = [_END if item[0] == "end" else ("error", first_err)] * world
            work = comm.scatter(objs)
            # ---- previous round's scores back to rank 0
            if fut is not None:
                res = comm.gather(fut.result())
                fut = None
                if rank == 0:
                    for s, e in res:
                        if e is not None and first_err is None:
                            first_err = _portable(e)
                    results[i - 1] = [s for s, _ in res]
            if work[0] != "work":
                break
            fut = pool.submit(score_local, work[1:])
            i += 1
        # ---- final result (or the first error) to every rank
        if rank == 0:
            if first_err is None and work[0] == "error":
                first_err = work[1]
            if first_err is not None:
                final = ("error", first_err)
            else:
                flat = np.empty(base, dtype=np.float32)
                for k, (b0, order, pos) in enumerate(out_parts):
                    for r in range(world):
                        flat[b0 + order[pos[r]]] = results[k][r]
                final = ("ok", flat)
        else:
            final = None
        final = comm.bcast(final)
    finally:
        stop.set()
        pool.shutdown(wait=True)
    if final[0] == "error":
        raise final[1]
    return final[1]


class DistributedEvaluator:
    """`Evaluator` over all ranks of an initialised torch.distributed group.

    Rank 0 reads the input (any iterable; other ranks may pass None — their
    argument is ignored) and streams it to the ranks in rounds of
    `stream_windows` windows; every rank returns the full report."""

    def __init__(self, config, group=None, stream_windows: int = 16):
        import torch.distributed as dist

        from .evaluate import Evaluator

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if config.device is None:
            config.device = int(os.environ.get("LOCAL_RANK", "0"))
        self.ev = Evaluator(config)
        self.config = config
        self.stream_windows = max(1, int(stream_windows))
        cg = None
        if self.world > 1:
            # host-side token ids / scores travel over gloo (no GPU involvement)
            backend = dist.get_backend(group)
            cg = group if backend == "gloo" else dist.new_group(
                ranks=dist.get_process_group_ranks(group) if group is not None else None,
                backend="gloo")
        self.comm = Comm(self.rank, self.world, cg)
        self.cost = CostModel.from_info(self.ev.model.info)

    @property
    def kind(self):
        return self.ev.kind

    def _run(self, make_rounds):
        per_round = self.config.batch.window * self.stream_windows
        rounds = make_rounds(per_round) if self.rank == 0 else None
        scores = stream_sharded(self.ev.model.score_packed, rounds, self.ev.kind,
                                self.config.batch, self.comm, self.cost)
        return ScoreReport(segment_scores=scores.tolist())

    def evaluate_lines(self, lines=None) -> ScoreReport:
        ev = self.ev
        return self._run(lambda per: _rounds_from_lines(ev.vocab, ev.kind, lines, ev.max_len, per,
                                                        self.config.tokenizer_threads))

    def evaluate(self, records=None) -> ScoreReport:
        ev = self.ev
        return self._run(lambda per: _rounds_from_records(ev.vocab, ev.kind, records, ev.max_len,
                                                          per, self.config.tokenizer_threads))

    def close(self):
        self.ev.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
