"""Multi-rank sharding logic (paper_2408_11853_b200.parallel) on CPU with the
gloo backend, world_size 2: LPT assignment, global plan, gather and order
restore. The scorer is a deterministic stand-in for the GPU model (records are
independent, so any per-record function exercises the data flow)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2408_11853_b200 as mf
from oracle import fixtures as fx
from paper_2408_11853_b200.parallel import batch_cost, lpt_assign, score_sharded, shard_plan


def fake_score(ids, cu, n):
    """Per-record function of its own token ids (role-major layout)."""
    n_roles = (len(cu) - 1) // n
    out = np.zeros(n, np.float32)
    for k in range(n_roles):
        for i in range(n):
            seg = ids[cu[k * n + i]:cu[k * n + i + 1]]
            out[i] += np.float32((k + 1) * (seg.astype(np.int64) * np.arange(1, len(seg) + 1)).sum() % 9973) / 100
    return out


def test_lpt_balances_and_is_deterministic():
    costs = [9, 7, 6, 5, 5, 4, 3, 2, 2, 1]
    a = lpt_assign(costs, 3)
    assert sorted(i for part in a for i in part) == list(range(10))
    loads = [sum(costs[i] for i in part) for part in a]
    assert max(loads) - min(loads) <= max(costs)
    assert a == lpt_assign(costs, 3)
    assert batch_cost([10, 10]) < batch_cost([20])


def test_shard_plan_covers_every_record_once():
    v = mf.Vocabulary(fx.fixture_vocab_lines())
    lines = fx.fixture_tsv_lines("comet", 500, seed=1)
    recs = [r.field_values(mf.Kind.COMET) for r in mf.records_from_tsv_lines(lines, mf.Kind.COMET)]
    ids, off = v.encode_batch(mf.Kind.COMET, recs, 128)
    order, batches, assign = shard_plan(off, 3, 500, mf.BatchConfig(mini_batch=32, maxi_batch_factor=2), 4)
    pos = sorted(p for part in assign for b in part for p in range(*batches[b]))
    assert pos == list(range(500))
    assert sorted(order.tolist()) == list(range(500))


def _worker(rank, world, port, lines, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = mf.Vocabulary(fx.fixture_vocab_lines())
        recs = [r.field_values(mf.Kind.COMET_QE) for r in mf.records_from_tsv_lines(lines, mf.Kind.COMET_QE)]

        def gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        scores = score_sharded(fake_score, v, "comet-qe", recs, 128,
                               mf.BatchConfig(mini_batch=16, maxi_batch_factor=4), rank, world, gather)
        result[rank] = scores.tolist()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_equal_single_process(world):
    lines = fx.fixture_tsv_lines("comet-qe", 300, seed=9)
    v = mf.Vocabulary(fx.fixture_vocab_lines())
    recs = [r.field_values(mf.Kind.COMET_QE) for r in mf.records_from_tsv_lines(lines, mf.Kind.COMET_QE)]
    solo = score_sharded(fake_score, v, "comet-qe", recs, 128,
                         mf.BatchConfig(mini_batch=16, maxi_batch_factor=4), 0, 1).tolist()
    # direct per-record reference
    ids, off = v.encode_batch(mf.Kind.COMET_QE, recs, 128)
    from paper_2408_11853_b200.batching import pack_roles
    direct = [float(fake_score(*pack_roles(ids, off, 2, [i]), 1)[0]) for i in range(300)]
    assert solo == direct
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    result = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lines, result)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert result[0] == result[1] == solo


def _worker_stream(rank, world, port, lines, cfg, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_11853_b200.parallel import Comm, _rounds_from_lines, stream_sharded
        v = mf.Vocabulary(fx.fixture_vocab_lines())
        batch = mf.BatchConfig(mini_batch=16, maxi_batch_factor=4)
        per_round = batch.window * cfg.get("stream_windows", 2)
        consumed = [0]
        trace = []

        def gen():  # a lazy source: counts how far the coordinator has read
            for ln in lines:
                consumed[0] += 1
                yield ln

        def score(ids, cu, n):
            trace.append(consumed[0])
            if cfg.get("fail_rank") == rank:
                raise RuntimeError(f"device failure on rank {rank}")
            return fake_score(ids, cu, n)

        rounds = (_rounds_from_lines(v, mf.Kind.COMET, gen(), cfg["max_len"], per_round, 0)
                  if rank == 0 else None)
        try:
            scores = stream_sharded(score, rounds, "comet", batch, Comm(rank, world))
            result[rank] = scores.tolist()
        except mf.errors.ColumnCountError as e:
            result[rank] = ("ColumnCountError", e.line_index, e.got)
        except ValueError as e:
            result[rank] = ("ValueError", str(e))
        except RuntimeError as e:
            result[rank] = ("RuntimeError", str(e))
        if rank == 0:
            result["trace"] = trace
            result["per_round"] = per_round
    finally:
        dist.destroy_process_group()


def _run_ranks(world, lines, cfg):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    result = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker_stream, args=(r, world, port, lines, cfg, result))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    return [result[r] for r in range(world)], dict(result)


def _solo(lines):
    v = mf.Vocabulary(fx.fixture_vocab_lines())
    recs = [r.field_values(mf.Kind.COMET) for r in mf.records_from_tsv_lines(lines, mf.Kind.COMET)]
    return score_sharded(fake_score, v, "comet", recs, 128,
                         mf.BatchConfig(mini_batch=16, maxi_batch_factor=4), 0, 1).tolist()


@pytest.mark.parametrize("world", [2, 3])
def test_streamed_ranks_equal_single_process(world):
    """stream_sharded: rank 0 reads a lazy source in rounds of 2 windows, every
    rank scores its LPT share, scores come back in input order on every rank."""
    lines = fx.fixture_tsv_lines("comet", 301, seed=5)
    got, res = _run_ranks(world, lines, {"max_len": 128})
    assert all(g == _solo(lines) for g in got)


def test_streamed_intake_is_bounded():
    """The coordinator reads at most 3 rounds ahead of the scoring (bounded
    queue), whatever the input size."""
    lines = fx.fixture_tsv_lines("comet", 2000, seed=8)
    got, res = _run_ranks(2, lines, {"max_len": 128})
    assert got[0] == got[1] == _solo(lines)
    per = res["per_round"]
    trace = res["trace"]
    assert len(trace) == -(-2000 // per)
    # round k scores while k+1 is scattered, k+2 queued and k+3 read by the producer
    assert all(c <= (k + 4) * per for k, c in enumerate(trace)), (trace, per)


def test_streamed_errors_match_on_every_rank():
    lines = fx.fixture_tsv_lines("comet", 400, seed=6)
    lines[350] = "only\ttwo"
    got, _ = _run_ranks(2, lines, {"max_len": 128})
    assert got[0] == got[1] == ("ColumnCountError", 350, 2)
    # max_len too small: raised at the first record on every rank
    got, _ = _run_ranks(2, lines, {"max_len": 1})
    assert got[0] == got[1] and got[0][0] == "ValueError"
    # a device error on a non-coordinator rank ends the stream everywhere
    got, _ = _run_ranks(3, lines[:300], {"max_len": 128, "fail_rank": 1})
    assert got[0] == got[1] == got[2] == ("RuntimeError", "device failure on rank 1")


def test_streamed_empty_and_tiny_inputs():
    got, _ = _run_ranks(2, [], {"max_len": 128})
    assert got == [[], []]
    lines = fx.fixture_tsv_lines("comet", 1, seed=3)  # fewer records than ranks
    got, _ = _run_ranks(3, lines, {"max_len": 128})
    assert got == [_solo(lines)] * 3


def test_lpt_costs_follow_the_model():
    from paper_2408_11853_b200.parallel import CostModel
    c2, c5 = CostModel(1024, 4096, 24), CostModel(2560, 10240, 36)
    # attention's share of a 500-token sequence grows with L relative to the GEMMs
    share2 = 500 * 500 * c2.c_attn / c2([500])
    assert 0 < share2 < 0.2
    assert c5([10]) / c2([10]) == pytest.approx(c5.c_gemm / c2.c_gemm, rel=1e-3)
