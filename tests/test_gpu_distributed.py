"""DistributedEvaluator with the real device path: two ranks (gloo for the
score gather) sharing cuda:0 score the config-1 workload, and every rank's
report is bitwise identical to the single-process Evaluator — the paper's
"1 vs 8 GPU scores identical" property, here with whole mini-batches LPT-sharded
across ranks and each rank's attention tiles packed from its own share."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, model, vocab, lines, result):
    import torch.distributed as dist

    import paper_2408_11853_b200 as mf
    from paper_2408_11853_b200.parallel import DistributedEvaluator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = mf.EvaluatorConfig(model=model, vocab=vocab, quiet=True, device=0,
                                 batch=mf.BatchConfig(mini_batch=32, maxi_batch_factor=4))
        with DistributedEvaluator(cfg) as ev:
            result[rank] = ev.evaluate_lines(lines).segment_scores
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_score_bitwise_like_one_process(fixture_dir, vocab_path, world):
    import torch.multiprocessing as mp

    import paper_2408_11853_b200 as mf
    from conftest import write_model
    from oracle import fixtures as fx

    c1 = fx.CONFIGS[1]
    man = fx.tiny_manifest("comet", **{k: c1[k] for k in
                                       ("d_model", "n_heads", "n_layers", "d_ffn", "head_hidden")})
    model = write_model(fixture_dir / "dist_c1.mfrg", man, fx.fixture_weights(man, 1234))
    lines = fx.fixture_tsv_lines("comet", 600, seed=3)
    with mf.Evaluator(mf.EvaluatorConfig(model=model, vocab=vocab_path, quiet=True,
                                         batch=mf.BatchConfig(mini_batch=32,
                                                              maxi_batch_factor=4))) as ev:
        solo = ev.evaluate_lines(lines).segment_scores
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, vocab_path, lines, result))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for r in range(world):
        assert result[r] == solo
    assert np.isfinite(solo).all()


def test_bench_self_launches_ranks_through_distributed_evaluator(tmp_path):
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (MFG_BENCH_BACKEND=gloo lets both share this box's GPU: a code-path check,
    not a measurement); the e2e leg runs DistributedEvaluator."""
    import json
    import subprocess
    import sys

    from conftest import ROOT
    env = dict(os.environ, MFG_BENCH_BACKEND="gloo", MFG_BENCH_DIR=str(tmp_path))
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "1",
                        "--steps", "2", "--warmup", "3", "--records-per-step", "512"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_records"] == 1024
    assert "DistributedEvaluator" in line["e2e"]["path"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
