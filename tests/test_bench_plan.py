"""bench.py's strong-scaling split (host logic, CPU): the reference plan of the
shared set, whole mini-batches LPT-assigned to ranks, each rank's share cut
into K steps. Every record is scored exactly once across ranks and steps,
steps hold whole mini-batches, and the ranks' costs are balanced."""

import numpy as np
import pytest

import bench
from paper_2408_11853_b200.batching import BatchConfig
from paper_2408_11853_b200.parallel import CostModel


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_rank_steps_cover_every_record_once(world):
    rng = np.random.default_rng(world)
    n, ns, K = 5000, 3, 7
    lens = rng.integers(3, 129, size=(n, ns))
    off = np.zeros(n * ns + 1, np.int64)
    np.cumsum(lens.ravel(), out=off[1:])
    cfg, cost = BatchConfig(), CostModel()
    seen, loads, order0 = [], [], None
    for r in range(world):
        order, steps = bench.rank_steps(off, ns, n, cfg, world, r, K, cost)
        order0 = order if order0 is None else order0
        assert np.array_equal(order, order0)  # every rank computes the same plan
        assert len(steps) == K
        for pos in steps:
            if len(pos):  # whole mini-batches: runs of 128 starting on a boundary
                assert pos[0] % cfg.mini_batch == 0
        mine = np.concatenate(steps)
        seen.append(mine)
        loads.append(cost(lens[order[mine]].ravel()))
    allpos = np.sort(np.concatenate(seen))
    assert np.array_equal(allpos, np.arange(n))
    if world > 1:
        assert max(loads) / (sum(loads) / world) < 1.15


def test_reference_arm_prints_one_line(tmp_path):
    """`bench.py --impl reference` (the driver's reference arm): the reference's
    own CPU Evaluator (baseline/_ref when installed, else the oracle port) on the
    config's workload; one JSON line with impl, cpu_baseline and a zero-copy e2e."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT
    env = dict(os.environ, MFG_BENCH_DIR=str(tmp_path))
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "segments/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
