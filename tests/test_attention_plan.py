"""Host-side attention work planner (att_plan_tiles in libmfgpu, called through
the test entry mfgt_plan_tiles; no GPU needed): every sequence is scheduled
exactly once, tiles hold <= 4 whole sequences at 32-aligned rows inside 128,
long sequences are covered by 128-query blocks."""

import ctypes as C

import numpy as np
import pytest

from paper_2408_11853_b200 import native


@pytest.fixture(scope="module")
def lib():
    return native.gpu()


def plan(lib, lens, tc_ok=1):
    cu = np.zeros(len(lens) + 1, np.int32)
    cu[1:] = np.cumsum(lens)
    cap = 4 * len(lens) + 16
    tiles = np.zeros(cap * 8, np.int32)
    work = np.zeros(cap * 2, np.int32)
    nt, nw = C.c_int32(), C.c_int32()
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    assert lib.mfgt_plan_tiles(P(cu), len(lens), tc_ok, P(tiles), C.byref(nt), P(work),
                               C.byref(nw), cap) == 0
    return cu, tiles[:nt.value * 8].reshape(-1, 8), work[:nw.value * 2].reshape(-1, 2)


@pytest.mark.parametrize("seed", range(6))
def test_plan_covers_every_sequence_once(lib, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 513, 300) if seed % 2 else rng.integers(2, 129, 500)
    cu, tiles, work = plan(lib, lens.tolist())
    seen = {}
    for t in tiles:
        t0, ln = t[:4], t[4:]
        used = ln > 0
        assert used.any() and used.sum() <= 4
        assert not (used[1:] & ~used[:-1]).any()          # slots fill from the front
        rows = sum((int(l) + 31) // 32 * 32 for l in ln[used])
        assert rows <= 128
        for a, l in zip(t0[used], ln[used]):
            s = int(np.searchsorted(cu, a))
            assert cu[s] == a and cu[s + 1] - cu[s] == l and l <= 128
            seen[s] = seen.get(s, 0) + 1
    for s, q0 in work:
        L = cu[s + 1] - cu[s]
        assert L > 128 and q0 % 128 == 0 and q0 < L
        seen[s] = seen.get(s, 0) + (1 if q0 == 0 else 0)
    long_blocks = {}
    for s, q0 in work:
        long_blocks.setdefault(int(s), []).append(int(q0))
    for s, qs in long_blocks.items():
        L = cu[s + 1] - cu[s]
        assert sorted(qs) == list(range(0, L, 128))
    assert sorted(seen) == list(range(len(lens))) and set(seen.values()) == {1}


def test_plan_without_tensor_cores_uses_64_query_blocks(lib):
    lens = [3, 64, 65, 200]
    cu, tiles, work = plan(lib, lens, tc_ok=0)
    assert len(tiles) == 0
    want = [(s, q) for s, L in enumerate(lens) for q in range(0, L, 64)]
    assert [tuple(w) for w in work] == want


def test_plan_packs_short_sequences(lib):
    # 32-row granules: four 20-token sequences share one tile, a 100-token one
    # (4 granules) starts the next
    cu, tiles, work = plan(lib, [20, 20, 20, 20, 100, 32, 33])
    assert len(work) == 0
    assert tiles[0][4:].tolist() == [20, 20, 20, 20]
    assert tiles[1][4:].tolist() == [100, 0, 0, 0]
    assert tiles[2][4:].tolist() == [32, 33, 0, 0]
