"""Window -> length-sorted mini-batch plan, padding and order restore.

Mirrors `pkg/src/metricforge/batching.py`: `BatchConfig`, `BatchPlan`,
`PaddedBatch`, `plan_batches`, `pad_batch`, `restore_order`. The plan is
computed by libmfhost (`mfh_plan`, a stable per-window sort on -length), which
is bit-identical to the reference's `sorted(key=(-len, idx))`.

The device path never pads: sequences travel token-packed with cu_seqlens
(`pack_roles`), which the reference's padding invariance (`SPEC.md:228`)
makes equivalent.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native

PAD_ID = 0


@dataclass
class BatchConfig:
    mini_batch: int = 128
    maxi_batch_factor: int = 8
    sort_by_length: bool = True
    workers: int = 1

    def __post_init__(self):
        for key in ("mini_batch", "maxi_batch_factor", "workers"):
            if getattr(self, key) < 1:
                raise ValueError(f"{key} must be positive")

    @property
    def window(self):
        return self.mini_batch * self.maxi_batch_factor


@dataclass
class BatchPlan:
    batches: list
    order: list = field(default_factory=list)

    def __post_init__(self):
        if not self.order:
            self.order = [i for b in self.batches for i in b]


@dataclass
class PaddedBatch:
    ids: np.ndarray
    mask: np.ndarray
    segment_of: str = ""


def plan_order(lengths, config: BatchConfig) -> np.ndarray:
    """order[scoring position] = original index, as int64 array."""
    lens = np.ascontiguousarray(lengths, dtype=np.int64)
    order = np.empty(len(lens), dtype=np.int64)
    rc = native.host().mfh_plan(native.ptr(lens, C.c_int64), len(lens), config.mini_batch,
                                config.maxi_batch_factor, int(bool(config.sort_by_length)),
                                native.ptr(order, C.c_int64))
    if rc != 0:
        raise ValueError("invalid batch configuration")
    return order


def plan_batches(lengths, config: BatchConfig) -> BatchPlan:
    order = plan_order(lengths, config).tolist()
    mb = config.mini_batch
    return BatchPlan(batches=[order[s:s + mb] for s in range(0, len(order), mb)], order=order)


def pad_batch(sequences, segment_of="", limit=None) -> PaddedBatch:
    if not sequences:
        raise ValueError("cannot pad an empty batch")
    widths = [len(s) for s in sequences]
    if limit is not None:
        over = [w for w in widths if w > limit]
        if over:
            raise ValueError(f"sequence length {over[0]} exceeds limit {limit}")
    ids = np.full((len(sequences), max(widths)), PAD_ID, dtype=np.int32)
    mask = np.zeros(ids.shape, dtype=bool)
    for r, s in enumerate(sequences):
        ids[r, :len(s)] = s
        mask[r, :len(s)] = True
    return PaddedBatch(ids=ids, mask=mask, segment_of=segment_of)


def restore_order(scores, plan):
    order = plan.order if isinstance(plan, BatchPlan) else plan
    if len(scores) != len(order):
        raise ValueError(f"got {len(scores)} scores for {len(order)} planned records")
    out = [None] * len(scores)
    for pos, orig in enumerate(order):
        out[orig] = scores[pos]
    return out


def pack_roles(ids, seq_off, n_seqs, order):
    """Record-major encoding -> role-major (ids, cu_seqlens) for records `order`."""
    order = np.ascontiguousarray(order, dtype=np.int64)
    m = len(order)
    lens = np.diff(seq_off).reshape(-1, n_seqs)[order]
    out = np.empty(int(lens.sum()), dtype=np.int32)
    cu = np.empty(n_seqs * m + 1, dtype=np.int64)
    native.host().mfh_pack_roles(native.ptr(ids, C.c_int32), native.ptr(seq_off, C.c_int64),
                                 n_seqs, native.ptr(order, C.c_int64), m,
                                 native.ptr(out, C.c_int32), native.ptr(cu, C.c_int64))
    return out, cu
