"""`GpuScoringModel`: the device replacement of the reference `ScoringModel`.

Same constructor shape `(container, compute_mode)` and the same
`score_records(encoded_records) -> np.float32[n]` contract as
`pkg/src/metricforge/encoder.py:94-226`, implemented by libmfgpu
(include/mfgpu.h) on one B200. `score_packed` is the zero-copy fast path used
by `Evaluator`: role-major token ids + cu_seqlens straight from libmfhost.

Precisions (`EvaluatorConfig.precision`):
  "fp32"    the parity path: every GEMM operand is an fp16 hi/lo pair (~22
            significant bits) and each k-step issues 3 tcgen05 MMAs into an fp32
            TMEM accumulator (|Δ| ≤ 1e-3 per segment against the fp32 reference)
  "bf16x3"  the same with bf16 pieces (~16 bits, full fp32 range)
  "bf16"    one bf16 MMA per k-step — reported separately with its error stats
  "fp16"    the reference's own fp16 mode (`encoder.py:105, 120-130`): binary16
            weights and activations, one fp16 MMA per k-step (fp16 products are
            exact in the fp32 accumulator), binary16 rounding at every point the
            reference rounds; selected by `fp16=True` / ComputeMode.FP16
"""

from __future__ import annotations

import ctypes as C
import enum
import functools
import os
import threading

import numpy as np

from . import native
from .errors import ContainerError, DeviceError
from .kinds import N_SEQUENCES, Kind

PRECISIONS = {"fp32": 0, "bf16": 1, "bf16x3": 2, "fp16": 3}


class ComputeMode(enum.Enum):
    FP32 = "fp32"
    FP16 = "fp16"

    @classmethod
    def parse(cls, value):
        if isinstance(value, cls):
            return value
        # the reference's own ComputeMode (metricforge.encoder) when the
        # reference Evaluator constructs this model through its seam
        value = getattr(value, "value", value)
        try:
            return cls(value)
        except ValueError:
            raise ValueError(f"unknown compute mode {value!r}") from None


def default_precision(compute_mode) -> str:
    """fp32 keeps the parity path; the reference's fp16 flag (binary16
    storage) selects the device path with the same binary16 semantics."""
    return "fp32" if ComputeMode.parse(compute_mode) is ComputeMode.FP32 else "fp16"


def _device_ordinal(device) -> int:
    if device is None:
        return int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("MFG_DEVICE_FROM_RANK") else 0
    if isinstance(device, int):
        return device
    s = str(device)
    if s.startswith("cuda"):
        return int(s.split(":", 1)[1]) if ":" in s else 0
    return int(s)


# feature width per kind, in units of d_model (`encoder.py:198-212`)
FEATURE_WIDTH = {Kind.COMET_QE: 4, Kind.COMET: 6, Kind.BLEURT: 1}


def required_tensor_shapes(manifest) -> dict:
    """Tensor name -> shape contract of a manifest, the one `mfg_create`
    enforces natively (`csrc/container.hpp`); same names and shapes as the
    reference's `required_tensor_shapes` (`encoder.py:69-91`)."""
    d, f = int(manifest.d_model), int(manifest.d_ffn)
    out = {"emb.tok": (int(manifest.vocab_size), d), "emb.pos": (int(manifest.max_position), d)}
    layer = {f"att.{p}.{t}": ((d, d) if t == "w" else (d,)) for p in "qkvo" for t in "wb"}
    layer.update({f"{n}.{t}": (d,) for n in ("norm1", "norm2") for t in "gb"})
    layer.update({"ffn.w1": (d, f), "ffn.b1": (f,), "ffn.w2": (f, d), "ffn.b2": (d,)})
    for i in range(int(manifest.n_layers)):
        out.update({f"layer.{i}.{k}": v for k, v in layer.items()})
    widths = [FEATURE_WIDTH[Kind.parse(manifest.like)] * d, *map(int, manifest.head_hidden), 1]
    for j, (a, b) in enumerate(zip(widths, widths[1:])):
        out[f"head.{j}.w"], out[f"head.{j}.b"] = (a, b), (b,)
    return out


@functools.lru_cache(maxsize=None)
def _reference_errors():
    import importlib
    ref = importlib.import_module("metricforge.errors")

    class ReferenceDeviceError(DeviceError, ref.MetricForgeError):
        """DeviceError that is also the reference's MetricForgeError."""

    return ref.ContainerError, ReferenceDeviceError


def _error_classes(container):
    """(ContainerError, DeviceError) to raise. When the caller is the reference
    itself (its `Evaluator` constructs the model at `evaluate.py:151` with a
    `metricforge.container.ModelContainer`), container errors are the
    reference's own `metricforge.errors.ContainerError` so its callers'
    `except` clauses still match (`encoder.py:108-115`)."""
    mod = type(container).__module__ or ""
    if mod.split(".")[0] == "metricforge":
        return _reference_errors()
    return ContainerError, DeviceError


class GpuScoringModel:
    """Drop-in for the reference `ScoringModel` at its seam: the constructor
    takes `(container, compute_mode)` (the reference's own container and
    ComputeMode objects, or a path / this package's), and `score_records`
    keeps the contract the reference `Evaluator` relies on
    (`evaluate.py:151, 166, 173-175`). The padded-batch internals `forward`,
    `pool`, `encode_pooled`, `features` and `head` (`encoder.py:154-212`)
    are not part of that contract and are not provided: the device path fuses
    them into one call per batch."""

    def __init__(self, container, compute_mode=ComputeMode.FP32, device=None, precision=None,
                 max_tokens=0, max_records=0, profile=False):
        path = container if isinstance(container, (str, os.PathLike)) else container.path
        self._ContainerError, self._DeviceError = _error_classes(container)
        self.manifest = None if isinstance(container, (str, os.PathLike)) else container.manifest
        self.mode = ComputeMode.parse(compute_mode)
        self.precision = precision or default_precision(self.mode)
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r} "
                             f"(known: {', '.join(PRECISIONS)})")
        self._lib = native.gpu()
        cfg = native.MfgConfig(os.fsencode(str(path)), _device_ordinal(device),
                               PRECISIONS[self.precision], int(max_tokens), int(max_records),
                               int(bool(profile)))
        handle = C.c_void_p()
        rc = self._lib.mfg_create(C.byref(cfg), C.byref(handle))
        if rc != 0:
            code, msg = native.last_error(None)
            raise self._error(rc, msg)
        self._h = handle
        self._lock = threading.Lock()
        info = native.MfgModelInfo()
        self._lib.mfg_get_model_info(self._h, C.byref(info))
        self.info = info
        self.kind = Kind.parse(("comet-qe", "comet", "bleurt")[info.kind])
        self.n_roles = int(info.n_roles)
        self.max_position = int(info.max_position)
        self.vocab_size = int(info.vocab_size)

    def _error(self, rc, msg):
        """C-ABI return code -> exception: 2 usage (ValueError, as the
        reference's id/length checks), 3 container, else device/runtime."""
        if rc == 2:
            return ValueError(msg)
        return (self._ContainerError if rc == 3 else self._DeviceError)(msg)

    # ------------------------------------------------------------------ core
    def score_packed(self, ids, cu_seqlens, n_records) -> np.ndarray:
        """ids int32 role-major, cu_seqlens int64[n_roles*n+1] -> float32[n]."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int64)
        out = np.empty(n_records, dtype=np.float32)
        if n_records == 0:
            return out
        with self._lock:
            if self._h is None:
                raise self._DeviceError("scoring model is closed")
            rc = self._lib.mfg_score_batch(self._h, int(n_records), self.n_roles,
                                           native.ptr(ids, C.c_int32), native.ptr(cu, C.c_int64),
                                           native.ptr(out, C.c_float))
            if rc != 0:
                _, msg = native.last_error(self._h)
                raise self._error(rc, msg)
        return out

    def score_device(self, ids_ptr, cu_seqlens, n_records, scores_ptr):
        """Device-resident variant: ids_ptr / scores_ptr are device addresses
        (int32 role-major ids, float32[n] out); cu_seqlens is a host int64 array."""
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int64)
        with self._lock:
            rc = self._lib.mfg_score_device(self._h, int(n_records), self.n_roles,
                                            C.c_void_p(ids_ptr), native.ptr(cu, C.c_int64),
                                            C.c_void_p(scores_ptr))
            if rc != 0:
                _, msg = native.last_error(self._h)
                raise self._error(rc, msg)

    def set_stream(self, stream_handle):
        """Route every launch to an external cudaStream_t (int handle; 0 = own)."""
        self._lib.mfg_set_stream(self._h, C.c_void_p(stream_handle or None))

    def score_records(self, encoded_records) -> np.ndarray:
        """`encoded_records`: per record, the TokenSequence list of encode_fields
        for this model's kind (role order). Returns float32 scores in order."""
        n = len(encoded_records)
        seqs = [encoded_records[i][k].ids for k in range(self.n_roles) for i in range(n)]
        lens = np.fromiter((len(s) for s in seqs), dtype=np.int64, count=len(seqs))
        if n and lens.max() > self.max_position:  # pad_batch's check (batching.py:83-86)
            raise ValueError(f"sequence length {int(lens.max())} exceeds limit {self.max_position}")
        cu = np.zeros(len(seqs) + 1, dtype=np.int64)
        np.cumsum(lens, out=cu[1:])
        ids = np.fromiter((t for s in seqs for t in s), dtype=np.int64, count=int(cu[-1]))
        if ids.size and (ids.min() < 0 or ids.max() >= self.vocab_size):
            raise ValueError(f"token id out of range for vocab_size {self.vocab_size}")
        return self.score_packed(ids.astype(np.int32), cu, n)

    # ------------------------------------------------------------------ stats
    def stats(self) -> dict:
        s = native.MfgStats()
        self._lib.mfg_get_stats(self._h, C.byref(s))
        out = {k: getattr(s, k) for k in ("device_ms", "calls", "records", "tokens", "chunks",
                                           "kernel_launches", "fallback_chunks",
                                           "fallback_records")}
        out["classes"] = {
            name: {"ms": s.class_ms[i], "launches": s.class_launches[i],
                   "flops": s.class_flops[i], "bytes": s.class_bytes[i]}
            for i, name in enumerate(native.CLASS_NAMES)}
        return out

    def set_profile(self, enable: bool):
        """Per-launch CUDA-event timing on / off (class_ms in stats())."""
        self._lib.mfg_set_profile(self._h, int(bool(enable)))

    def load_phases(self) -> dict:
        """mfg_create phase timings in ms (context, open, embeddings, layers, head, workspaces)."""
        return {k: float(self.info.load_ms[i]) for i, k in enumerate(native.LOAD_PHASES)}

    def reset_stats(self):
        self._lib.mfg_reset_stats(self._h)

    def close(self):
        with self._lock:
            if self._h is not None:
                self._lib.mfg_destroy(self._h)
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def n_sequences(kind) -> int:
    return N_SEQUENCES[Kind.parse(kind)]
