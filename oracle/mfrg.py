"""Independent `.mfrg` container codec for tests (oracle side).

Layout restated from the reference's module docstring and writer
(`pkg/src/metricforge/container.py:1-17, 181-243`):

    "MFRG0001" | u32le header_len | canonical-JSON header | 0-pad to 64
    | payload (tensor regions at 64-byte aligned payload offsets)

The manifest checksum is sha256 over the payload bytes only. Canonical JSON
is `sort_keys=True, separators=(",", ":"), ensure_ascii=False`.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np

MAGIC = b"MFRG0001"
ALIGN = 64
_ELEM = {"f32": 4, "f16": 2}
_NP = {"f32": "<f4", "f16": "<f2"}


def _pad(n: int) -> int:
    return (-n) % ALIGN


def manifest_dict(like, vocab_size, d_model, n_heads, n_layers, d_ffn, max_position,
                  norm_style="post", head_hidden=(), checksum=""):
    return {
        "format_version": 1,
        "like": str(like),
        "vocab_size": int(vocab_size),
        "d_model": int(d_model),
        "n_heads": int(n_heads),
        "n_layers": int(n_layers),
        "d_ffn": int(d_ffn),
        "max_position": int(max_position),
        "norm_style": str(norm_style),
        "head_hidden": [int(w) for w in head_hidden],
        "checksum": checksum,
    }


def write(path, manifest: dict, tensors):
    """tensors: iterable of (name, dtype_str, np.ndarray). Returns checksum.

    Streams the payload twice (hash pass, write pass) instead of joining it,
    so multi-GB synthetic models do not need 2x their size in RAM.
    """
    tensors = list(tensors)
    index = []
    offset = 0
    for name, dtype, arr in tensors:
        nbytes = int(arr.size) * _ELEM[dtype]
        offset += _pad(offset)
        index.append({"name": name, "dtype": dtype, "shape": [int(s) for s in arr.shape],
                      "offset": offset, "nbytes": nbytes})
        offset += nbytes

    def payload_chunks():
        pos = 0
        for (name, dtype, arr), ent in zip(tensors, index):
            if ent["offset"] > pos:
                yield b"\x00" * (ent["offset"] - pos)
            yield np.ascontiguousarray(arr, dtype=_NP[dtype]).tobytes()
            pos = ent["offset"] + ent["nbytes"]

    h = hashlib.sha256()
    for c in payload_chunks():
        h.update(c)
    digest = h.hexdigest()
    man = dict(manifest)
    man["checksum"] = digest
    header = json.dumps({"manifest": man, "tensors": index}, sort_keys=True,
                        separators=(",", ":"), ensure_ascii=False).encode("utf-8")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(len(header).to_bytes(4, "little"))
        f.write(header)
        f.write(b"\x00" * _pad(len(MAGIC) + 4 + len(header)))
        for c in payload_chunks():
            f.write(c)
    return digest


def read(path):
    """Returns (manifest_dict, {name: np.ndarray(float32 or float16)})."""
    blob = open(path, "rb").read()
    if blob[:8] != MAGIC:
        raise ValueError("bad magic")
    hlen = int.from_bytes(blob[8:12], "little")
    header = json.loads(blob[12:12 + hlen].decode("utf-8"))
    start = 12 + hlen
    start += _pad(start)
    out = {}
    for ent in header["tensors"]:
        raw = blob[start + ent["offset"]: start + ent["offset"] + ent["nbytes"]]
        out[ent["name"]] = np.frombuffer(raw, dtype=_NP[ent["dtype"]]).reshape(ent["shape"])
    return header["manifest"], out
