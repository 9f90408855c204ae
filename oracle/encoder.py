"""Encoder oracle: numpy restatement of the reference scoring model.

Numerics follow `pkg/src/metricforge/encoder.py`:

  x     = E_tok[ids] + E_pos[0..L-1]                             (:166-168)
  post  : x = LN1(x + Attn(x));  x = LN2(x + FFN(x))             (:176-178)
  pre   : x = x + Attn(LN1(x));  x = x + FFN(LN2(x))             (:173-175)
  Attn  : per-head softmax(q kᵀ / sqrt(d/h), PAD keys -> -inf) v  (:132-147, 60-66)
  FFN   : gelu_tanh(x W1 + b1) W2 + b2                           (:47-49, 149-152)
  LN    : population variance, eps 1e-5                          (:52-57)
  pool  : BOS row of the last layer                              (:181-185)
  feats : QE [t,s,t*s,|t-s|]  COMET [t,r,t*s,t*r,|t-s|,|t-r|]  BLEURT [j]  (:198-212)
  head  : affine+tanh per hidden width, final affine, column 0    (:190-196)

"fp16" mode keeps weights/activations in IEEE binary16 and rounds at the
same points as the reference (matmul result, bias add, LN output, GELU,
residual sums, attention inputs/outputs, head stages) with fp32
accumulation (`:105, 120-130`).
"""

from __future__ import annotations

import math

import numpy as np

from .fixtures import tensor_shapes

F32 = np.float32
ROLES = {"comet-qe": 2, "comet": 3, "bleurt": 1}


def _gelu(x):
    c = math.sqrt(2.0 / math.pi)
    return 0.5 * x * (1.0 + np.tanh(c * (x + 0.044715 * x ** 3)))


def _ln(x, g, b, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


class OracleModel:
    def __init__(self, manifest: dict, weights: dict, mode: str = "fp32"):
        self.m = dict(manifest)
        self.kind = str(self.m["like"])
        self.store = np.float16 if mode == "fp16" else F32
        self.w = {}
        for name, shape in tensor_shapes(self.m):
            arr = np.asarray(weights[name])
            if tuple(arr.shape) != tuple(shape):
                raise ValueError(f"tensor {name!r} has shape {arr.shape}, expected {shape}")
            self.w[name] = arr.astype(self.store)
        self.scale = 1.0 / math.sqrt(self.m["d_model"] / self.m["n_heads"])
        self.n_stages = len(self.m["head_hidden"]) + 1

    # -- primitives in the reference's rounding order ---------------------
    def _mm(self, a, b):
        return (a.astype(F32, copy=False) @ b.astype(F32, copy=False)).astype(self.store, copy=False)

    def _aff(self, x, p):
        return self._mm(x, self.w[p + ".w"]) + self.w[p + ".b"]

    def _norm(self, x, g, b):
        return _ln(x.astype(F32, copy=False), g.astype(F32), b.astype(F32)).astype(self.store, copy=False)

    def _attn(self, x, keymask, i):
        B, L, d = x.shape
        H = self.m["n_heads"]
        dh = d // H

        def heads(t):
            return t.reshape(B, L, H, dh).transpose(0, 2, 1, 3).astype(F32)

        p = f"layer.{i}.att"
        q, k, v = (heads(self._aff(x, f"{p}.{n}")) for n in "qkv")
        s = (q @ k.transpose(0, 1, 3, 2)) * self.scale
        s = np.where(keymask[:, None, None, :], s, -np.inf)
        s = np.exp(s - s.max(axis=-1, keepdims=True))
        s = s / s.sum(axis=-1, keepdims=True)
        ctx = (s @ v).transpose(0, 2, 1, 3).reshape(B, L, d)
        return self._aff(ctx.astype(self.store, copy=False), f"{p}.o")

    def _ffn(self, x, i):
        p = f"layer.{i}.ffn"
        h = self._mm(x, self.w[p + ".w1"]) + self.w[p + ".b1"]
        h = _gelu(h.astype(F32)).astype(self.store, copy=False)
        return self._mm(h, self.w[p + ".w2"]) + self.w[p + ".b2"]

    # -- public --------------------------------------------------------------
    def encode(self, seqs):
        """Final-layer states [B, Lmax, d] for a list of id lists (padded)."""
        L = max(len(s) for s in seqs)
        if L > self.m["max_position"]:
            raise ValueError(f"sequence length {L} exceeds max_position {self.m['max_position']}")
        ids = np.zeros((len(seqs), L), dtype=np.int64)
        mask = np.zeros((len(seqs), L), dtype=bool)
        for r, s in enumerate(seqs):
            ids[r, :len(s)] = s
            mask[r, :len(s)] = True
        if ids.min() < 0 or ids.max() >= self.m["vocab_size"]:
            raise ValueError("token id out of range")
        x = (self.w["emb.tok"][ids] + self.w["emb.pos"][:L]).astype(self.store, copy=False)
        pre = self.m.get("norm_style", "post") == "pre"
        for i in range(self.m["n_layers"]):
            g1, b1 = self.w[f"layer.{i}.norm1.g"], self.w[f"layer.{i}.norm1.b"]
            g2, b2 = self.w[f"layer.{i}.norm2.g"], self.w[f"layer.{i}.norm2.b"]
            if pre:
                x = x + self._attn(self._norm(x, g1, b1), mask, i)
                x = x + self._ffn(self._norm(x, g2, b2), i)
            else:
                x = self._norm(x + self._attn(x, mask, i), g1, b1)
                x = self._norm(x + self._ffn(x, i), g2, b2)
        return x

    def pooled(self, seqs):
        if any(len(s) == 0 for s in seqs):
            raise ValueError("cannot pool a row with no tokens")
        return self.encode(seqs)[:, 0, :]

    def features(self, pooled):
        p = [a.astype(F32) for a in pooled]
        if self.kind == "comet-qe":
            s, t = p
            parts = [t, s, t * s, np.abs(t - s)]
        elif self.kind == "comet":
            s, t, r = p
            parts = [t, r, t * s, t * r, np.abs(t - s), np.abs(t - r)]
        else:
            parts = [p[0]]
        return np.concatenate(parts, axis=1)

    def head(self, feats):
        x = feats.astype(self.store, copy=False)
        for j in range(self.n_stages):
            x = self._mm(x, self.w[f"head.{j}.w"]) + self.w[f"head.{j}.b"]
            if j < self.n_stages - 1:
                x = np.tanh(x.astype(F32)).astype(self.store, copy=False)
        return x[:, 0].astype(F32)

    def score(self, records):
        """records: list of per-record id-list lists in role order -> float32[n]."""
        n_roles = ROLES[self.kind]
        pooled = [self.pooled([rec[r] for rec in records]) for r in range(n_roles)]
        return self.head(self.features(pooled))
