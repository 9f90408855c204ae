"""Seeded fixtures and synthetic workloads (test / bench infrastructure).

Two families:

1. The reference's own test fixtures, restated so the golden files it ships
   (`pkg/tests/golden/eval_qe.txt`) can be reproduced without importing it:
   the 64-line vocabulary (`pkg/tests/fixturegen.py:29-37`), the tiny
   manifest defaults (`:46-59`), the weight RNG draw order (`:62-75`, which
   walks `required_tensor_shapes` order, `pkg/src/metricforge/encoder.py:69-91`)
   and the random TSV text generator (`:133-148`).

2. The synthetic workloads of SURVEY.md §8(d) for configs 1-5: a
   `▁w<i>` vocabulary in which every word is exactly one piece, uniform or
   log-normal content lengths, and N(0, 0.02²) BERT-scale weights.
"""

from __future__ import annotations

import numpy as np

MARKER = "▁"
SPECIALS = ["<pad>", "<unk>", "<s>", "</s>", "<sep>"]
FEATURE_MULT = {"comet-qe": 4, "comet": 6, "bleurt": 1}
FIELDS = {"comet-qe": ("S", "T"), "comet": ("S", "T", "R"), "bleurt": ("T", "R")}

_FIXTURE_WORDS = (
    "the north wind and sun were disputing which was stronger when a traveler "
    "came along wrapped in warm cloak they agreed that one who first succeeded "
    "making take his"
).split()


# --------------------------------------------------------------------------
# reference fixture family
# --------------------------------------------------------------------------

def fixture_vocab_lines():
    toks = list(SPECIALS)
    toks += [MARKER + w for w in _FIXTURE_WORDS]
    toks += [MARKER, "ing", "ed", "er"]
    toks += [chr(c) for c in range(ord("a"), ord("z") + 1)]
    assert len(toks) == 64
    return toks


def write_vocab(path, lines):
    with open(path, "w", encoding="utf-8") as f:
        f.write("\n".join(lines) + "\n")
    return str(path)


def tiny_manifest(kind, **over):
    m = dict(like=kind, vocab_size=64, d_model=16, n_heads=2, n_layers=2, d_ffn=32,
             max_position=128, norm_style="post", head_hidden=[16])
    m.update(over)
    return m


def tensor_shapes(man) -> list:
    """Ordered (name, shape) pairs, the order weights are drawn and stored in."""
    d, f = man["d_model"], man["d_ffn"]
    out = [("emb.tok", (man["vocab_size"], d)), ("emb.pos", (man["max_position"], d))]
    for i in range(man["n_layers"]):
        p = f"layer.{i}"
        for proj in "qkvo":
            out += [(f"{p}.att.{proj}.w", (d, d)), (f"{p}.att.{proj}.b", (d,))]
        for nm in ("norm1", "norm2"):
            out += [(f"{p}.{nm}.g", (d,)), (f"{p}.{nm}.b", (d,))]
        out += [(f"{p}.ffn.w1", (d, f)), (f"{p}.ffn.b1", (f,)),
                (f"{p}.ffn.w2", (f, d)), (f"{p}.ffn.b2", (d,))]
    widths = [FEATURE_MULT[str(man["like"])] * d] + list(man["head_hidden"]) + [1]
    for j in range(len(widths) - 1):
        out += [(f"head.{j}.w", (widths[j], widths[j + 1])), (f"head.{j}.b", (widths[j + 1],))]
    return out


def fixture_weights(man, seed) -> dict:
    """Same RNG consumption as the reference fixture generator."""
    rng = np.random.default_rng(seed)
    w = {}
    for name, shape in tensor_shapes(man):
        z = rng.standard_normal(shape)
        if name.endswith(".g"):
            a = 1.0 + 0.1 * z
        elif name.endswith(".b") and ".norm" in name:
            a = 0.05 * z
        else:
            a = 0.25 * z
        w[name] = a.astype(np.float32)
    return w


def _fixture_texts(rng, count):
    texts = []
    for _ in range(count):
        n = int(rng.integers(1, 12))
        words = [_FIXTURE_WORDS[int(rng.integers(0, len(_FIXTURE_WORDS)))] for _ in range(n)]
        if rng.random() < 0.15:
            words.insert(int(rng.integers(0, n)), "Zq!7")
        texts.append(" ".join(words))
    return texts


def fixture_tsv_lines(kind, count, seed=0):
    rng = np.random.default_rng(seed)
    cols = [_fixture_texts(rng, count) for _ in FIELDS[str(kind)]]
    return ["\t".join(v) for v in zip(*cols)]


# --------------------------------------------------------------------------
# synthetic workloads, SURVEY.md §8(d)
# --------------------------------------------------------------------------

CONFIGS = {
    1: dict(like="comet", vocab_size=64, d_model=256, n_heads=4, n_layers=2, d_ffn=1024,
            max_position=128, norm_style="post", head_hidden=[256]),
    2: dict(like="comet", vocab_size=250002, d_model=1024, n_heads=16, n_layers=24,
            d_ffn=4096, max_position=512, norm_style="post", head_hidden=[3072, 1024]),
    3: dict(like="comet-qe", vocab_size=250002, d_model=1024, n_heads=16, n_layers=24,
            d_ffn=4096, max_position=512, norm_style="post", head_hidden=[3072, 1024]),
    4: dict(like="bleurt", vocab_size=119547, d_model=1152, n_heads=18, n_layers=32,
            d_ffn=4608, max_position=512, norm_style="post", head_hidden=[1152]),
    5: dict(like="comet-qe", vocab_size=250880, d_model=2560, n_heads=32, n_layers=36,
            d_ffn=10240, max_position=512, norm_style="post", head_hidden=[3072, 1024]),
}
CONFIG_NAMES = {
    1: "tiny-comet-d256-l2", 2: "wmt22-comet-da (XLM-R-large shape)",
    3: "wmt22-cometkiwi-da (InfoXLM-large shape)", 4: "bleurt-20 (RemBERT shape)",
    5: "wmt23-cometkiwi-da-xl (XLM-R-XL shape)",
}
TEXT_SEED = 2408
WEIGHT_SEED = 11853


def synthetic_vocab_lines(vocab_size):
    return list(SPECIALS) + [f"{MARKER}w{i}" for i in range(vocab_size - len(SPECIALS))]


def synthetic_weights(man, seed=WEIGHT_SEED):
    """Generator of (name, float32 array): matrices/embeddings N(0,0.02²),
    LN gains 1+0.02·N, biases 0.02·N. Yields one tensor at a time so
    multi-GB models never sit in RAM twice."""
    rng = np.random.default_rng(seed)
    for name, shape in tensor_shapes(man):
        z = rng.standard_normal(shape, dtype=np.float32)
        if name.endswith(".g"):
            z *= np.float32(0.02)
            z += np.float32(1.0)
        else:
            z *= np.float32(0.02)
        yield name, z


def _content_lengths(cfg, rng, n):
    if cfg == 5:
        L = np.rint(np.exp(rng.normal(np.log(24.0), 0.8, size=n)))
        return np.clip(L, 1, 510).astype(np.int64)
    hi = 62 if cfg == 4 else 126
    return rng.integers(1, hi + 1, size=n)


def synthetic_tsv_lines(cfg, count, seed=TEXT_SEED):
    """Records of `cfg`'s kind. Each word `w<i>` encodes to exactly one id,
    so a field with n words becomes n+2 tokens ([BOS] .. [EOS])."""
    man = CONFIGS[cfg]
    kind = man["like"]
    rng = np.random.default_rng(seed)
    n_words = man["vocab_size"] - len(SPECIALS)
    cols = []
    for _ in FIELDS[kind]:
        lens = _content_lengths(cfg, rng, count)
        ids = rng.integers(0, n_words, size=int(lens.sum()))
        words = np.char.add("w", ids.astype(str))
        out, pos = [], 0
        for L in lens.tolist():
            out.append(" ".join(words[pos:pos + L].tolist()))
            pos += L
        cols.append(out)
    return ["\t".join(v) for v in zip(*cols)]


# --------------------------------------------------------------------------
# full-size parity subsets (SURVEY.md §8(d) parity protocol)
# --------------------------------------------------------------------------

PARITY_POOL = 20000
PARITY_SEED = TEXT_SEED + 31
PARITY_SIZES = {2: 512, 3: 512, 4: 512, 5: 64}


def parity_subset(cfg, n_sub=None, pool=PARITY_POOL, seed=PARITY_SEED):
    """Length-stratified subset of config `cfg`'s synthetic workload.

    Draws `pool` records from the §8(d) generator, ranks them by total
    content length (ties by index) and keeps `n_sub` records at evenly spaced
    ranks, the shortest and the longest included (config 5's 510-token tail
    reaches the long-sequence attention path). Returned in pool order, as a
    stream would present them. Returns (pool_indices, lines)."""
    n_sub = PARITY_SIZES[cfg] if n_sub is None else n_sub
    lines = synthetic_tsv_lines(cfg, pool, seed=seed)
    total = np.array([sum(len(c.split()) for c in ln.split("\t")) for ln in lines])
    ranked = np.lexsort((np.arange(pool), total))
    picks = ranked[np.rint(np.linspace(0, pool - 1, n_sub)).astype(np.int64)]
    idx = np.sort(np.unique(picks))
    return idx.tolist(), [lines[i] for i in idx]
