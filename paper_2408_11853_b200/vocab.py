"""Plain-text vocabulary and bit-exact greedy segmentation (C++ backed).

API mirrors `pkg/src/metricforge/vocab.py`: `Vocabulary(tokens)`, `.encode`,
`load_vocab(path)`, `TokenSequence`, `encode_fields(vocab, record, like,
max_len)`. Matching runs in libmfhost (code-point trie; `csrc/host/tokenizer.cpp`);
`encode_batch` tokenises a whole window of records in one multi-threaded call.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import VocabularyError
from .kinds import KIND_CODE, N_SEQUENCES, Kind

PAD_ID, UNK_ID, BOS_ID, EOS_ID, SEP_ID = 0, 1, 2, 3, 4
SPECIAL_TOKENS = ("<pad>", "<unk>", "<s>", "</s>", "<sep>")
MARKER = "▁"


def _utf8(text: str) -> bytes:
    # surrogatepass keeps lone surrogates as one code point each, as in Python
    return text.encode("utf-8", "surrogatepass")


class Vocabulary:
    """Token table; ids are line numbers. Specials (ids 0-4) never match text."""

    def __init__(self, tokens):
        self.tokens = list(tokens)
        ids = {}
        for i, tok in enumerate(self.tokens):
            if not tok:
                raise VocabularyError(f"empty token at line {i + 1}")
            if tok in ids:
                raise VocabularyError(f"duplicate token {tok!r} at line {i + 1}")
            if "\n" in tok:
                raise VocabularyError(f"token at line {i + 1} contains a newline")
            ids[tok] = i
        if tuple(self.tokens[:5]) != SPECIAL_TOKENS:
            raise VocabularyError(
                f"first five tokens must be {list(SPECIAL_TOKENS)}, got {self.tokens[:5]}")
        self._ids = ids
        blob = "\n".join(self.tokens).encode("utf-8", "surrogatepass")
        handle = C.c_void_p()
        rc = native.host().mfh_vocab_create(blob, len(blob), len(self.tokens), C.byref(handle))
        if rc != 0:
            raise VocabularyError("native vocabulary construction failed")
        self._h = handle
        self._lib = native.host()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.mfh_vocab_destroy(h)
            self._h = None

    def __len__(self):
        return len(self.tokens)

    def id_of(self, token):
        return self._ids[token]

    @property
    def max_piece(self):
        return int(self._lib.mfh_vocab_max_piece(self._h))

    def encode(self, text: str) -> list:
        raw = _utf8(text)
        cap = 2 * len(raw) + 1  # ids <= code points + one marker per word
        out = np.empty(cap, dtype=np.int32)
        n = self._lib.mfh_encode(self._h, raw, len(raw), native.ptr(out, C.c_int32), cap)
        return out[:n].tolist()

    def encode_batch(self, kind: Kind, field_texts, max_len: int, n_threads: int = 0):
        """Tokenise n records at once. field_texts: list of per-record field
        string lists in (S, T, R) kind order. Returns (ids int32[total],
        seq_off int64[n * n_seqs + 1]) record-major."""
        kind = Kind.parse(kind)
        n = len(field_texts)
        pieces = [_utf8(v) for rec in field_texts for v in rec]
        offsets = np.zeros(len(pieces) + 1, dtype=np.int64)
        np.cumsum([len(p) for p in pieces], out=offsets[1:])
        blob = b"".join(pieces)
        ns = N_SEQUENCES[kind]
        cap = 2 * int(offsets[-1]) + 4 * ns * n + 8
        ids = np.empty(cap, dtype=np.int32)
        seq_off = np.zeros(n * ns + 1, dtype=np.int64)
        rc = self._lib.mfh_encode_records(
            self._h, KIND_CODE[kind], n, blob, native.ptr(offsets, C.c_int64), int(max_len),
            int(n_threads), native.ptr(ids, C.c_int32), cap, native.ptr(seq_off, C.c_int64))
        if rc == 2:
            need = 3 if kind is Kind.BLEURT else 2
            what = "BOS, SEP and EOS" if kind is Kind.BLEURT else "BOS and EOS"
            raise ValueError(f"max_len {max_len} cannot hold {what}" if max_len < need else
                             "tokenizer failed")
        if rc != 0:
            raise RuntimeError(f"mfh_encode_records failed ({rc})")
        return ids[:int(seq_off[-1])], seq_off


    def encode_tsv(self, kind: Kind, lines, max_len: int, n_threads: int = 0, first_index: int = 0):
        """records_from_tsv_lines + field_values + encode_batch for a list of str
        lines in one native call (`evaluate.py:117-123`). Raises
        ColumnCountError(first_index + i, ...) for the first bad line. Returns
        (ids int32[total], seq_off int64[n * n_seqs + 1]) record-major."""
        from .errors import ColumnCountError
        from .kinds import FIELDS_REQUIRED
        kind = Kind.parse(kind)
        n = len(lines)
        blob, line_off = lines_blob(lines)
        ns = N_SEQUENCES[kind]
        cap = 2 * len(blob) + 4 * ns * n + 8
        ids = np.empty(cap, dtype=np.int32)
        seq_off = np.zeros(n * ns + 1, dtype=np.int64)
        bad_line, bad_cols = C.c_int64(-1), C.c_int32(0)
        rc = self._lib.mfh_encode_tsv(
            self._h, KIND_CODE[kind], blob, native.ptr(line_off, C.c_int64), n, int(max_len),
            int(n_threads), native.ptr(ids, C.c_int32), cap, native.ptr(seq_off, C.c_int64),
            C.byref(bad_line), C.byref(bad_cols))
        if rc == 3:
            raise ColumnCountError(first_index + bad_line.value, len(FIELDS_REQUIRED[kind]),
                                   bad_cols.value)
        if rc == 2:
            need = 3 if kind is Kind.BLEURT else 2
            what = "BOS, SEP and EOS" if kind is Kind.BLEURT else "BOS and EOS"
            raise ValueError(f"max_len {max_len} cannot hold {what}" if max_len < need else
                             "tokenizer failed")
        if rc != 0:
            raise RuntimeError(f"mfh_encode_tsv failed ({rc})")
        return ids[:int(seq_off[-1])], seq_off


def lines_blob(lines):
    """UTF-8 bytes of str lines back to back + their byte offsets [n + 1]."""
    n = len(lines)
    off = np.zeros(n + 1, dtype=np.int64)
    text = "".join(lines)
    blob = _utf8(text)
    if len(blob) == len(text):  # ASCII: byte lengths = str lengths
        np.cumsum(np.fromiter(map(len, lines), dtype=np.int64, count=n), out=off[1:])
    else:
        np.cumsum(np.fromiter((len(_utf8(l)) for l in lines), dtype=np.int64, count=n),
                  out=off[1:])
    return blob, off


def load_vocab(path) -> Vocabulary:
    with open(path, "r", encoding="utf-8") as f:  # universal newlines, like the reference
        text = f.read()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise VocabularyError(f"{path}: empty vocabulary file")
    return Vocabulary(lines)


@dataclass
class TokenSequence:
    ids: list = field(default_factory=list)

    def __len__(self):
        return len(self.ids)


def encode_fields(vocab: Vocabulary, record, like, max_len: int) -> list:
    """Sequences of one record in the kind's field order (`vocab.py:132-143`)."""
    like = Kind.parse(like)
    values = record.field_values(like)
    ids, off = vocab.encode_batch(like, [values], max_len, n_threads=1)
    return [TokenSequence(ids[off[i]:off[i + 1]].tolist()) for i in range(len(off) - 1)]
