"""Tokenizer oracle: plain-Python restatement of the reference segmentation.

Follows `pkg/src/metricforge/vocab.py`:
  * vocab file = UTF-8 text, universal-newline read, split on "\\n", one
    trailing empty line dropped (`:82-90`); ids = line numbers; the first
    five lines are the specials (`:39-42`); specials never match text (`:45`).
  * encode (`:54-79`): `str.split()` words, stream = "▁" + "▁".join(words),
    greedy longest match at each code point (piece lengths capped by the
    longest non-special piece), unmatched code point -> UNK (id 1).
  * sequence assembly (`:104-143`): [BOS x EOS] per field with right
    truncation keeping EOS; BLEURT joint [BOS T SEP R EOS] trimming the
    longer side first, ties trim R.
"""

from __future__ import annotations

PAD, UNK, BOS, EOS, SEP = 0, 1, 2, 3, 4
MARKER = "▁"


def read_vocab_file(path):
    with open(path, "r", encoding="utf-8") as f:
        text = f.read()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    return lines


class OracleVocab:
    def __init__(self, tokens):
        self.tokens = list(tokens)
        self.pieces = {t: i for i, t in enumerate(self.tokens) if i >= 5}
        self.max_piece = max((len(t) for t in self.pieces), default=0)

    def encode(self, text):
        words = text.split()
        if not words:
            return []
        s = MARKER + MARKER.join(words)
        out, i = [], 0
        while i < len(s):
            hit = None
            for n in range(min(self.max_piece, len(s) - i), 0, -1):
                pid = self.pieces.get(s[i:i + n])
                if pid is not None:
                    hit = (pid, n)
                    break
            if hit is None:
                out.append(UNK)
                i += 1
            else:
                out.append(hit[0])
                i += hit[1]
        return out


def single(vocab, text, max_len):
    ids = [BOS] + vocab.encode(text) + [EOS]
    if len(ids) > max_len:
        if max_len < 2:
            raise ValueError("max_len cannot hold BOS and EOS")
        ids = ids[:max_len - 1] + [EOS]
    return ids


def joint(vocab, first, second, max_len):
    if max_len < 3:
        raise ValueError("max_len cannot hold BOS, SEP and EOS")
    a, b = vocab.encode(first), vocab.encode(second)
    budget = max_len - 3
    if len(a) + len(b) > budget:
        # closed form of "pop from the longer, ties pop the second"
        keep_a = min(len(a), max(-(-budget // 2), budget - len(b)))
        a, b = a[:keep_a], b[:budget - keep_a]
    return [BOS] + a + [SEP] + b + [EOS]


def encode_record(vocab, kind, fields, max_len):
    """fields: the kind's field strings in (S, T, R) order."""
    if kind == "bleurt":
        return [joint(vocab, fields[0], fields[1], max_len)]
    return [single(vocab, v, max_len) for v in fields]
