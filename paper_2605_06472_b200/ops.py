"""Builders for the tree operation stream (csrc/host/ops.hpp).

The same int64 word stream drives the product's RadixMirror (HostTree) and,
in the tests, the reference CacheTree (oracle/_ref), so both trees can be
compared field by field.
"""
from __future__ import annotations

import struct
from typing import Iterable, List

OP_INSERT, OP_MATCH, OP_TERMINATE, OP_DEMOTE, OP_PROMOTE, OP_DROP, OP_SET_SCORE = 1, 2, 3, 4, 5, 6, 7

_MASK = (1 << 64) - 1


def _tok(t: int) -> int:
    t &= _MASK
    return t - (1 << 64) if t >= (1 << 63) else t


class OpStream:
    def __init__(self):
        self.words: List[int] = []

    def insert(self, tokens: Iterable[int], w: int, agent: int, budget: int = -1) -> "OpStream":
        """CacheTree::insert_suffix (cache.hpp:159)"""
        toks = [_tok(t) for t in tokens]
        self.words += [OP_INSERT, int(w), int(agent), int(budget), len(toks), *toks]
        return self

    def match(self, tokens: Iterable[int], w: int, agent: int) -> "OpStream":
        """CacheTree::match_prefix (cache.hpp:121)"""
        toks = [_tok(t) for t in tokens]
        self.words += [OP_MATCH, int(w), int(agent), len(toks), *toks]
        return self

    def terminate(self, w: int) -> "OpStream":
        self.words += [OP_TERMINATE, int(w)]
        return self

    def demote(self, node: int) -> "OpStream":
        self.words += [OP_DEMOTE, int(node)]
        return self

    def promote(self, node: int) -> "OpStream":
        self.words += [OP_PROMOTE, int(node)]
        return self

    def drop(self, node: int) -> "OpStream":
        self.words += [OP_DROP, int(node)]
        return self

    def set_score(self, node: int, score: float) -> "OpStream":
        bits = struct.unpack("<q", struct.pack("<d", float(score)))[0]
        self.words += [OP_SET_SCORE, int(node), bits]
        return self

    def __len__(self):
        return len(self.words)
