"""Pure-Python brute force for tiny tries: an independent check of the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Shares no code with oracle/xbeam_oracle.py:
no numpy arithmetic, no packing, no sorting of keys.

* legal set: every tuple of [0, V)^ND is enumerated and kept iff it is in the item set
  ("pre-built valid item vocabulary"; SPEC.md S:L337 hash-set membership oracle).
* children(prefix): every token t of [0, V) is tried, kept iff some legal item starts with
  prefix + (t,).
* log-softmax over the legal tokens with math.exp / math.log loops.
* path score of an item = sum over its ND positions of the legal-only log-softmax of its token
  at its prefix; with BW >= number of items, beam search must return every item with exactly this
  score (SURVEY 8(c.5) "exhaustive case").
"""
from __future__ import annotations

import itertools
import math


def legal_set(items, vocab: int, nd: int):
    s = set(tuple(int(t) for t in it) for it in items)
    return {tup for tup in itertools.product(range(vocab), repeat=nd) if tup in s}


def children(legal, prefix, vocab: int):
    prefix = tuple(prefix)
    d = len(prefix)
    return [t for t in range(vocab)
            if any(it[:d] == prefix and it[d] == t for it in legal)]


def log_softmax_py(values):
    m = max(values)
    z = 0.0
    for x in values:
        z += math.exp(x - m)
    lse = m + math.log(z)
    return [x - lse for x in values]


def path_scores(legal, vocab: int, nd: int, row_fn):
    """{item: score} with row_fn(prefix) -> list of V floats (the logits row at that prefix)."""
    kids = {}
    for it in legal:
        for d in range(nd):
            p = it[:d]
            if p not in kids:
                kids[p] = children(legal, p, vocab)
    logp = {}
    for p, ks in kids.items():
        row = row_fn(p)
        lp = log_softmax_py([float(row[t]) for t in ks])
        for t, l in zip(ks, lp):
            logp[p + (t,)] = l
    out = {}
    for it in legal:
        s = 0.0
        for d in range(nd):
            s += logp[it[: d + 1]]
        out[it] = s
    return out
