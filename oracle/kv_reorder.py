"""KV-cache reorder after a beam step -- TEST INFRASTRUCTURE ONLY.

PAPER.md L333 (section 5.1, Fig. 6): the unshared per-beam cache "updates block contents based on
beam indices" after each selection, in place, "first perform[ing] all upward writes in downward
order" (the two-pass scheme). SPEC.md S:L70-87 fixes the operations:

  gather(rows, src)             the plain definition, out of place: new row b = old row src[b].
  plan_reorder(src)             S:L70-78: stable sort of the caller's source indices (non-decreasing),
                                the permutation mapping caller order to plan order, and
                                dir[b] = sign(src_sorted[b] - b).
  apply_reorder_in_place(rows, plan)
                                S:L79-87: one buffer, pass 1 performs every dir = +1 write in
                                ascending destination order, pass 2 every dir = -1 write in
                                descending destination order, dir = 0 rows untouched; a
                                non-monotone src is rejected.

Rows are numpy arrays indexed by beam on axis 0. Writes are counted so the identity plan can be
checked to perform none.
"""
import numpy as np


class ReorderError(ValueError):
    pass


def gather(rows: np.ndarray, src) -> np.ndarray:
    """Out-of-place gather oracle: out[b] = rows[src[b]]."""
    src = np.asarray(src, dtype=np.int64)
    if src.ndim != 1 or src.shape[0] != rows.shape[0]:
        raise ReorderError("src must be [BW]")
    if np.any(src < 0) or np.any(src >= rows.shape[0]):
        raise ReorderError("source index out of range")
    return rows[src].copy()


def plan_reorder(src):
    """S:L70-78. Returns (src_sorted, permutation, dir): src_sorted = src stably sorted
    non-decreasing; permutation[i] = the caller index placed at plan position i (callers apply
    it to scores/tokens too); dir[b] = sign(src_sorted[b] - b)."""
    src = np.asarray(src, dtype=np.int64)
    bw = src.shape[0]
    if np.any(src < 0) or np.any(src >= bw):
        raise ReorderError("source index out of range")
    perm = np.argsort(src, kind="stable")
    s = src[perm]
    d = np.sign(s - np.arange(bw))
    return s, perm, d


def apply_reorder_in_place(rows: np.ndarray, src_sorted, dir_=None) -> int:
    """S:L79-87 on `rows` (modified in place). Returns the number of row writes."""
    s = np.asarray(src_sorted, dtype=np.int64)
    bw = s.shape[0]
    if np.any(np.diff(s) < 0):
        raise ReorderError("non-monotone src: hazard not provably avoided")
    d = np.sign(s - np.arange(bw)) if dir_ is None else np.asarray(dir_)
    writes = 0
    for b in range(bw):                 # pass 1: upward reads (src > b), ascending destinations
        if d[b] > 0:
            rows[b] = rows[s[b]]
            writes += 1
    for b in range(bw - 1, -1, -1):     # pass 2: downward reads (src < b), descending destinations
        if d[b] < 0:
            rows[b] = rows[s[b]]
            writes += 1
    return writes
