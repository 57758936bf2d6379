"""The paper's own selection procedure, as a second independent selection oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md L385 (section 6.2, "Early Sorting Termination"): "xBeam maintains a global min heap of
size BW to store the top-ranking token sequences along with their associated log_prob values.
During sorting, xBeam visits the leaves of each sub-beam tree sequentially. During the traversal
of each beam, if the leaf's log_prob exceeds that of the heap's top element, it is inserted into
the heap, and the heap structure is adjusted to maintain order. Otherwise, the sorting operation
of that beam is terminated immediately. After traversing all beams, xBeam retrieves the top-BW
token sequences."  L376: "the log_prob results for each beam are inherently in descending order".

Followed step by step, in the paper's order:
  1. visit beams b = 0, 1, ... in slot order; within a beam visit its candidates in descending
     log_prob (ties: ascending token, reading R4);
  2. while the heap holds fewer than BW entries, insert;
  3. otherwise insert (replacing the minimum) iff log_prob > heap minimum (strictly, "exceeds"),
     else terminate that beam;
  4. extension from the sorted beam scores: once the heap is full and S_b <= heap
     minimum, no candidate of beam b or any later beam can enter (c <= S_b, and later beams have
     larger flat indices), so stop the outer loop;
  5. retrieve the heap content sorted (c desc, flat asc).
Counts candidate visits and skipped beams.
"""
from __future__ import annotations

import heapq


def heap_select(rows, bw: int, vocab: int, top_k: int | None = None):
    """rows: list over beams b of (S_b, [(c, v), ...]) with candidates in any order.
    top_k: the per-beam Top-K lists the paper feeds the heap:
    only each beam's first top_k candidates in descending order are visited.

    Returns (selected [(c, flat)], stats dict). Heap entries are keyed so the heap top is the
    minimum under the total order (c desc, flat asc): the smallest c, and among equal c the
    largest flat.
    """
    heap = []            # entries (c, -flat)
    visits = 0
    beams_skipped = 0
    for b, (s_b, cands) in enumerate(rows):
        if len(heap) == bw and s_b <= heap[0][0]:
            beams_skipped = len(rows) - b
            break
        ordered = sorted(cands, key=lambda cv: (-cv[0], cv[1]))
        if top_k is not None:
            ordered = ordered[:top_k]
        for c, v in ordered:
            visits += 1
            flat = b * vocab + v
            if len(heap) < bw:
                heapq.heappush(heap, (c, -flat))
            elif c > heap[0][0]:
                heapq.heapreplace(heap, (c, -flat))
            else:
                break
    out = sorted(((c, -nf) for c, nf in heap), key=lambda cf: (-cf[0], cf[1]))
    return out, {"visits": visits, "beams_skipped": beams_skipped}
