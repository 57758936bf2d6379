"""Plain fp64 CPU definition of one xBeam decode step and of a whole ND-step beam search.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

What is computed, and where the paper says so (PAPER.md line numbers, /root/reference/PAPER.md):

* Valid-item vocabulary (L361 section 6.1 "pre-built valid item vocabulary"; L309 section 5 "the
  resulting TID triplet represents an item ID"): the item tuples are sorted lexicographically and
  de-duplicated; item_rank(tuple) = its index in that list (reading R9/R10).
  children(prefix) = sorted distinct next tokens of the items extending `prefix`.
* Valid path constraint (L361: "incorporates the mask into the model's output logits through
  element-wise addition. Once the masked logits are processed by the Softmax function, the
  probabilities of invalid token IDs become vanishingly small"): read as the -inf limit of the
  additive mask (reading R1/R2): the log-softmax of row b is taken over its legal tokens L_b only
      m = max_{v in L_b} x_v,  Z = sum_{v in L_b} exp(x_v - m),  lse = m + ln Z,
      logp_v = x_v - lse.
* Log-prob accumulation (L376 section 6.2 "beam search accumulates log-probabilities (log_prob)
  rather than multiplying raw probabilities"): candidate score c_{b,v} = S_b + logp_v.
* Selection (L154-156 section 2.2.2; L356 section 6): each beam keeps its Top-K, then the global
  Top-BW of the BW x K pool by cumulative log-probability. With K >= BW (reading R3) per-beam
  truncation cannot drop a global Top-BW member, so the step's result is exactly: the first
  min(BW, total) legal candidates under (c descending, flat = b*V + v ascending) (reading R4
  tie-break, R5 slot order, R7 under-full pool).
* Beam state (L392 section 6.3: BW fixed, structures reused): slot j of the next step holds
  parent b_j, token v_j, score c_j, prefix prefix_{b_j} + (v_j,).

Arithmetic is fp64 on the exactly widened fp32 logits (reading R11). No blocking, fusion,
pruning or reordering: every legal candidate is materialised and fully sorted.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class OracleInputError(ValueError):
    """Bad vocabulary input. `.kind` is 'TOKEN_RANGE', 'EMPTY_VOCAB' or 'INVALID_ARG'."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


class Vocabulary:
    """Sorted, de-duplicated list of legal ND-tuples with prefix queries.

    Tuples are packed into uint64 keys with w = ceil(log2 V) bits per token, most significant
    token first, so numeric key order is lexicographic tuple order. Requires w * ND <= 64.
    """

    def __init__(self, items, vocab: int, nd: int):
        if vocab < 1 or nd < 1:
            raise OracleInputError("INVALID_ARG", "vocab and nd must be >= 1")
        items = np.asarray(items)
        if items.size == 0:
            raise OracleInputError("EMPTY_VOCAB", "no legal items: no beam could live")
        if items.ndim != 2 or items.shape[1] != nd:
            raise OracleInputError("INVALID_ARG", f"items must be [N][{nd}]")
        if items.min() < 0 or items.max() >= vocab:
            raise OracleInputError("TOKEN_RANGE", "token outside [0, V)")
        self.vocab = int(vocab)
        self.nd = int(nd)
        self.w = max(1, int(vocab - 1).bit_length())
        if self.w * nd > 64:
            raise OracleInputError("INVALID_ARG", "nd * ceil(log2 V) > 64 bits")
        key = np.zeros(items.shape[0], dtype=np.uint64)
        for d in range(nd):
            key |= items[:, d].astype(np.uint64) << np.uint64(self.w * (nd - 1 - d))
        key = np.sort(key)
        keep = np.ones(key.shape[0], dtype=bool)
        keep[1:] = key[1:] != key[:-1]
        self.keys = key[keep]                      # sorted unique item keys
        self._children_cache: dict = {}

    # --- item list -------------------------------------------------------------------------
    @property
    def n_items(self) -> int:
        return int(self.keys.shape[0])

    def _pack(self, tup) -> int:
        k = 0
        for t in tup:
            k = (k << self.w) | int(t)
        return k

    def tuple_of(self, rank: int) -> tuple:
        k = int(self.keys[rank])
        return tuple((k >> (self.w * (self.nd - 1 - d))) & ((1 << self.w) - 1)
                     for d in range(self.nd))

    def item_rank(self, tup) -> int:
        """Index of `tup` in the sorted de-duplicated legal list, or -1 if not legal."""
        if len(tup) != self.nd or any(int(t) < 0 or int(t) >= self.vocab for t in tup):
            return -1
        k = np.uint64(self._pack(tup))
        i = int(np.searchsorted(self.keys, k))
        return i if i < self.n_items and self.keys[i] == k else -1

    def contains(self, tup) -> bool:
        return self.item_rank(tup) >= 0

    # --- prefix queries --------------------------------------------------------------------
    def _range(self, prefix):
        d = len(prefix)
        s = self.w * (self.nd - d)
        if d == 0:
            return 0, self.n_items
        p = self._pack(prefix)
        lo = int(np.searchsorted(self.keys, np.uint64(p << s), side="left"))
        hi = int(np.searchsorted(self.keys, np.uint64(((p + 1) << s) - 1), side="right"))
        return lo, hi

    def children(self, prefix) -> np.ndarray:
        """Sorted distinct tokens t with prefix + (t,) a prefix of some legal item (int64)."""
        prefix = tuple(int(t) for t in prefix)
        hit = self._children_cache.get(prefix)
        if hit is not None:
            return hit
        d = len(prefix)
        if d >= self.nd:
            raise OracleInputError("INVALID_ARG", "prefix already complete")
        lo, hi = self._range(prefix)
        tok = (self.keys[lo:hi] >> np.uint64(self.w * (self.nd - d - 1))) & np.uint64((1 << self.w) - 1)
        if tok.shape[0]:
            keep = np.ones(tok.shape[0], dtype=bool)
            keep[1:] = tok[1:] != tok[:-1]        # the slice is sorted, so tokens are sorted
            tok = tok[keep]
        out = tok.astype(np.int64)
        self._children_cache[prefix] = out
        return out

    def n_nodes(self, level: int) -> int:
        """Number of distinct prefixes of length `level` (level 0: the root)."""
        if level == 0:
            return 1
        p = self.keys >> np.uint64(self.w * (self.nd - level))
        return int(1 + np.count_nonzero(p[1:] != p[:-1]))


# --- one row: legal-only log-softmax ----------------------------------
def log_softmax_legal(row, legal):
    """fp64 log-probabilities of the legal tokens of one fp32 logit row.

    Returns (logp[len(legal)], m, Z, lse, finite) where finite is False if a legal logit is NaN or
    +inf, or every legal logit is -inf (reading R12; -inf alone is a legal zero-probability token).
    """
    x = np.asarray(row)[np.asarray(legal, dtype=np.int64)].astype(np.float64)
    m = float(np.max(x))
    with np.errstate(invalid="ignore", over="ignore"):
        e = np.exp(x - m)
        Z = float(np.sum(e))
        lse = m + math.log(Z) if (Z > 0 and math.isfinite(Z)) else float("nan")
        logp = x - lse
    finite = bool(math.isfinite(lse)) and not bool(np.isnan(x).any()) and not bool(np.isposinf(x).any())
    return logp, m, Z, lse, finite


def select_top_bw(c, flat, bw: int) -> np.ndarray:
    """Indices of the first min(bw, n) candidates under (c desc, flat asc). Full sort."""
    c = np.asarray(c, dtype=np.float64)
    flat = np.asarray(flat, dtype=np.int64)
    order = np.lexsort((flat, -c))
    return order[: min(bw, c.shape[0])]


# --- beam state and one step ------------------------------------------------------------------
@dataclass
class BeamState:
    """One request's live beams after some step (slot order = selection order)."""
    prefixes: list                         # list of tuples, len n_live
    scores: np.ndarray                     # fp64 [n_live]
    parents: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    tokens: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    nonfinite: bool = False

    @property
    def n_live(self) -> int:
        return len(self.prefixes)

    @staticmethod
    def root() -> "BeamState":
        """Step-1 input: one live beam, the empty prefix, score 0 (reading R6)."""
        return BeamState(prefixes=[()], scores=np.zeros(1, dtype=np.float64))


def step_candidates(vocab: Vocabulary, state: BeamState, logits):
    """All legal candidates of one request's step: (c fp64, flat int64, b, v, nonfinite).

    logits: array [rows][ld] (fp32); row b is slot b's next-token distribution (reading R21).
    """
    V = vocab.vocab
    cs, flats, bs, vs = [], [], [], []
    nonfinite = False
    for b in range(state.n_live):
        legal = vocab.children(state.prefixes[b])     # never empty (reading R8)
        logp, _, _, _, finite = log_softmax_legal(logits[b], legal)
        nonfinite |= not finite
        c = state.scores[b] + logp                     # c = S_b + (x - lse), fp64
        cs.append(c)
        flats.append(b * V + legal)
        bs.append(np.full(legal.shape[0], b, dtype=np.int64))
        vs.append(legal)
    return (np.concatenate(cs), np.concatenate(flats), np.concatenate(bs),
            np.concatenate(vs), nonfinite)


def per_beam_topk(c, flat, b, k: int) -> np.ndarray:
    """Indices of each beam's first min(k, n_b) candidates under (c desc, flat asc) -- within a
    row that is (score desc, token asc) -- the per-beam Top-K of PAPER.md L156 (section 2.2.2,
    "selects the Top-K most likely next-token candidates") and SPEC S:L356-364. Full sort."""
    c = np.asarray(c, dtype=np.float64)
    flat = np.asarray(flat, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    order = np.lexsort((flat, -c, b))            # by beam, then (c desc, flat asc)
    bo = b[order]
    start = np.searchsorted(bo, bo, side="left")  # first index of each element's beam run
    rank = np.arange(order.shape[0]) - start
    return np.sort(order[rank < k])


def beam_step(vocab: Vocabulary, state: BeamState, logits, bw: int, top_k: int | None = None) -> BeamState:
    """One decode step of one request (DESIGN.md readings).
    top_k (NEXT f3): keep each beam's Top-K candidates first, then the global
    Top-BW of that BW x K pool; None or top_k >= BW is the plain definition (reading R3)."""
    c, flat, b, v, nonfinite = step_candidates(vocab, state, logits)
    if top_k is not None and top_k < bw:
        keep = per_beam_topk(c, flat, b, top_k)
        c, flat, b, v = c[keep], flat[keep], b[keep], v[keep]
    sel = select_top_bw(c, flat, bw)
    parents = b[sel]
    tokens = v[sel]
    prefixes = [state.prefixes[int(p)] + (int(t),) for p, t in zip(parents, tokens)]
    return BeamState(prefixes=prefixes, scores=c[sel], parents=parents, tokens=tokens,
                     nonfinite=state.nonfinite or nonfinite)


@dataclass
class FinalItems:
    tokens: np.ndarray       # int64 [BW][ND], -1 for dead slots
    item_rank: np.ndarray    # int64 [BW], -1 for dead slots
    scores: np.ndarray       # fp64 [BW], -inf for dead slots
    n_live: int


def finalize(vocab: Vocabulary, state: BeamState, bw: int) -> FinalItems:
    """Item IDs of the final beams (the TID tuple is the item ID)."""
    tok = np.full((bw, vocab.nd), -1, dtype=np.int64)
    rank = np.full(bw, -1, dtype=np.int64)
    sc = np.full(bw, -np.inf, dtype=np.float64)
    for j, p in enumerate(state.prefixes):
        tok[j, :] = p
        rank[j] = vocab.item_rank(p)
        sc[j] = state.scores[j]
    return FinalItems(tokens=tok, item_rank=rank, scores=sc, n_live=state.n_live)


def run_request(vocab: Vocabulary, logits_per_step, bw: int, top_k: int | None = None):
    """Free-running ND-step beam search of one request. logits_per_step[t] is [rows][ld]
    (row 0 only at t = 0). Returns (FinalItems, [BeamState after each step])."""
    state = BeamState.root()
    states = []
    for t in range(vocab.nd):
        state = beam_step(vocab, state, logits_per_step[t], bw, top_k)
        states.append(state)
    return finalize(vocab, state, bw), states


def state_from_history(parent_hist, token_hist, scores, n_live) -> BeamState:
    """Rebuild a BeamState from per-step parent/token histories (teacher forcing, reading R15).

    parent_hist, token_hist: int arrays [t][BW] of the steps so far; scores: fp32 [BW]."""
    t = len(parent_hist)
    prefixes = []
    for j in range(int(n_live)):
        toks = []
        s = j
        for k in range(t - 1, -1, -1):
            toks.append(int(token_hist[k][s]))
            s = int(parent_hist[k][s])
        prefixes.append(tuple(reversed(toks)))
    return BeamState(prefixes=prefixes,
                     scores=np.asarray(scores[: int(n_live)], dtype=np.float32).astype(np.float64),
                     parents=np.asarray(parent_hist[-1][: int(n_live)], dtype=np.int64) if t else np.zeros(0, np.int64),
                     tokens=np.asarray(token_hist[-1][: int(n_live)], dtype=np.int64) if t else np.zeros(0, np.int64))

