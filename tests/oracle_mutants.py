"""pytest plugin for the oracle mutation check (tests/test_oracle_mutations.py): when the
environment names a mutant (XGR_ORACLE_MUTANT), one plausible mistake is patched into
oracle/xbeam_oracle.py before the pins run. Each mutant must make at least one pin fail, which
shows the pins fix the oracle's arithmetic rather than restate it."""
import math
import os

import numpy as np

from oracle import xbeam_oracle as O


def _tie_break_reversed(c, flat, bw):
    order = np.lexsort((-np.asarray(flat, dtype=np.int64), -np.asarray(c, dtype=np.float64)))
    return order[: min(bw, len(order))]


def _lse_mutant(shift=0.0, full_vocab=False):
    orig = O.log_softmax_legal

    def f(row, legal):
        if full_vocab:   # normalise over every token of the row instead of the legal ones only
            x = np.asarray(row, dtype=np.float64)
            x = x[np.isfinite(x)]
            m = float(np.max(x))
            lse_all = m + math.log(float(np.sum(np.exp(x - m))))
            logp, m2, Z, lse, fin = orig(row, legal)
            return logp + lse - lse_all, m2, Z, lse_all, fin
        logp, m, Z, lse, fin = orig(row, legal)
        return logp - shift, m, Z, lse + shift, fin
    return f


def _dropped_score(vocab, state, logits):
    zero = O.BeamState(prefixes=state.prefixes, scores=np.zeros_like(state.scores))
    return _orig_step_candidates(vocab, zero, logits)


def _negated_logp(vocab, state, logits):
    c, flat, b, v, nf = _orig_step_candidates(vocab, state, logits)
    s = state.scores[b]
    return s - (c - s), flat, b, v, nf


def _wrong_parent(vocab, state, logits, bw, top_k=None):
    new = _orig_beam_step(vocab, state, logits, bw, top_k)
    n = state.n_live
    pref = [state.prefixes[(int(p) + 1) % n] + (int(t),) for p, t in zip(new.parents, new.tokens)]
    return O.BeamState(prefixes=pref, scores=new.scores, parents=new.parents, tokens=new.tokens,
                       nonfinite=new.nonfinite)


def _no_dedup_init(self, items, vocab, nd):
    _orig_vocab_init(self, items, vocab, nd)
    a = np.asarray(items)
    key = np.zeros(a.shape[0], dtype=np.uint64)
    for d in range(nd):
        key |= a[:, d].astype(np.uint64) << np.uint64(self.w * (nd - 1 - d))
    self.keys = np.sort(key)          # duplicates kept


def _range_end_exclusive(self, prefix):
    d = len(prefix)
    if d == 0:
        return 0, self.n_items
    s = self.w * (self.nd - d)
    p = self._pack(prefix)
    lo = int(np.searchsorted(self.keys, np.uint64(p << s), side="left"))
    hi = int(np.searchsorted(self.keys, np.uint64(((p + 1) << s) - 1), side="left"))   # drops the last
    return lo, hi


_orig_step_candidates = O.step_candidates
_orig_beam_step = O.beam_step
_orig_vocab_init = O.Vocabulary.__init__

MUTANTS = {
    "tie_break_reversed": lambda: setattr(O, "select_top_bw", _tie_break_reversed),
    "lse_perturbed": lambda: setattr(O, "log_softmax_legal", _lse_mutant(shift=1e-7)),
    "lse_full_vocab": lambda: setattr(O, "log_softmax_legal", _lse_mutant(full_vocab=True)),
    "score_term_dropped": lambda: setattr(O, "step_candidates", _dropped_score),
    "logp_sign": lambda: setattr(O, "step_candidates", _negated_logp),
    "wrong_parent": lambda: setattr(O, "beam_step", _wrong_parent),
    "no_dedup": lambda: setattr(O.Vocabulary, "__init__", _no_dedup_init),
    "range_end": lambda: setattr(O.Vocabulary, "_range", _range_end_exclusive),
}


def pytest_configure(config):
    name = os.environ.get("XGR_ORACLE_MUTANT")
    if name:
        MUTANTS[name]()
