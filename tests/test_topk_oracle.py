"""Pins of the per-beam Top-K variant (section 2.2.2: per-beam
Top-K, then the global Top-BW of the BW x K pool) in the oracle: SPEC's worked
examples, the K = 1 closed form, the K >= BW equivalence (reading R3), and the paper's heap fed
per-beam Top-K lists (oracle/paper_heap.py) on tie-heavy random cases. No GPU."""
import math

import numpy as np
import pytest

from oracle import paper_heap
from oracle import xbeam_oracle as O


def test_spec_per_beam_topk_examples():
    # K = 1 on a row with a unique max -> that token
    c = np.array([0.1, 0.7, 0.3]); flat = np.arange(3); b = np.zeros(3, np.int64)
    assert O.per_beam_topk(c, flat, b, 1).tolist() == [1]
    # row [5, 5, 1], K = 2 -> tokens (0, 1) in that order (ties to the lower token)
    row = np.array([5.0, 5.0, 1.0])
    logp = row - math.log(sum(math.exp(x) for x in row))
    keep = O.per_beam_topk(logp, np.arange(3), np.zeros(3, np.int64), 2)
    assert keep.tolist() == [0, 1]
    sel = O.select_top_bw(logp[keep], keep, 2)
    assert keep[sel].tolist() == [0, 1]


def test_spec_select_two_beams_example():
    # two beams, lists [(9), (7)] and [(8), (1)], BW = 2 -> scores {9, 8}
    rows = [(9.0, [(9.0, 0), (7.0, 1)]), (8.0, [(8.0, 0), (1.0, 1)])]
    got, _ = paper_heap.heap_select(rows, 2, 2)
    assert sorted(s for s, _ in got) == [8.0, 9.0]
    c = np.array([9.0, 7.0, 8.0, 1.0]); flat = np.array([0, 1, 2, 3]); b = np.array([0, 0, 1, 1])
    for k in (1, 2):
        keep = O.per_beam_topk(c, flat, b, k)
        assert sorted(c[keep][O.select_top_bw(c[keep], flat[keep], 2)].tolist()) == [8.0, 9.0]


def _rand_case(rng, quant):
    vocab = int(rng.choice([4, 8, 16, 32]))
    nd = int(rng.choice([2, 3]))
    items = rng.integers(0, vocab, size=(int(rng.integers(1, 150)), nd))
    voc = O.Vocabulary(items, vocab, nd)
    n = int(rng.integers(1, 20))
    pref = []
    for _ in range(n):
        d = int(rng.integers(0, nd))
        pref.append(voc.tuple_of(int(rng.integers(0, voc.n_items)))[:d])
    s = -np.sort(rng.exponential(2.0, size=n)) if not quant else -np.sort(rng.integers(0, 4, size=n).astype(float))
    st = O.BeamState(prefixes=pref, scores=np.sort(s)[::-1].astype(np.float64))
    logits = rng.standard_normal((n, vocab))
    if quant:
        logits = np.round(logits * 2) / 2
    return voc, st, logits.astype(np.float32)


def test_k1_closed_form():
    """K = 1: each beam contributes its best candidate (max logit, lowest token on ties); the step
    keeps the best BW of those by (score desc, beam asc)."""
    rng = np.random.default_rng(11)
    for case in range(200):
        voc, st, logits = _rand_case(rng, case % 2 == 0)
        bw = int(rng.choice([1, 2, 4, 8]))
        best = []
        for bb in range(st.n_live):
            legal = voc.children(st.prefixes[bb])
            xs = [float(logits[bb][t]) for t in legal]
            j = max(range(len(legal)), key=lambda i: (xs[i], -int(legal[i])))
            m = max(xs)
            lse = m + math.log(sum(math.exp(x - m) for x in xs))
            best.append((st.scores[bb] + (xs[j] - lse), bb, int(legal[j])))
        best.sort(key=lambda t: (-t[0], t[1]))
        want = [(bb, v) for _, bb, v in best[:bw]]
        nxt = O.beam_step(voc, st, logits, bw, top_k=1)
        assert list(zip(nxt.parents.tolist(), nxt.tokens.tolist())) == want, case


def test_k_ge_bw_is_the_plain_definition():
    rng = np.random.default_rng(12)
    for case in range(150):
        voc, st, logits = _rand_case(rng, case % 3 == 0)
        bw = int(rng.choice([1, 2, 4, 8, 32]))
        a = O.beam_step(voc, st, logits, bw)
        for k in (bw, bw + 3):
            b = O.beam_step(voc, st, logits, bw, top_k=k)
            assert a.parents.tolist() == b.parents.tolist() and a.tokens.tolist() == b.tokens.tolist()


@pytest.mark.parametrize("k", [1, 2, 3, 8])
def test_paper_heap_with_topk_lists_equals_oracle(k):
    rng = np.random.default_rng(100 + k)
    for case in range(150):
        voc, st, logits = _rand_case(rng, case % 2 == 0)
        bw = int(rng.choice([1, 2, 4, 8, 32]))
        c, flat, b, v, _ = O.step_candidates(voc, st, logits)
        rows = [(st.scores[bb], list(zip(c[b == bb].tolist(), v[b == bb].tolist()))) for bb in range(st.n_live)]
        got, _ = paper_heap.heap_select(rows, bw, voc.vocab, top_k=k)
        nxt = O.beam_step(voc, st, logits, bw, top_k=k)
        assert [f for _, f in got] == (nxt.parents * voc.vocab + nxt.tokens).tolist(), case
        assert [s for s, _ in got] == nxt.scores.tolist()
