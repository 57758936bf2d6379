"""Pins of the CPU oracle to things other than itself (not-gpu).

Each test names what fixes the expected value: a worked example printed in SPEC.md (the paper
prints none for this path), a closed form, brute-force enumeration (oracle/brute.py, pure
Python), the paper's own heap procedure (oracle/paper_heap.py), or an invariant
of the method. A plausible mistake in the oracle (a full-vocabulary LSE instead of legal-only, a
wrong tie-break, a dropped score term, an off-by-one in the trie ranges, a transposed parent and
token) fails at least one of them; see DESIGN.md "Oracle pins".
"""
import math
import random

import numpy as np
import pytest

from oracle import brute, paper_heap
from oracle import xbeam_oracle as O
from synth import config, make_items, prefix_keyed_row


# --- log-softmax ------------------------------------------------------------------------------
def test_spec_log_softmax_examples(golden):
    for ex in golden["log_softmax"]:
        row = np.asarray(ex["row"], dtype=np.float32)
        logp, m, Z, lse, finite = O.log_softmax_legal(row, np.arange(row.shape[0]))
        assert finite
        np.testing.assert_allclose(logp, ex["expect"], rtol=0, atol=ex["atol"], err_msg=ex["cite"])


def test_spec_random_row_sums_to_one():
    """exp-sum of a random row's log-softmax = 1 +- 1e-6."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        row = (rng.standard_normal(4096) * 3).astype(np.float32)
        legal = np.sort(rng.choice(4096, size=rng.integers(1, 4096), replace=False))
        logp, *_ = O.log_softmax_legal(row, legal)
        assert abs(math.fsum(math.exp(v) for v in logp) - 1.0) < 1e-6


def test_legal_only_normalisation_vector(golden):
    """Reading R2: the softmax support is the legal set only. Under a full-vocabulary LSE row 0
    would give -1.8176 instead of -0.0067 for token 0."""
    g = golden["legal_only_vector"]
    for key in ("row0", "row1"):
        row = np.asarray(g[key], dtype=np.float32)
        logp, *_ = O.log_softmax_legal(row, g["legal"])
        assert abs(logp[0] - g["expect_logp_tok0"]) < 1e-15, key


def test_single_legal_child_is_exactly_zero():
    """Closed form: |L_b| = 1 -> Z = 1, ln Z = 0, logp = 0 exactly, whatever the logit."""
    for x in (0.0, -3.25, 17.0, 1e30, -1e-30):
        row = np.full(8, np.nan, dtype=np.float32)
        row[5] = x
        logp, m, Z, lse, finite = O.log_softmax_legal(row, [5])
        assert finite and logp[0] == 0.0 and Z == 1.0


def test_equal_logits_give_minus_ln_n():
    for n in (1, 2, 3, 7, 100):
        row = np.zeros(128, dtype=np.float32)
        logp, *_ = O.log_softmax_legal(row, np.arange(n))
        assert np.all(logp == -math.log(n))


def test_nonfinite_flags():
    row = np.zeros(4, dtype=np.float32)
    row[1] = np.nan
    assert not O.log_softmax_legal(row, [0, 1])[4]
    assert O.log_softmax_legal(row, [0, 2])[4]          # illegal positions may hold anything
    row[1] = np.inf
    assert not O.log_softmax_legal(row, [0, 1])[4]
    row[1] = -np.inf                                     # -inf alone: probability zero, legal
    logp, _, _, _, fin = O.log_softmax_legal(row, [0, 1])
    assert fin and logp[1] == -np.inf and logp[0] == 0.0
    row[:] = -np.inf
    assert not O.log_softmax_legal(row, [0, 1])[4]


# --- vocabulary / trie --------------------------------------------------------------------------
def test_spec_vocab_examples(golden):
    for ex in golden["build_vocab"]:
        voc = O.Vocabulary(np.asarray(ex["items"]), ex["vocab"], ex["nd"])
        for prefix, kids in ex["children"]:
            assert list(voc.children(tuple(prefix))) == kids, ex["cite"]


def test_vocab_errors_and_dedupe():
    with pytest.raises(O.OracleInputError) as e:
        O.Vocabulary(np.zeros((0, 3), np.int32), 8, 3)
    assert e.value.kind == "EMPTY_VOCAB"
    with pytest.raises(O.OracleInputError) as e:
        O.Vocabulary(np.array([[1, 8, 0]]), 8, 3)
    assert e.value.kind == "TOKEN_RANGE"
    with pytest.raises(O.OracleInputError) as e:
        O.Vocabulary(np.array([[1, -1, 0]]), 8, 3)
    assert e.value.kind == "TOKEN_RANGE"
    voc = O.Vocabulary(np.array([[1, 2, 3], [0, 0, 1], [1, 2, 3], [0, 0, 1]]), 8, 3)
    assert voc.n_items == 2
    assert voc.item_rank((0, 0, 1)) == 0 and voc.item_rank((1, 2, 3)) == 1
    assert voc.item_rank((1, 2, 4)) == -1


def test_vocab_membership_hashset():
    """10,000 random tuples, V=256, membership agrees with a hash set on 1,000
    probes."""
    rng = np.random.default_rng(11)
    items = rng.integers(0, 256, size=(10_000, 3))
    hs = set(map(tuple, items.tolist()))
    voc = O.Vocabulary(items, 256, 3)
    assert voc.n_items == len(hs)
    probes = [tuple(items[i]) for i in rng.integers(0, 10_000, 500)]
    probes += [tuple(t) for t in rng.integers(0, 256, size=(500, 3)).tolist()]
    for p in probes:
        assert voc.contains(p) == (tuple(int(t) for t in p) in hs)
    ranked = sorted(hs)
    for j in rng.integers(0, len(ranked), 200):
        assert voc.item_rank(ranked[j]) == j
        assert voc.tuple_of(int(j)) == ranked[j]


@pytest.mark.parametrize("vocab,nd,n", [(16, 3, 200), (8, 4, 300), (5, 3, 60), (16, 2, 256)])
def test_children_vs_bruteforce(vocab, nd, n):
    """Every prefix of every level: oracle children == pure-Python enumeration over all tokens."""
    rng = np.random.default_rng(vocab * 100 + nd)
    items = rng.integers(0, vocab, size=(n, nd))
    voc = O.Vocabulary(items, vocab, nd)
    legal = brute.legal_set(items.tolist(), vocab, nd)
    assert voc.n_items == len(legal)
    for d in range(nd):
        prefixes = {it[:d] for it in legal}
        assert voc.n_nodes(d) == len(prefixes)
        for p in prefixes:
            assert list(voc.children(p)) == brute.children(legal, p, vocab), (d, p)


def test_c1_generator_trie_bruteforce():
    c = config("C1")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    voc = O.Vocabulary(items, c["vocab"], c["nd"])
    legal = brute.legal_set(items.tolist(), c["vocab"], c["nd"])
    assert voc.n_items == len(legal) == 200
    for it in legal:
        for d in range(c["nd"]):
            assert it[d] in voc.children(it[:d])


# --- selection ----------------------------------------------------------------------------------
def test_spec_per_beam_tie(golden):
    g = golden["per_beam_topk"]
    c = np.asarray(g["row"], dtype=np.float64)
    sel = O.select_top_bw(c, np.arange(3), g["k"])
    assert list(sel) == g["expect_tokens"]


def test_spec_select_lists(golden):
    g = golden["select_top_bw"]
    c, flat = [], []
    for b, lst in enumerate(g["lists"]):
        for v, s in enumerate(lst):
            c.append(s)
            flat.append(b * 10 + v)
    sel = O.select_top_bw(c, flat, g["bw"])
    assert [c[i] for i in sel] == g["expect_scores"]
    # BW = 1 is the global argmax
    assert list(O.select_top_bw(c, flat, 1)) == [int(np.argmax(c))]


def test_final_items_single_item(golden):
    g = golden["final_items_single"]
    voc = O.Vocabulary(np.asarray(g["items"]), g["vocab"], g["nd"])
    rng = np.random.default_rng(3)
    logits = [rng.standard_normal((1, g["vocab"])).astype(np.float32) * 5 for _ in range(g["nd"])]
    fin, _ = O.run_request(voc, logits, g["bw"])
    assert list(fin.tokens[0]) == g["expect_tuple"]
    assert fin.scores[0] == g["expect_score"]          # exactly 0: one legal child per step
    assert fin.item_rank[0] == 0 and fin.n_live == 1


def _rand_state(rng, voc, n, quantized):
    # n live beams on random legal prefixes of depth d, sorted scores (some equal)
    d = int(rng.integers(0, voc.nd))
    pref = []
    for _ in range(n):
        it = voc.tuple_of(int(rng.integers(0, voc.n_items)))
        pref.append(it[:d])
    s = -np.sort(rng.exponential(2.0, size=n))[::-1] if not quantized else \
        -np.sort(rng.integers(0, 4, size=n).astype(np.float64))
    s = np.sort(s)[::-1]
    return O.BeamState(prefixes=pref, scores=s.astype(np.float64))


def test_paper_heap_equals_full_sort():
    """PAPER.md L385 heap with early termination == the plain definition (300 cases, half with
    quantised logits and equal beam scores, i.e. full of exact ties)."""
    rng = np.random.default_rng(2024)
    total_visits = total_cands = 0
    for case in range(300):
        vocab = int(rng.choice([4, 8, 16, 32]))
        nd = int(rng.choice([2, 3]))
        items = rng.integers(0, vocab, size=(int(rng.integers(1, 120)), nd))
        voc = O.Vocabulary(items, vocab, nd)
        quant = case % 2 == 0
        st = _rand_state(rng, voc, int(rng.integers(1, 20)), quant)
        bw = int(rng.choice([1, 2, 4, 8, 32]))
        logits = rng.standard_normal((len(st.prefixes), vocab))
        if quant:
            logits = np.round(logits * 2) / 2
        logits = logits.astype(np.float32)
        c, flat, b, v, _ = O.step_candidates(voc, st, logits)
        sel = O.select_top_bw(c, flat, bw)
        rows = []
        for bb in range(st.n_live):
            m = b == bb
            rows.append((st.scores[bb], list(zip(c[m].tolist(), v[m].tolist()))))
        got, stats = paper_heap.heap_select(rows, bw, vocab)
        assert [f for _, f in got] == flat[sel].tolist(), case
        assert [s for s, _ in got] == c[sel].tolist()
        total_visits += stats["visits"]
        total_cands += c.shape[0]
    assert total_visits < total_cands          # early termination did skip candidates


def test_uniform_logits_closed_form():
    """All logits equal (0): logp = -ln|L_b| exactly, so the selection is rows ranked by
    S_b - ln|L_b| (ties: lower b), each row's tokens ascending, truncated at BW. Built here by a
    greedy row-wise construction, not by a global sort."""
    rng = np.random.default_rng(5)
    for case in range(50):
        vocab, nd = 16, 3
        items = rng.integers(0, vocab, size=(int(rng.integers(5, 300)), nd))
        voc = O.Vocabulary(items, vocab, nd)
        st = _rand_state(rng, voc, int(rng.integers(1, 12)), quantized=True)
        bw = int(rng.integers(1, 40))
        logits = np.zeros((st.n_live, vocab), dtype=np.float32)
        new = O.beam_step(voc, st, logits, bw)
        rows = []
        for b, p in enumerate(st.prefixes):
            kids = list(voc.children(p))
            rows.append((st.scores[b] - math.log(len(kids)), b, kids))
        rows.sort(key=lambda r: (-r[0], r[1]))
        exp = []
        for s, b, kids in rows:
            for t in kids:
                if len(exp) < bw:
                    exp.append((b, t, s))
        assert list(zip(new.parents.tolist(), new.tokens.tolist())) == [(b, t) for b, t, _ in exp]
        assert np.all(new.scores == np.array([s for _, _, s in exp]))


def test_exhaustive_case_matches_bruteforce_path_scores():
    """BW >= number of items: nothing is ever dropped, so the final beams are ALL legal items,
    each with the brute-force path score (sum of legal-only log-softmax along its path), in
    non-increasing score order."""
    c = config("C1")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    voc = O.Vocabulary(items, c["vocab"], c["nd"])
    legal = brute.legal_set(items.tolist(), c["vocab"], c["nd"])
    seed, req = 99, 0
    want = brute.path_scores(legal, c["vocab"], c["nd"],
                             lambda p: prefix_keyed_row(seed, req, p, c["vocab"]).tolist())
    state = O.BeamState.root()
    bw = 256
    for t in range(c["nd"]):
        logits = np.stack([prefix_keyed_row(seed, req, p, c["vocab"]) for p in state.prefixes])
        state = O.beam_step(voc, state, logits, bw)
    fin = O.finalize(voc, state, bw)
    assert fin.n_live == len(legal) == 200
    got = {tuple(fin.tokens[j]): fin.scores[j] for j in range(fin.n_live)}
    assert set(got) == legal
    for it, s in want.items():
        assert abs(got[it] - s) < 1e-12
    assert np.all(np.diff(fin.scores[: fin.n_live]) <= 0)
    # brute ranking (by its own scores) agrees wherever scores are separated by > 1e-9
    order = sorted(want, key=lambda it: -want[it])
    pos = {tuple(fin.tokens[j]): j for j in range(fin.n_live)}
    for a, b in zip(order, order[1:]):
        if want[a] - want[b] > 1e-9:
            assert pos[a] < pos[b]
    for j in range(fin.n_live):
        assert fin.item_rank[j] == sorted(legal).index(tuple(fin.tokens[j]))
    assert np.all(fin.item_rank[fin.n_live:] == -1) and np.all(np.isneginf(fin.scores[fin.n_live:]))


def test_multistep_invariants_random():
    """Validity (every output is a legal item), S' <= S_parent, non-increasing slot scores,
    additivity (final score = sum of per-step logp recomputed in pure Python), n_live."""
    rng = random.Random(1)
    for case in range(40):
        vocab = rng.choice([4, 8, 16])
        nd = rng.choice([2, 3, 4])
        n = rng.randint(1, 200)
        items = np.array([[rng.randrange(vocab) for _ in range(nd)] for _ in range(n)])
        voc = O.Vocabulary(items, vocab, nd)
        legal = set(map(tuple, items.tolist()))
        bw = rng.choice([1, 3, 8, 64])
        nrng = np.random.default_rng(case)
        state = O.BeamState.root()
        per_step_logp = []
        for t in range(nd):
            logits = (nrng.standard_normal((max(1, state.n_live), vocab)) * 2).astype(np.float32)
            new = O.beam_step(voc, state, logits, bw)
            assert new.n_live == min(bw, sum(len(voc.children(p)) for p in state.prefixes))
            assert np.all(np.diff(new.scores) <= 0)
            for j in range(new.n_live):
                p = int(new.parents[j])
                assert new.scores[j] <= state.scores[p]
                kids = list(voc.children(state.prefixes[p]))
                lp = brute.log_softmax_py([float(logits[p][k]) for k in kids])
                per_step_logp.append(((t, j), lp[kids.index(int(new.tokens[j]))]))
            state = new
        fin = O.finalize(voc, state, bw)
        for j in range(fin.n_live):
            assert tuple(fin.tokens[j]) in legal
            assert fin.item_rank[j] == sorted(legal).index(tuple(fin.tokens[j]))


def test_step_one_reads_only_row0():
    voc = O.Vocabulary(np.array([[0, 1], [2, 3], [2, 1]]), 4, 2)
    a = np.array([[0.5, 1.0, 2.0, 0.0]], dtype=np.float32)
    b = np.concatenate([a, np.full((3, 4), np.nan, np.float32)])
    s1 = O.beam_step(voc, O.BeamState.root(), a, 2)
    s2 = O.beam_step(voc, O.BeamState.root(), b, 2)
    assert s1.tokens.tolist() == s2.tokens.tolist() == [2, 0]
    assert not s2.nonfinite
