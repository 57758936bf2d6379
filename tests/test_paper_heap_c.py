"""The paper's heap selection in C (oracle/paper_heap.c: PAPER.md L385 min-heap with per-beam early
termination, fp32, threaded over requests) against the fp64 plain definition (oracle/xbeam_oracle.py)
under the same adjudicated parity rules as the GPU path (tests/parity.py), teacher forced from its
own states. It is bench.py's cpu_baseline.paper_heap, so it must compute the same thing. Not gpu."""
import numpy as np
import pytest

from oracle import xbeam_oracle as O
from synth import config, make_items, make_logits
from tests.parity import compare_step

paper_heap_c = pytest.importorskip("oracle.paper_heap_c", exc_type=OSError)


def _run(items, vocab, nd, bw, batch, sigma, seed, top_k=0, threads=3, quant=False):
    voc = O.Vocabulary(items, vocab, nd)
    ph = paper_heap_c.PaperHeap(voc.keys, vocab, nd)
    lg = []
    for r in range(batch):
        steps = []
        for t in range(nd):
            x = make_logits((1 if t == 0 else bw, vocab), seed + 31 * r + t, sigma)
            if quant:
                x = np.round(x * 2) / 2
            steps.append(x.astype(np.float32))
        lg.append(steps)
    out = ph.run(lg, bw, threads=threads, top_k=top_k)
    res = {"strict": 0, "adjudicated": 0}
    for r in range(batch):
        state = O.BeamState.root()
        hp, ht = [], []
        for t in range(nd):
            par, tok, sc, nl = out["parent"][r, t], out["token"][r, t], out["score"][r, t], out["n_live"][r, t]
            res[compare_step(voc, state, lg[r][t], bw, par, tok, sc, nl, where=f"C heap r{r} t{t + 1}",
                             top_k=top_k or None)] += 1
            hp.append(par)
            ht.append(tok)
            state = O.state_from_history(hp, ht, sc, nl)
    return out, res


@pytest.mark.parametrize("case", [(16, 3, 300, 4, 4), (64, 3, 3000, 32, 3), (1000, 3, 50000, 64, 2),
                                  (256, 2, 20000, 128, 2), (8, 4, 2000, 8, 5), (3, 3, 20, 5, 2)])
def test_c_paper_heap_random_tries(case):
    vocab, nd, n, bw, batch = case
    rng = np.random.default_rng(vocab + nd)
    items = rng.integers(0, vocab, size=(n, nd)).astype(np.int32)
    out, res = _run(items, vocab, nd, bw, batch, 3.0, 11)
    assert out["visits"] <= out["cands"]


def test_c_paper_heap_ties_and_topk():
    rng = np.random.default_rng(4)
    items = rng.integers(0, 512, size=(30000, 3)).astype(np.int32)
    _run(items, 512, 3, 32, 3, 2.0, 5, quant=True)
    for k in (1, 5):
        _run(items, 512, 3, 32, 3, 2.0, 7, top_k=k)


def test_c_paper_heap_c1_exhaustive_and_early_termination():
    c = config("C1")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    out, _ = _run(items, c["vocab"], c["nd"], 256, 1, 2.0, 3)
    assert out["n_live"][0, -1] == 200                  # BW >= items: every item comes back
    out, _ = _run(items, c["vocab"], c["nd"], 4, 4, 2.0, 9)
    assert out["visits"] < out["cands"]                # the heap terminated beams early
