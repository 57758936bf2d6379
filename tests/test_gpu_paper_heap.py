"""The paper's selection procedure on the GPU (XGR_CFG_PAPER_HEAP; per-beam sorted
Top-K lists, then the sequential global min-heap with early termination of PAPER.md L385) is an
exact selection: parity with the teacher-forced fp64 oracle on every request and step, with and
without a per-beam K < BW."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import xbeam_oracle as O  # noqa: E402
from synth import config, make_items, make_logits  # noqa: E402
from tests.parity import compare_step  # noqa: E402

XGR_CFG_PAPER_HEAP = 0x10


@pytest.fixture(scope="module")
def xgr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11529_b200 as xgr
    return xgr


def _run(xgr, items, vocab, nd, bw, batch, k=0, flags=0, sigma=2.0, seed=0):
    voc = O.Vocabulary(items, vocab, nd)
    bs = xgr.BeamSearch(vocab, nd, bw, batch, flags=flags | XGR_CFG_PAPER_HEAP | 2, top_k=k)
    bs.mask_build(items)
    hist_p, hist_t = [], []
    sc = nl = None
    for t in range(nd):
        x = make_logits((batch, 1 if t == 0 else bw, vocab), 500 + seed + t, sigma)
        if t == 0:
            states = [O.BeamState.root() for _ in range(batch)]
        else:
            states = [O.state_from_history([h[r] for h in hist_p], [h[r] for h in hist_t], sc[r], nl[r])
                      for r in range(batch)]
        bs.step(torch.from_numpy(x).cuda())
        v = bs.view()
        par, tok = v["parent"].cpu().numpy().copy(), v["token"].cpu().numpy().copy()
        sc, nl = v["score"].cpu().numpy().copy(), v["n_live"].cpu().numpy().copy()
        for r in range(batch):
            compare_step(voc, states[r], x[r], bw, par[r], tok[r], sc[r], nl[r], where=f"heap r{r} t{t + 1}",
                         top_k=k or None)
        hist_p.append(par)
        hist_t.append(tok)
    cnt = bs.counters()
    bs.finalize(on_device=False)
    return cnt


@pytest.mark.parametrize("case", [(1024, 3, 200000, 64, 3), (8192, 3, 400000, 128, 2), (4096, 2, 200000, 256, 2),
                                  (16384, 2, 100000, 64, 2)])
@pytest.mark.parametrize("flags", [0, 4])
def test_paper_heap_parity(xgr, case, flags):
    vocab, nd, n, bw, batch = case
    rng = np.random.default_rng(vocab + nd + bw)
    items = rng.integers(0, vocab, size=(n, nd)).astype(np.int32)
    _run(xgr, items, vocab, nd, bw, batch, flags=flags, seed=vocab)


@pytest.mark.parametrize("k", [1, 16])
def test_paper_heap_topk_and_c2(xgr, k):
    c = config("C2")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    cnt = _run(xgr, items, c["vocab"], c["nd"], c["beam_width"], 4, k=k, seed=k)
    assert cnt["survivors"] > 0   # heap visits were counted
