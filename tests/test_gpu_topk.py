"""Per-beam Top-K with K < BW (each beam's Top-K, then the
global Top-BW of that pool) through the CUDA path against the oracle's beam_step(top_k=K) (pinned
in tests/test_topk_oracle.py). Sparse and dense routes, the survivor-overflow fallback, K = 1."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import xbeam_oracle as O  # noqa: E402
from synth import config, make_items, make_logits  # noqa: E402
from tests.parity import compare_step  # noqa: E402


@pytest.fixture(scope="module")
def xgr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11529_b200 as xgr
    return xgr


def _check(xgr, items, vocab, nd, bw, batch, k, flags=0, sigma=2.0, seed=0, check=None, quant=False):
    voc = O.Vocabulary(items, vocab, nd)
    bs = xgr.BeamSearch(vocab, nd, bw, batch, flags=flags, top_k=k)
    bs.mask_build(items)
    check = list(range(batch)) if check is None else check
    hist_p, hist_t = [], []
    sc = nl = None
    for t in range(nd):
        x = make_logits((batch, 1 if t == 0 else bw, vocab), 700 + 10 * seed + t, sigma)
        if quant:
            x = np.round(x * 2) / 2
        if t == 0:
            states = {r: O.BeamState.root() for r in check}
        else:
            states = {r: O.state_from_history([h[r] for h in hist_p], [h[r] for h in hist_t], sc[r], nl[r])
                      for r in check}
        bs.step(torch.from_numpy(x).cuda())
        v = bs.view()
        par, tok = v["parent"].cpu().numpy().copy(), v["token"].cpu().numpy().copy()
        sc, nl = v["score"].cpu().numpy().copy(), v["n_live"].cpu().numpy().copy()
        for r in check:
            ref = O.beam_step(voc, states[r], x[r], bw, top_k=k)
            assert int(nl[r]) == ref.n_live, (r, t)
            compare_step(voc, states[r], x[r], bw, par[r], tok[r], sc[r], nl[r], where=f"topk{k} req {r} step {t + 1}",
                         top_k=k)
        hist_p.append(par)
        hist_t.append(tok)
    out = bs.finalize(on_device=False)
    return out, bs


@pytest.mark.parametrize("k", [1, 2, 7, 32])
@pytest.mark.parametrize("flags", [0, 4])
def test_topk_random_trie(xgr, k, flags):
    """V = 1024 (dense steps stream, or every step sparse with flags 0 on small tries)."""
    rng = np.random.default_rng(50 + k)
    vocab, nd, bw, batch = 1024, 3, 64, 3
    items = rng.integers(0, vocab, size=(100000, nd)).astype(np.int32)
    _check(xgr, items, vocab, nd, bw, batch, k, flags=flags, seed=k)


@pytest.mark.parametrize("k", [1, 16, 100])
def test_topk_c2_dense_step(xgr, k):
    """C2 trie (V = 8192, BW = 128): step 2 streams 128 dense rows, step 3 is sparse."""
    c = config("C2")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    _check(xgr, items, c["vocab"], c["nd"], c["beam_width"], 4, k, flags=2, seed=k, check=[0, 3])


@pytest.mark.parametrize("k", [1, 3])
def test_topk_ties_and_odd_vocab(xgr, k):
    """Quantised logits (exact ties) and V % 128 != 0 (the legacy dense route, no theta)."""
    rng = np.random.default_rng(9)
    vocab, nd, bw, batch = 100, 3, 32, 2
    items = rng.integers(0, vocab, size=(20000, nd)).astype(np.int32)
    _check(xgr, items, vocab, nd, bw, batch, k, flags=4, quant=True, seed=3)


def test_topk_overflow_fallback(xgr):
    """A tiny survivor buffer forces the exact multi-pass fallback with per-beam truncation."""
    rng = np.random.default_rng(10)
    vocab, nd, bw, batch = 2048, 2, 128, 2
    items = rng.integers(0, vocab, size=(150000, nd)).astype(np.int32)
    voc = O.Vocabulary(items, vocab, nd)
    for k in (1, 5, 64):
        bs = xgr.BeamSearch(vocab, nd, bw, batch, flags=4 | 2, top_k=k, survivor_cap=bw)
        bs.mask_build(items)
        xs = [make_logits((batch, 1 if t == 0 else bw, vocab), 900 + t, 2.0) for t in range(nd)]
        states = [O.BeamState.root() for _ in range(batch)]
        for t in range(nd):
            bs.step(torch.from_numpy(xs[t]).cuda())
            v = bs.view()
            for r in range(batch):
                compare_step(voc, states[r], xs[t][r], bw, v["parent"][r].cpu().numpy(), v["token"][r].cpu().numpy(),
                             v["score"][r].cpu().numpy(), int(v["n_live"][r]), where=f"ovf k{k} r{r} t{t}", top_k=k)
                states[r] = O.beam_step(voc, states[r], xs[t][r], bw, top_k=k)
        assert bs.counters()["overflow"] > 0
        bs.finalize(on_device=True)


@pytest.mark.parametrize("k", [1, 50])
def test_topk_v16384_many_rows_per_cta(xgr, k):
    """V = 16384 with per-beam Top-K (the histogram seed + 512-thread streaming kernel) and far more
    rows than CTAs (8 x 512 rows on 148 SMs), peaky logits so skipped and streamed rows interleave."""
    vocab, nd, bw, batch = 16384, 3, 512, 8
    items = make_items(20_000_000, vocab, nd, 161616)
    _check(xgr, items, vocab, nd, bw, batch, k, flags=2, sigma=4.0, seed=k, check=[0, 3, 7])
