"""Skewed (clustered) semantic-ID tries (synth.make_items_clustered, Zipf s = 1 per level): one
trie level mixes dense nodes (thousands of children) and sparse ones (a handful), so a step needs
both routes. Per request, the previous step's commit decides the route (sparse if the request's
candidates fit on chip); the dense path hands its sparse-parent rows to k_sparse_rows. Parity with
the teacher-forced oracle on every request and step."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import xbeam_oracle as O  # noqa: E402
from synth import config, make_config_items, make_items_clustered, make_logits_torch  # noqa: E402
from tests.test_gpu_parity import run_checked  # noqa: E402


@pytest.fixture(scope="module")
def xgr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11529_b200 as xgr
    return xgr


@pytest.mark.parametrize("vocab,n,bw,batch", [(1024, 1_000_000, 64, 6), (8192, 3_000_000, 128, 4),
                                              (16384, 4_000_000, 256, 3)])
@pytest.mark.parametrize("flags", [2, 2 | 4])
@pytest.mark.parametrize("sigma", [2.0, 4.0])
def test_clustered_trie_parity(xgr, vocab, n, bw, batch, flags, sigma):
    nd = 3
    items = make_items_clustered(n, vocab, nd, 777 + vocab)
    voc = O.Vocabulary(items, vocab, nd)
    bs = xgr.BeamSearch(vocab, nd, bw, batch, flags=flags)
    bs.mask_build(items)
    info = bs.info()
    assert 0 < info["dense"][1] < info["nodes"][1] or 0 < info["dense"][2] < info["nodes"][2], info
    steps = [make_logits_torch((batch, 1 if t == 0 else bw, vocab), 60 + t, sigma) for t in range(nd)]
    bs.counters()
    out, stats = run_checked(bs, voc, steps, bw, list(range(batch)))
    cnt = bs.counters()
    assert stats["adjudicated"] <= 2, stats
    assert cnt["overflow"] == 0 or sigma == 4.0, cnt


@pytest.mark.slow
def test_c3z_full_size_all_requests(xgr):
    """C3 shape on the clustered 100M-item trie: every request at every step."""
    c = config("C3Z")
    items = make_config_items(c)
    voc = O.Vocabulary(items, c["vocab"], c["nd"])
    B, bw = c["batch"], c["beam_width"]
    bs = xgr.BeamSearch(c["vocab"], c["nd"], bw, B, flags=2)
    bs.mask_build(items)
    del items
    steps = [make_logits_torch((B, 1 if t == 0 else bw, c["vocab"]), 11 * t + 1, 2.0) for t in range(c["nd"])]
    bs.counters()
    out, stats = run_checked(bs, voc, steps, bw, list(range(B)))
    assert stats["adjudicated"] <= max(3, (stats["strict"] + stats["adjudicated"]) // 20), stats
    print("C3Z counters", bs.counters())
