"""bf16 logits through xgr_beam_step_ex: the kernels widen every bf16 value
exactly to fp32 and compute as on the fp32 path; the oracle widens the same values (fp64). Same
parity bar as tests/test_gpu_parity.py. bf16 rounding makes exact logit ties common, which the
tie-break (lower flat index) must decide identically on both sides."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import xbeam_oracle as O  # noqa: E402
from synth import config, make_items, make_logits, make_logits_torch  # noqa: E402
from tests.test_gpu_parity import _bs, run_checked  # noqa: E402


@pytest.fixture(scope="module")
def xgr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11529_b200 as xgr
    return xgr


def _bf16(x: np.ndarray):
    return torch.from_numpy(x).cuda().to(torch.bfloat16)


@pytest.mark.parametrize("flags", [0, 1])
def test_c1_bf16(xgr, flags):
    """C1 (V = 16): every step takes the sparse route, which gathers bf16 logits by label (the
    dense route for V % 128 != 0 is fp32 only)."""
    c = config("C1")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    voc = O.Vocabulary(items, c["vocab"], c["nd"])
    for seed in range(4):
        bs = _bs(xgr, voc, c["beam_width"], 3, flags=flags)
        bs.mask_build(items)
        steps = [_bf16(make_logits((3, c["beam_width"], c["vocab"]), 500 + 10 * seed + t, 2.0))
                 for t in range(c["nd"])]
        run_checked(bs, voc, steps, c["beam_width"], [0, 1, 2])


BF16_CASES = [
    # vocab, nd, n_items, bw, batch   (V % 128 == 0: dense steps stream bf16 rows)
    (1024, 3, 50000, 64, 2),
    (4096, 2, 200000, 256, 2),
    (8192, 3, 400000, 128, 2),
    (16384, 2, 100000, 64, 2),
    (128, 3, 20000, 16, 3),
]


@pytest.mark.parametrize("case", BF16_CASES)
@pytest.mark.parametrize("flags", [0, 4, 5])
def test_random_tries_bf16(xgr, case, flags):
    vocab, nd, n, bw, batch = case
    rng = np.random.default_rng(vocab * 11 + nd + bw)
    items = rng.integers(0, vocab, size=(n, nd)).astype(np.int32)
    voc = O.Vocabulary(items, vocab, nd)
    bs = _bs(xgr, voc, bw, batch, flags=flags)
    bs.mask_build(items)
    ld = vocab + 8   # padded rows (ld % 8 == 0) exercise ld > V
    steps = []
    for t in range(nd):
        x = np.full((batch, bw, ld), np.nan, np.float32)
        x[:, :, :vocab] = make_logits((batch, bw, vocab), 2000 + t, 3.0)
        steps.append(_bf16(x))
    run_checked(bs, voc, steps, bw, list(range(batch)))


def test_bf16_pruning_never_changes_results(xgr):
    rng = np.random.default_rng(5)
    vocab, nd, n, bw, batch = 8192, 3, 300000, 64, 3
    items = rng.integers(0, vocab, size=(n, nd)).astype(np.int32)
    steps = [_bf16(make_logits((batch, bw, vocab), 60 + t, 2.0)) for t in range(nd)]
    outs = []
    for flags in (4 | 2, 4 | 1):
        bs = xgr.BeamSearch(vocab, nd, bw, batch, flags=flags)
        bs.mask_build(items)
        for lg in steps:
            bs.step(lg)
        outs.append(bs.finalize(on_device=False))
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_bf16_equals_fp32_of_the_same_values(xgr):
    """bf16 input == the fp32 path fed the same values widened: identical selections."""
    rng = np.random.default_rng(8)
    vocab, nd, n, bw, batch = 4096, 3, 200000, 128, 3
    items = rng.integers(0, vocab, size=(n, nd)).astype(np.int32)
    steps = [_bf16(make_logits((batch, bw, vocab), 80 + t, 2.0)) for t in range(nd)]
    outs = []
    for widen in (False, True):
        bs = xgr.BeamSearch(vocab, nd, bw, batch)
        bs.mask_build(items)
        for lg in steps:
            bs.step(lg.float() if widen else lg)
        outs.append(bs.finalize(on_device=False))
    for k in ("tokens", "item_rank", "n_live"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
    np.testing.assert_allclose(outs[0]["score"], outs[1]["score"], rtol=1e-5, atol=1e-5)


def test_bf16_argument_errors(xgr):
    rng = np.random.default_rng(1)
    items = rng.integers(0, 100, size=(500, 2)).astype(np.int32)   # V = 100: no bf16 dense steps
    x = torch.zeros((1, 8, 104), device="cuda", dtype=torch.bfloat16)
    bs = xgr.BeamSearch(100, 2, 8, 1)
    bs.mask_build(items)
    with pytest.raises(xgr.XgrError) as e:
        bs.step(torch.zeros((1, 8, 100), device="cuda", dtype=torch.bfloat16))   # ld % 8 != 0
    assert e.value.name == "XGR_ERR_ALIGNMENT"
    bs.step(x)   # sparse route (root: <= 100 children): supported
    bs.step(x)
    assert int(bs.finalize(on_device=False)["n_live"][0]) == 8
    bs2 = xgr.BeamSearch(100, 2, 8, 1, flags=xgr.XGR_CFG_NO_SPARSE_KERNEL)
    bs2.mask_build(items)
    with pytest.raises(xgr.XgrError) as e:
        bs2.step(x)   # dense route, V % 128 != 0
    assert e.value.name == "XGR_ERR_UNSUPPORTED"
    bs2.step(x.float())   # the fp32 path serves it


@pytest.mark.slow
def test_c2_full_size_bf16(xgr):
    c = config("C2")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    voc = O.Vocabulary(items, c["vocab"], c["nd"])
    B, bw = c["batch"], c["beam_width"]
    bs = _bs(xgr, voc, bw, B, flags=2)
    bs.mask_build(items)
    del items
    steps = [make_logits_torch((B, 1 if t == 0 else bw, c["vocab"]), 11 * t + 3, 2.0).to(torch.bfloat16)
             for t in range(c["nd"])]
    out, _ = run_checked(bs, voc, steps, bw, [0, 31, 63])
    assert np.all(out["n_live"] == bw)
    cnt = bs.counters()
    assert cnt["overflow"] == 0, cnt


@pytest.mark.parametrize("vocab,nd,n,bw,batch", [(16384, 3, 20_000_000, 256, 4), (65536, 2, 3_000_000, 32, 2)])
def test_bf16_cluster_rows(xgr, vocab, nd, n, bw, batch):
    """bf16 rows wider than 8192 columns: 2-CTA (V 16384, dense level-1 nodes) and 8-CTA (V 65536,
    the root row) column-split clusters."""
    items = make_items(n, vocab, nd, 9090 + vocab)
    voc = O.Vocabulary(items, vocab, nd)
    bs = _bs(xgr, voc, bw, batch, flags=2)
    bs.mask_build(items)
    steps = [make_logits_torch((batch, 1 if t == 0 else bw, vocab), 70 + t, 2.0).to(torch.bfloat16)
             for t in range(nd)]
    bs.counters()
    run_checked(bs, voc, steps, bw, list(range(batch)))
    assert bs.counters()["rows_read"] > 0
