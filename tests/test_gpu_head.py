"""LM-head fusion at sparse steps (xgr_beam_step_head): the step computes only
the legal tokens' logits from the hidden states and the bf16 LM head. The oracle computes the full
logits in fp64 from the same bf16 values (a matrix product, then its plain step); same parity bar
as tests/test_gpu_parity.py."""
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


def _head(V, d, seed, bias=True):
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn((V, d), generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    b = (torch.randn((V,), generator=g) * 0.5) if bias else None
    return w, b


def _run(xgr, items, vocab, nd, bw, batch, d, check, seed=0, bias=True, pad=0):
    voc = O.Vocabulary(items, vocab, nd)
    bs = xgr.BeamSearch(vocab, nd, bw, batch)
    bs.mask_build(items)
    w, bvec = _head(vocab, d, 100 + seed, bias)
    wd = w.cuda()
    bd = bvec.cuda() if bvec is not None else None
    hist_p, hist_t = [], []
    sc = nl = None
    used_head = 0
    for t in range(nd):
        rows = 1 if t == 0 else bw
        if t == 0:
            states = {r: O.BeamState.root() for r in check}
        else:
            states = {r: O.state_from_history([h[r] for h in hist_p], [h[r] for h in hist_t], sc[r], nl[r])
                      for r in check}
        if t > 0 and bs.next_is_sparse():
            g = torch.Generator().manual_seed(1000 * seed + t)
            hid = torch.randn((batch, rows, d + pad), generator=g).to(torch.bfloat16)
            bs.step_head(hid.cuda()[:, :, :d], wd, bd)
            used_head += 1
            hw = hid[:, :, :d].double() @ w.double().T       # [batch][rows][V], fp64
            if bvec is not None:
                hw = hw + bvec.double()
            lg = hw.numpy()
        else:
            x = make_logits((batch, rows, vocab), 300 + 10 * seed + t, 2.0)
            bs.step(torch.from_numpy(x).cuda())
            lg = x
        v = bs.view()
        par, tok = v["parent"].cpu().numpy().copy(), v["token"].cpu().numpy().copy()
        sc, nl = v["score"].cpu().numpy().copy(), v["n_live"].cpu().numpy().copy()
        for r in check:
            compare_step(voc, states[r], lg[r], bw, par[r], tok[r], sc[r], nl[r], where=f"head req {r} step {t + 1}")
        hist_p.append(par)
        hist_t.append(tok)
    out = bs.finalize(on_device=False)
    for r in check:
        for j in range(int(out["n_live"][r])):
            tup = tuple(int(a) for a in out["tokens"][r, j])
            assert voc.item_rank(tup) == int(out["item_rank"][r, j])
    return used_head


@pytest.mark.parametrize("d,bias,pad", [(256, True, 0), (512, False, 8), (1024, True, 0)])
def test_head_fusion_random_trie(xgr, d, bias, pad):
    rng = np.random.default_rng(d)
    vocab, nd, bw, batch = 1024, 3, 64, 3
    items = rng.integers(0, vocab, size=(60000, nd)).astype(np.int32)
    assert _run(xgr, items, vocab, nd, bw, batch, d, [0, 1, 2], seed=d, bias=bias, pad=pad) >= 1


def test_head_fusion_c2_shape(xgr):
    """C2 trie (10M items, V = 8192): step 3 is sparse (about 1.08 legal tokens per row)."""
    c = config("C2")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    assert _run(xgr, items, c["vocab"], c["nd"], c["beam_width"], 8, 512, [0, 5], seed=7) == 1


def test_head_route_errors(xgr):
    rng = np.random.default_rng(3)
    vocab, nd, bw = 1024, 3, 64
    items = rng.integers(0, vocab, size=(60000, nd)).astype(np.int32)
    bs = xgr.BeamSearch(vocab, nd, bw, 1)
    bs.mask_build(items)
    w = torch.zeros((vocab, 64), dtype=torch.bfloat16, device="cuda")
    h = torch.zeros((1, 1, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(xgr.XgrError) as e:
        bs.step_head(h, w)                      # the root step takes logits
    assert e.value.name == "XGR_ERR_UNSUPPORTED"
    bs.step(torch.zeros((1, 1, vocab), device="cuda"))
    if not bs.next_is_sparse():
        with pytest.raises(xgr.XgrError) as e:
            bs.step_head(torch.zeros((1, bw, 64), dtype=torch.bfloat16, device="cuda"), w)
        assert e.value.name == "XGR_ERR_UNSUPPORTED"
    with pytest.raises(xgr.XgrError) as e:
        bs.step_head(torch.zeros((1, bw, 60), dtype=torch.bfloat16, device="cuda"), w[:, :60])   # d % 8
    assert e.value.name in ("XGR_ERR_INVALID_ARG", "XGR_ERR_UNSUPPORTED")
